"""Device loop of the box engines by PSF size: fused one-launch iteration vs the
two-pass box engine (square boxes, 4096^2) and the row-resident engine vs the
two-pass box engine (horizontal lines, 512^2 x 100 iterations like config 0)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1304_7211_b200 import RlConfig, OperatorKind as K, RlSolver  # noqa: E402
from paper_1304_7211_b200.psf import makeBoxPsf, makeLinePsf  # noqa: E402
from paper_1304_7211_b200._lib import lib  # noqa: E402


def rate(solver, f, u, it, reps=3):
    for _ in range(2):
        solver.run(f, u)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        solver.run(f, u)
    torch.cuda.synchronize()
    return f.numel() * it * reps / (time.perf_counter() - t0) / 1e6


what = sys.argv[1] if len(sys.argv) > 1 else "boxes"
if what == "rects":
    n, it = 4096, 50
    f = torch.rand(n, n, device='cuda') + 0.1
    u = torch.empty_like(f)
    for mx, my in ((15, 9), (9, 15), (17, 5), (5, 17), (7, 13), (1, 9), (1, 15)):
        for fused in (0, 1):
            lib().fdg_set_option(b"fused", fused)
            s = RlSolver(makeBoxPsf(mx, my), RlConfig(iterations=it, op=K.Box2dSliding), n, n)
            print(f"box {mx}x{my} 4096^2: engine {s.engine():6s} {rate(s, f, u, it):9.0f} Mpx*it/s")
elif what == "boxes":
    n, it = 4096, 50
    f = torch.rand(n, n, device='cuda') + 0.1
    u = torch.empty_like(f)
    for m in (3, 5, 7, 11, 13):
        for fused in (0, 1):
            lib().fdg_set_option(b"fused", fused)
            s = RlSolver(makeBoxPsf(m, m), RlConfig(iterations=it, op=K.Box2dSliding), n, n)
            print(f"box {m}x{m} 4096^2: engine {s.engine():6s} {rate(s, f, u, it):9.0f} Mpx*it/s")
else:
    import os
    n, it = 512, 100
    f = torch.rand(n, n, device='cuda') + 0.1
    u = torch.empty_like(f)
    for m in (5, 7, 11, 21, 25, 30):
        s = RlSolver(makeLinePsf(m), RlConfig(iterations=it, op=K.Box1dSliding), n, n)
        print(f"line {m} 512^2 x {it}: engine {s.engine():6s} {rate(s, f, u, it, 20):9.0f} Mpx*it/s "
              f"(FDG_NO_ROWRES={os.environ.get('FDG_NO_ROWRES', '')})")
