import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1304_7211_b200 import RlConfig, OperatorKind as K, RlSolver
from paper_1304_7211_b200.psf import makeBoxPsf
from paper_1304_7211_b200._lib import lib
n = 4096; it = 50
f = torch.rand(n, n, device='cuda') + 0.1
u = torch.empty_like(f)
for m in (3, 5, 7, 11, 13):
    for fused in (0, 1):
        lib().fdg_set_option(b"fused", fused)
        s = RlSolver(makeBoxPsf(m, m), RlConfig(iterations=it, op=K.Box2dSliding), n, n)
        for _ in range(2): s.run(f, u)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(3): s.run(f, u)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 3
        print(f"box {m}x{m} 4096^2: engine {s.engine():6s} {n*n*it/dt/1e6:9.0f} Mpx*it/s")
