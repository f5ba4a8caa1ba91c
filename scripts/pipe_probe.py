"""Time-skewed strip pipeline (fdg_rl_deconvolve on page-locked buffers, fused
engine) against the plain upload / iterate / download path: same call, option
"pipeline" 0 / 1; result difference and wall time per call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import RlConfig, OperatorKind, rlDeconvolve, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import Context, lib  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "16384"
width, height = (int(v) for v in arg.split("x")) if "x" in arg else (int(arg), int(arg))  # SIZE or WxH
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
pinned = (sys.argv[4] if len(sys.argv) > 4 else "pinned") == "pinned"
f64 = len(sys.argv) > 5 and sys.argv[5] == "f64"  # the reference's pixel type (pageable doubles)
cfg = W.CONFIGS["cfg4"]
ctx = Context(0)
rng = np.random.default_rng(4)
f = (0.2 + 0.8 * rng.random((height, width), dtype=np.float32))
f[height // 3: height // 3 + 900, :] *= 0.25  # structure, so iterations move
psf = W.make_psf(cfg.psf)
fp = f.astype(np.float64) if f64 else (torch.from_numpy(f).pin_memory().numpy() if pinned else f)
outs = {}
for mode in (0, 2, 1):  # never, forced, the library's own choice
    lib().fdg_set_option(b"pipeline", mode)
    up = np.empty_like(fp) if f64 else (torch.empty(f.shape, dtype=torch.float32).pin_memory().numpy() if pinned else np.empty_like(f))
    rc = RlConfig(iterations=iters, op=OperatorKind.Box2dSliding)
    for _ in range(2):
        res = rlDeconvolve(fp, psf, rc, ctx=ctx, out=up)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        res = rlDeconvolve(fp, psf, rc, ctx=ctx, out=up)
    dt = (time.perf_counter() - t0) / reps
    outs[mode] = up.copy()
    res = rlDeconvolve(fp, psf, rc, ctx=ctx, out=up)
    print(f"  repeat call bit-identical: {np.array_equal(outs[mode], up)}")
    tr = res.trace.records
    print(f"{'float64' if f64 else 'pinned' if pinned else 'pageable'} pipeline={mode}: {dt * 1e3:.2f} ms per call, {width * height * iters / dt / 1e6:.0f} Mpx*it/s e2e; "
          f"trace maxc[0]={tr[0].maxAbsChange:.4g} maxc[-1]={tr[-1].maxAbsChange:.4g} "
          f"sum(sec)={sum(r.seconds for r in tr) * 1e3:.2f} ms, schedule {ctx.last_schedule()}", flush=True)
d = np.abs(outs[0] - outs[2])
rel = d / np.maximum(np.abs(outs[0]), 1e-6)
print(f"pipelined vs plain: max abs {d.max():.3e}, max rel {rel.max():.3e}")
