"""Per-call cost of the host-buffer rlDeconvolve on the small configs (0, 1, 2):
wall time per call vs the device loop, with the C side's phase log (FDG_PROFILE)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import RlConfig, OperatorKind as K, rlDeconvolve, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import Context  # noqa: E402

ops = {"cfg0": K.Box1dSliding, "cfg1": K.GenericBox, "cfg2": K.GenericBox}
ctx = Context(0)
for name in ("cfg0", "cfg1", "cfg2"):
    cfg = W.CONFIGS[name]
    g, f = W.make_input(cfg)
    psf = W.make_psf(cfg.psf)
    fp = torch.from_numpy(f.astype(np.float32)).pin_memory().numpy()
    out = torch.empty(fp.shape, dtype=torch.float32).pin_memory().numpy()
    rc = RlConfig(iterations=cfg.iterations, op=ops[name])
    for _ in range(5):
        rlDeconvolve(fp, psf, rc, ctx=ctx, out=out)
    n = 50
    t0 = time.perf_counter()
    for _ in range(n):
        res = rlDeconvolve(fp, psf, rc, ctx=ctx, out=out)
    dt = (time.perf_counter() - t0) / n
    dev = sum(r.seconds for r in res.trace.records)
    px = f.shape[0] * f.shape[1] * cfg.iterations
    print(f"{name}: {dt * 1e6:.0f} us per call ({px / dt / 1e6:.0f} Mpx*it/s), device loop {dev * 1e6:.0f} us "
          f"({px / dev / 1e6:.0f} Mpx*it/s), host overhead {(dt - dev) * 1e6:.0f} us", flush=True)
