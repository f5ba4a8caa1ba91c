"""rlDeconvolveBatch on config 4b's batch: wall time per call with 0 and 100
iterations (page-locked buffers), against the device loop alone."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolveBatch, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import Context  # noqa: E402

cfg = W.CONFIGS["cfg4b"]
psf = W.make_psf(cfg.psf)
rng = np.random.default_rng(0)
imgs = (rng.random((cfg.batch, cfg.height, cfg.width), dtype=np.float32) * 0.8 + 0.2)
fp = torch.from_numpy(imgs).pin_memory().numpy()
up = torch.empty(imgs.shape, dtype=torch.float32).pin_memory().numpy()
ctx = Context(0)
for it in (0, 100):
    rc = RlConfig(iterations=it, op=K.Box1dSliding)
    for _ in range(2):
        rlDeconvolveBatch(fp, psf, rc, ctx=ctx, out=up)
    ts = []
    for _ in range(3):
        a = time.perf_counter()
        r = rlDeconvolveBatch(fp, psf, rc, ctx=ctx, out=up)
        ts.append(time.perf_counter() - a)
    loop = r.trace.totalSeconds() if it else 0.0
    print(f"iterations {it}: {min(ts) * 1e3:.1f} ms per call, device loop (summed over chunks) {loop * 1e3:.1f} ms")
