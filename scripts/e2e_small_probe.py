"""Per-call overhead of the host-buffer rlDeconvolve on a small image
(FDG_PROFILE=1 prints the phases).  usage: python scripts/e2e_small_probe.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, workloads as W  # noqa: E402
from paper_1304_7211_b200._lib import Context  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg0"
cfg = W.CONFIGS[name]
g, f = W.make_input(cfg)
psf = W.make_psf(cfg.psf)
op = {"box1d-sliding": K.Box1dSliding, "generic-box": K.GenericBox, "naive": K.Naive,
      "box2d-sliding": K.Box2dSliding}[cfg.op]
fp = torch.from_numpy(f).pin_memory().numpy()
up = torch.empty(f.shape, dtype=torch.float32).pin_memory().numpy()
ctx = Context(0)
rc = RlConfig(iterations=cfg.iterations, op=op)
for _ in range(5):
    rlDeconvolve(fp, psf, rc, ctx=ctx, out=up)
ts = []
for _ in range(20):
    a = time.perf_counter()
    r = rlDeconvolve(fp, psf, rc, ctx=ctx, out=up)
    ts.append(time.perf_counter() - a)
ts.sort()
print(f"{name}: per call median {ts[10] * 1e3:.3f} ms, loop {r.trace.totalSeconds() * 1e3:.3f} ms")

# the C call alone (arguments prepared once) vs the Python wrapper
import ctypes as C  # noqa: E402

from paper_1304_7211_b200._lib import Desc, RlRecordC, fptr, lib  # noqa: E402

d = Desc(psf)
c = rc.c()
recs = (RlRecordC * cfg.iterations)()
hh, w = f.shape
L = lib()
ts = []
for _ in range(20):
    a = time.perf_counter()
    L.fdg_rl_deconvolve(ctx.h, d.ref, C.byref(c), fptr(fp), w, hh, fptr(up), recs)
    ts.append(time.perf_counter() - a)
ts.sort()
ts2 = []
for _ in range(20):
    a = time.perf_counter()
    L.fdg_rl_deconvolve(ctx.h, d.ref, C.byref(c), fptr(fp), w, hh, fptr(up), None)
    ts2.append(time.perf_counter() - a)
ts2.sort()
print(f"C call only: {ts[10] * 1e3:.3f} ms with trace, {ts2[10] * 1e3:.3f} ms without")
