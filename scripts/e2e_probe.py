"""Phase breakdown of the host-buffer API on cfg4 (FDG_PROFILE=1 prints
per-phase milliseconds from inside fdg_rl_deconvolve)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FDG_PROFILE"] = "1"
import numpy as np, torch
import bench
from paper_1304_7211_b200 import RlConfig, OperatorKind as K, rlDeconvolve, workloads as W
from paper_1304_7211_b200._lib import Context
cfg = W.CONFIGS["cfg4"]
psf = W.make_psf(cfg.psf)
dev = torch.device("cuda", 0)
f = bench.make_input_gpu(cfg, psf, dev).cpu().numpy()
ctx = Context(0)
rc = RlConfig(iterations=100, op=K.Box2dSliding)
fp = torch.from_numpy(f).pin_memory().numpy()
for name, arr in [("pageable", f), ("pinned", fp)]:
    for rep in range(2):
        t = time.perf_counter()
        r = rlDeconvolve(arr, psf, rc, ctx=ctx)
        print(name, rep, f"{time.perf_counter() - t:.3f} s", flush=True)
