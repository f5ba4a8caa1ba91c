import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, workloads as W
from paper_1304_7211_b200._lib import Context
import bench
cfg = W.CONFIGS["cfg4"]
psf = W.make_psf(cfg.psf)
dev = torch.device("cuda", 0)
f = bench.make_input_gpu(cfg, psf, dev).cpu()
fp = f.pin_memory().numpy()
ctx = Context(0)
rc = RlConfig(iterations=100, op=K.Box2dSliding)
for _ in range(3): rlDeconvolve(fp, psf, rc, ctx=ctx)
for _ in range(3):
    torch.cuda.synchronize(); a = time.perf_counter(); r = rlDeconvolve(fp, psf, rc, ctx=ctx); print("e2e ms", (time.perf_counter() - a) * 1e3, "loop ms", r.trace.totalSeconds() * 1e3, flush=True)
