"""Time the device RL loop (RlSolver.run, CUDA events) on config 4's shape for
the current FDG_* engine environment.  usage: fused_probe.py [W H iters]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver, workloads as W  # noqa: E402

w, h, it = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 4096, 10)
dev = torch.device("cuda", 0)
f = torch.rand((h, w), device=dev) + 0.1
u = torch.empty_like(f)
s = RlSolver(W.make_psf("box15x15"), RlConfig(iterations=it, op=K.Box2dSliding), w, h)
s.use_stream(torch.cuda.current_stream(dev).cuda_stream)
for _ in range(3):
    s.run(f, u)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    s.run(f, u)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5 / it
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FDG_"))
print(f"{env or 'default'}: {w}x{h} {ms:.4f} ms/iteration  {w*h/ms/1e3:.0f} Mpx*it/s", flush=True)
