"""Device-loop RL throughput of every engine on one image size (the engines
no BASELINE config exercises included): Mpx*it/s, the solver's engine, and
the canonical 24 B/px*it HBM fraction.  usage: python scripts/engine_probe.py [N] [iters]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver, workloads as W  # noqa: E402
from paper_1304_7211_b200.psf import (SparsePsf, makeBoxPsf, makeDiagonalPsf, makeDiscPsf,  # noqa: E402
                                      makeLinePsf)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
PEAK = 6549.4e9
cases = [
    ("box 9x9 box2d", makeBoxPsf(9, 9), K.Box2dSliding),
    ("box 17x17 box2d", makeBoxPsf(17, 17), K.Box2dSliding),
    ("box 31x3 box2d", makeBoxPsf(31, 3), K.Box2dSliding),
    ("box 15x15 box2d-cumul", makeBoxPsf(15, 15), K.Box2dCumulated),
    ("line 9 box1d", makeLinePsf(9), K.Box1dSliding),
    ("line 40 box1d", makeLinePsf(40), K.Box1dSliding),
    ("disc 9 generic", makeDiscPsf(9), K.GenericBox),
    ("disc 17 generic", makeDiscPsf(17), K.GenericBox),
    ("disc 31 generic", makeDiscPsf(31), K.GenericBox),
    ("diag 9 list", makeDiagonalPsf(9), K.List),
    ("diag 17 list", makeDiagonalPsf(17), K.List),
    ("disc 9 list", SparsePsf([(dx, dy, 1.0) for dx, dy, _ in __import__("paper_1304_7211_b200.psf", fromlist=["taps_of"]).taps_of(makeDiscPsf(9))]), K.List),
    ("gauss 31 naive", W.gaussian31(), K.Naive),
    ("box 9x9 naive", makeBoxPsf(9, 9), K.Naive),
]
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
f = torch.rand((n, n), device=dev, generator=g) * 0.8 + 0.2
u = torch.empty_like(f)
st = torch.cuda.current_stream(dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, psf, op in cases:
    s = RlSolver(psf, RlConfig(iterations=iters, op=op), n, n)
    s.use_stream(st.cuda_stream)
    for _ in range(2):
        s.run(f, u, iters)
    e0.record(st)
    s.run(f, u, iters)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    v = n * n * iters / (ms * 1e-3) / 1e6
    print(f"{name:24s} {s.engine():12s} {v:10.0f} Mpx*it/s  {v * 1e6 * 24 / PEAK:5.2f} of HBM (24 B/px*it)", flush=True)
