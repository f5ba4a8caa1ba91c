"""Masked vs unmasked dense passes on config 3 (4096^2, 31x31): selective RL
at threshold 0 (every pixel active: the masked kernels do the full work) and
standard RL, device loop seconds per iteration; for ncu captures of both
kernels.  usage: python scripts/thin_probe.py [iterations] [threshold]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, rlDeconvolveSelective  # noqa: E402
from paper_1304_7211_b200 import workloads as W  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 10
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
cfg = W.CONFIGS["cfg3"]
_, f = W.make_input(cfg)
psf = W.make_psf(cfg.psf)
rc = RlConfig(iterations=it, op=K.Naive)
for rep in range(2):
    a = rlDeconvolve(f, psf, rc).trace.totalSeconds()
    b = rlDeconvolveSelective(f, psf, rc, thr, 10).trace.totalSeconds()
    print(f"standard {a / it * 1e3:.3f} ms/it   selective(thr={thr}) {b / it * 1e3:.3f} ms/it   ratio {a / b:.3f}",
          flush=True)
