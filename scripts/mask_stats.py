"""Spatial structure (GPU run) of cfg3's thinning masks: fraction of active pixels vs
fraction of 4x4 / 2x2 / 1x4 / 1x8 groups containing an active pixel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolveSelective, workloads as W
cfg = W.CONFIGS["cfg3"]
_, f = W.make_input(cfg)
psf = W.make_psf(cfg.psf)
thr = {k: {"threshold": v} for k, v in W.CFG3_THRESHOLDS.items()}
for label in ("active50", "active25"):
    r = rlDeconvolveSelective(f, psf, RlConfig(iterations=150, op=K.Naive), thr[label]["threshold"], 10, thin_start=20, record_masks=True)
    m = r.masks[21:150:7].astype(bool)  # sample of thinned iterations
    def grp(a, gy, gx):
        k, h, w = a.shape
        return a.reshape(k, h // gy, gy, w // gx, gx).any(axis=(2, 4)).mean()
    print(label, "px", round(m.mean(), 3), "4x4", round(grp(m, 4, 4), 3), "2x2", round(grp(m, 2, 2), 3),
          "1x4", round(grp(m, 1, 4), 3), "2x4", round(grp(m, 2, 4), 3), "1x2", round(grp(m, 1, 2), 3), "1x8", round(grp(m, 1, 8), 3), "16x16", round(grp(m, 16, 16), 3),
          "64x64", round(grp(m, 64, 64), 3), flush=True)
