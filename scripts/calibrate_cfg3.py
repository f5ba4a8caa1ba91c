#!/usr/bin/env python
"""Calibrate config 3's thinning thresholds: bisect the
absolute threshold so that, with thinning from iteration 20 (period 10),
the mean active fraction over 1-based iterations 21..150 is ~50 % and ~25 %.
Uses the device's free-running selective RL on the full 4096^2 input (the
oracle's masks differ only at threshold ties), then freezes the values in
profiles/r01_cfg3_thresholds.json (full_parity.py replays the oracle masks)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolveSelective  # noqa: E402
from paper_1304_7211_b200 import workloads as W  # noqa: E402


def active(f, psf, thr):
    r = rlDeconvolveSelective(f, psf, RlConfig(iterations=150, op=K.Naive), thr, 10, thin_start=20)
    inact = np.array([x.inactiveFraction for x in r.trace.records])
    return float(1 - inact[20:].mean()), r.trace.totalSeconds()


def main():
    cfg = W.CONFIGS["cfg3"]
    _, f = W.make_input(cfg)
    psf = W.make_psf(cfg.psf)
    out = {}
    for label, target in (("active50", 0.50), ("active25", 0.25)):
        lo, hi = 1e-7, 1e-2  # active fraction decreases with the threshold
        for _ in range(30):
            mid = float(np.sqrt(lo * hi))
            a, _ = active(f, psf, mid)
            if a > target:
                lo = mid
            else:
                hi = mid
            if abs(a - target) < 0.005:
                break
        a, secs = active(f, psf, mid)
        out[label] = {"threshold": mid, "active_fraction": a, "device_loop_s": secs}
        print(label, out[label], flush=True)
    path = os.path.join(ROOT, "profiles", "r01_cfg3_thresholds.json")
    json.dump(out, open(path, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()
