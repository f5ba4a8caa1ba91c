"""One thinned cfg3 run (30 iterations: 20 full + 10 thinned at the 25 %
calibration) for an ncu launch list."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolveSelective  # noqa: E402
from paper_1304_7211_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS["cfg3"]
thr = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                  "r01_cfg3_thresholds.json")))[sys.argv[1] if len(sys.argv) > 1 else "active25"]["threshold"]
_, f = W.make_input(cfg)
r = rlDeconvolveSelective(f, W.make_psf(cfg.psf), RlConfig(iterations=32, op=K.Naive), thr, 10, thin_start=20)
print([round(x.inactiveFraction, 3) for x in r.trace.records[18:]])
print([round(x.seconds * 1e3, 3) for x in r.trace.records[18:]])
