import sys, numpy as np
sys.path.insert(0, '.')
from paper_1304_7211_b200 import convolve, OperatorKind as K, makeBoxPsf, ConvPlan
psf = makeBoxPsf(15, 15)
rng = np.random.default_rng(0)
for kind in [K.Box2dSliding]:
    for (h, w) in [(130, 67), (600, 45), (37, 29), (5, 5), (45, 600)]:
        print(kind.name, h, w, ConvPlan(psf, kind).engine(), flush=True)
        convolve(rng.random((h, w)), psf, kind)
        print("  ok", flush=True)
