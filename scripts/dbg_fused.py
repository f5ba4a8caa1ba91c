import sys, numpy as np
sys.path.insert(0, '.')
from paper_1304_7211_b200 import RlConfig, rlDeconvolve, OperatorKind as K, workloads as W
from paper_1304_7211_b200._lib import lib
from paper_1304_7211_b200.psf import makeBoxPsf
for (w, h, it) in [(1024, 768, 1), (1024, 768, 2), (1000, 300, 1), (2000, 300, 1)]:
    rng = np.random.default_rng(5)
    f = (rng.random((h, w)) + 0.1).astype(np.float32)
    psf = makeBoxPsf(15, 15)
    lib().fdg_set_option(b"fused", 1)
    a = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding)).image
    lib().fdg_set_option(b"fused", 0)
    b = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding)).image
    lib().fdg_set_option(b"fused", 1)
    err = np.abs(a - b) / b
    bad = np.argwhere(err > 1e-5)
    print(w, h, it, "max", err.max(), "nbad", len(bad))
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("  rows", ys.min(), ys.max(), "cols", np.unique(xs)[:20], np.unique(xs)[-10:])
