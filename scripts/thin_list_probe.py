"""Thinned List RL (masked tap-list passes, per-tile compaction of active
pixels): device seconds per iteration against the unthinned List loop on the
same input, for a few thresholds (free-running GPU masks, reactivation every
10, thinning from iteration 20).  usage: python scripts/thin_list_probe.py [N] [iters]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, rlDeconvolveSelective  # noqa: E402
from paper_1304_7211_b200 import workloads as W  # noqa: E402
from paper_1304_7211_b200.psf import makeDiagonalPsf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
it = int(sys.argv[2]) if len(sys.argv) > 2 else 100
psf = makeDiagonalPsf(17)
g = W.scene(n, n, 7, n * n // 65536, n * n // 131072)
rng = np.random.default_rng(7)
f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, g.shape), 1e-6).astype(np.float32)
rc = RlConfig(iterations=it, op=K.List)
for _ in range(2):
    base = rlDeconvolve(f, psf, rc).trace.totalSeconds()
print(f"unthinned List {n}^2 x {it}: {base / it * 1e3:.3f} ms/it")
for thr in (0.0, 1e-4, 3e-4, 1e-3, 3e-3):
    for _ in range(2):
        r = rlDeconvolveSelective(f, psf, rc, thr, 10, thin_start=20)
    t = r.trace.totalSeconds()
    act = 1 - np.mean([x.inactiveFraction for x in r.trace.records[20:]])
    print(f"threshold {thr:g}: active {act * 100:.1f} % (it 21..), {t / it * 1e3:.3f} ms/it, speed-up {base / t:.2f}x",
          flush=True)
