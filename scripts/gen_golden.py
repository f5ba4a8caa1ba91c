#!/usr/bin/env python
"""Generate tests/golden/golden_v1.npz from the UNMODIFIED reference.

Runs the reference library compiled from /root/reference/proj/include
(oracle/_ref/libfdref.so, built by `make ref`) on small seeded inputs and
stores inputs + outputs.  The committed fixtures pin the oracle restatement
(tests/test_oracle.py) bit-exactly without /root/reference being present.
Re-run only when the case list changes:  python scripts/gen_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import pyoracle as O  # noqa: E402
from tests.golden_cases import CONV_CASES, RL_CASES, SEL_CASES, make_psf  # noqa: E402


def main():
    assert O.ref_available(), "build the reference shim first: make ref"
    out = {}
    rng = np.random.default_rng(20261019)
    for name, (spec, kind, (h, w)) in CONV_CASES.items():
        psf = make_psf(spec)
        img = rng.random((h, w)) * 255.0
        res, cnt = O.ref_convolve(img, psf, kind, counters=True)
        out[f"conv/{name}/img"] = img
        out[f"conv/{name}/out"] = res
        out[f"conv/{name}/counters"] = cnt.astype(np.int64)
        act = (rng.random((h, w)) < 0.5).astype(np.uint8)
        fb = rng.random((h, w))
        if kind in (O.NAIVE, O.LIST):
            mres, mcnt = O.ref_masked_convolve(img, psf, kind, act, fb, counters=True)
            out[f"conv/{name}/mask"] = act
            out[f"conv/{name}/fallback"] = fb
            out[f"conv/{name}/masked"] = mres
            out[f"conv/{name}/masked_counters"] = mcnt.astype(np.int64)
    for name, (spec, op, (h, w), iters) in RL_CASES.items():
        psf = make_psf(spec)
        f = rng.random((h, w)) + 0.05
        u, mc, _ = O.ref_rl_deconvolve(f, psf, iters, op)
        out[f"rl/{name}/f"] = f
        out[f"rl/{name}/u"] = u
        out[f"rl/{name}/max_change"] = mc
    for name, (spec, op, (h, w), iters, thr, period, start) in SEL_CASES.items():
        psf = make_psf(spec)
        f = rng.random((h, w)) + 0.05
        u, inact, mc, masks = O.ref_rl_selective_from(f, psf, iters, thr, period, start, op, record_masks=True)
        out[f"sel/{name}/f"] = f
        out[f"sel/{name}/u"] = u
        out[f"sel/{name}/inactive"] = inact
        out[f"sel/{name}/max_change"] = mc
        out[f"sel/{name}/masks"] = np.packbits(masks, axis=-1)
        if start == 0:  # the reference API itself (rlDeconvolveSelective)
            u2, i2, m2 = O.ref_rl_selective(f, psf, iters, thr, period, op)
            assert np.array_equal(u, u2) and np.array_equal(inact, i2)
    path = os.path.join(ROOT, "tests", "golden", "golden_v1.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
