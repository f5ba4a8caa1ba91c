"""Pin the CPU oracle (oracle/, a C restatement of the reference) before
trusting it as the GPU path's checker:

* against the reference's own frozen test vectors
  (proj/tests/test_convolve.cpp:60-78, test_image.cpp:36-59),
* against golden outputs of the UNMODIFIED reference committed in
  tests/golden/golden_v1.npz (scripts/gen_golden.py) -- bit-exact,
* and, where oracle/_ref (the reference compiled here) is available,
  against the live reference on fresh random inputs -- bit-exact.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import psf as P
from tests.golden_cases import CONV_CASES, RL_CASES, SEL_CASES, make_psf

GOLD = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_frozen_box1d_vectors():
    row = np.array([[1.0, 2, 3, 4, 5]])
    exp = np.array([4 / 3, 2, 3, 4, 14 / 3])
    for kind in (O.BOX1D_SLIDING, O.BOX1D_CUMUL, O.NAIVE, O.LIST):
        np.testing.assert_allclose(O.convolve(row, P.makeLinePsf(3), kind)[0], exp, atol=1e-12)
    np.testing.assert_allclose(O.convolve(np.array([[1.0, 2, 3]]), P.makeLinePsf(3), O.BOX1D_CUMUL)[0],
                               [4 / 3, 2, 8 / 3], atol=1e-12)


def test_replicate_continuation():
    # padReplicate row [1 1 1 2 3 3 3] and nearest-corner corners, seen
    # through single-tap shift PSFs (out(x) = in(clamp(x + dx)))
    row = np.array([[1.0, 2.0, 3.0]])
    for dx, exp in [(-2, [1, 1, 1]), (-1, [1, 1, 2]), (1, [2, 3, 3]), (2, [3, 3, 3])]:
        out = O.convolve(row, P.SparsePsf([(dx, 0, 1.0)]), O.LIST)
        assert out[0].tolist() == exp
    img = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert O.convolve(img, P.SparsePsf([(-2, -2, 1.0)]), O.LIST)[0, 0] == 1.0
    assert O.convolve(img, P.SparsePsf([(2, 2, 1.0)]), O.LIST)[1, 1] == 4.0


@pytest.mark.parametrize("name", sorted(CONV_CASES))
def test_conv_matches_reference_golden(gold, name):
    spec, kind, _ = CONV_CASES[name]
    psf = make_psf(spec)
    img = gold[f"conv/{name}/img"]
    out, cnt = O.convolve(img, psf, kind, counters=True)
    assert np.array_equal(out, gold[f"conv/{name}/out"])
    assert np.array_equal(cnt.astype(np.int64), gold[f"conv/{name}/counters"])
    if f"conv/{name}/masked" in gold.files:
        m, mc = O.masked_convolve(img, psf, kind, gold[f"conv/{name}/mask"], gold[f"conv/{name}/fallback"],
                                  counters=True)
        assert np.array_equal(m, gold[f"conv/{name}/masked"])
        assert np.array_equal(mc.astype(np.int64), gold[f"conv/{name}/masked_counters"])


@pytest.mark.parametrize("name", sorted(RL_CASES))
def test_rl_matches_reference_golden(gold, name):
    spec, op, _, iters = RL_CASES[name]
    u, mc, _ = O.rl_deconvolve(gold[f"rl/{name}/f"], make_psf(spec), iters, op)
    assert np.array_equal(u, gold[f"rl/{name}/u"])
    assert np.array_equal(mc, gold[f"rl/{name}/max_change"])


@pytest.mark.parametrize("name", sorted(SEL_CASES))
def test_selective_matches_reference_golden(gold, name):
    spec, op, (h, w), iters, thr, period, start = SEL_CASES[name]
    u, inact, mc, masks = O.rl_selective(gold[f"sel/{name}/f"], make_psf(spec), iters, thr, period, start, op,
                                         record_masks=True)
    assert np.array_equal(u, gold[f"sel/{name}/u"])
    assert np.array_equal(inact, gold[f"sel/{name}/inactive"])
    assert np.array_equal(mc, gold[f"sel/{name}/max_change"])
    assert np.array_equal(np.packbits(masks, axis=-1), gold[f"sel/{name}/masks"])


def test_mask_runs_restate_the_run_walk():
    m = np.array([[1, 1, 0, 1, 0, 0, 1], [0, 0, 0, 0, 0, 0, 0], [1, 1, 1, 1, 1, 1, 1]], np.uint8)
    assert O.mask_runs(m).tolist() == [[0, 0, 2], [0, 3, 1], [0, 6, 1], [2, 0, 7]]
    assert O.active_list(m).tolist() == [0, 1, 3, 6] + list(range(14, 21))


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.ref
def test_oracle_bit_identical_to_live_reference():
    rng = np.random.default_rng(5)
    psfs = [P.makeLinePsf(1), P.makeLinePsf(4), P.makeLinePsf(15), P.makeBoxPsf(5, 3), P.makeBoxPsf(15, 15),
            P.makeDiscPsf(9), P.makeDiscPsf(4), P.makeDiagonalPsf(5),
            P.SparsePsf([(2, -1, 1.0), (0, 0, 2.0), (-3, 1, 0.5)]), P.DensePsf(3, 1, 1, 0, [1, 2, 1]),
            P.DensePsf(5, 4, 1, 3, rng.random(20))]
    n = 0
    for psf in psfs:
        for kind in range(9):
            assert O.dispatch(psf, kind) == O.ref_dispatch(psf, kind)
            if O.dispatch(psf, kind) < 0 or kind == O.FOURIER:
                continue
            img = rng.random((int(rng.integers(5, 40)), int(rng.integers(5, 40)))) * 255
            a, ca = O.convolve(img, psf, kind, counters=True)
            b, cb = O.ref_convolve(img, psf, kind, counters=True)
            assert np.array_equal(a, b) and np.array_equal(ca, cb)
            n += 1
        f = rng.random((31, 27)) + 0.05
        for op in (O.AUTO, O.NAIVE):
            if O.dispatch(psf, op) < 0:
                continue
            u1, m1, _ = O.rl_deconvolve(f, psf, 12, op)
            u2, m2, _ = O.ref_rl_deconvolve(f, psf, 12, op)
            assert np.array_equal(u1, u2) and np.array_equal(m1, m2)
        for op in (O.AUTO, O.NAIVE, O.LIST):
            u1, i1, m1, k1 = O.rl_selective(f, psf, 25, 0.002, 10, 7, op, record_masks=True)
            u2, i2, m2, k2 = O.ref_rl_selective_from(f, psf, 25, 0.002, 10, 7, op, record_masks=True)
            assert np.array_equal(u1, u2) and np.array_equal(k1, k2) and np.array_equal(i1, i2)
    assert n > 50


@needs_ref
@pytest.mark.ref
def test_selective_from_zero_is_the_reference_api():
    rng = np.random.default_rng(8)
    f = rng.random((22, 25)) + 0.05
    psf = make_psf("densedisc:3")
    u1, i1, _, _ = O.ref_rl_selective_from(f, psf, 21, 0.002, 10, 0, O.NAIVE)
    u2, i2, _ = O.ref_rl_selective(f, psf, 21, 0.002, 10, O.NAIVE)
    assert np.array_equal(u1, u2) and np.array_equal(i1, i2)
