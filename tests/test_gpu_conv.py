"""GPU parity of the convolution operators against the CPU oracle.

The oracle (oracle/, pinned bit-exact to the reference in test_oracle.py)
computes in fp64; the device computes in fp32, so the bound is relative:
max|gpu - oracle| <= 2e-6 * max|oracle| per operator application
(fp32 epsilon 6e-8 times the <= 32 summands per PSF row, with margin).
Masked semantics are checked exactly (they select between values, they do
not add arithmetic).  Mirrors proj/tests/test_convolve.cpp.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import (ConvCounters, ConvPlan, OperatorKind as K, convolve, maskedConvolve,
                                  workloads as W)
from paper_1304_7211_b200.convolve import (box1dCumulatedConvolve, box1dSlidingConvolve, maskRuns)
from paper_1304_7211_b200.psf import (DensePsf, SparsePsf, UniformConvexPsf, makeBoxPsf, makeDiagonalPsf,
                                      makeDiscPsf, makeLinePsf)

pytestmark = pytest.mark.gpu
REL = 2e-6


def close(gpu, ref, rel=REL):
    scale = max(float(np.max(np.abs(ref))), 1e-30)
    err = float(np.max(np.abs(np.asarray(gpu, np.float64) - ref)))
    assert err <= rel * scale, f"max abs err {err:.3e} > {rel:.1e} * {scale:.3e}"


def psf_zoo():
    rng = np.random.default_rng(7)
    return {
        "line1": makeLinePsf(1), "line2": makeLinePsf(2), "line9": makeLinePsf(9), "line15": makeLinePsf(15),
        "line17": makeLinePsf(17), "line31": makeLinePsf(31), "line40": makeLinePsf(40),
        "box3": makeBoxPsf(3, 3), "box5x3": makeBoxPsf(5, 3), "box15": makeBoxPsf(15, 15), "box2x9": makeBoxPsf(2, 9),
        "disc1": makeDiscPsf(1), "disc4": makeDiscPsf(4), "disc9": makeDiscPsf(9), "disc17": makeDiscPsf(17),
        "disc10": W.disc_r10(), "oblique": W.oblique_line(),
        "diag5": makeDiagonalPsf(5), "diag9": makeDiagonalPsf(9),
        "sparse_asym": SparsePsf([(2, -1, 1.0), (0, 0, 2.0), (-3, 1, 0.5)]),
        "dense_blob": DensePsf(3, 1, 1, 0, [1.0, 2.0, 1.0]),
        "dense_rand": DensePsf(5, 4, 1, 3, rng.random(20)),
        "dense_wide": DensePsf(37, 3, 18, 1, rng.random(111) + 0.1),
        "gauss31": W.gaussian31(),
    }


SIZES = [(5, 5), (37, 29), (130, 67), (600, 45)]


@pytest.mark.parametrize("name", sorted(psf_zoo()))
def test_every_accepted_operator_matches_oracle(name):
    psf = psf_zoo()[name]
    rng = np.random.default_rng(abs(hash(name)) % 2**31)
    for kind in K:
        if kind == K.Fourier:
            continue
        if O.dispatch(psf, int(kind)) < 0:
            continue
        for h, w in SIZES:
            img = rng.random((h, w)) * 255.0
            img32 = img.astype(np.float32).astype(np.float64)
            ref = O.convolve(img32, psf, int(kind))
            close(convolve(img32, psf, kind), ref)


def test_fourier_is_cyclic():
    rng = np.random.default_rng(36)
    img = rng.random((8, 8)).astype(np.float32).astype(np.float64)
    psf = makeDiscPsf(3)
    close(convolve(img, psf, K.Fourier), O.convolve(img, psf, O.FOURIER))
    img = rng.random((6, 6)).astype(np.float32).astype(np.float64)
    close(convolve(img, makeBoxPsf(9, 9), K.Fourier), O.convolve(img, makeBoxPsf(9, 9), O.FOURIER))


def test_box1d_frozen_vectors():
    # proj/tests/test_convolve.cpp:60-78
    row = np.array([[1, 2, 3, 4, 5]], dtype=np.float64)
    exp = np.array([4 / 3, 2, 3, 4, 14 / 3])
    np.testing.assert_allclose(box1dSlidingConvolve(row, 3)[0], exp, rtol=1e-6)
    np.testing.assert_allclose(box1dCumulatedConvolve(row, 3)[0], exp, rtol=1e-6)
    row = np.array([[1, 2, 3]], dtype=np.float64)
    np.testing.assert_allclose(box1dCumulatedConvolve(row, 3)[0], [4 / 3, 2, 8 / 3], rtol=1e-6)


def test_identity_and_constant():
    rng = np.random.default_rng(32)
    img = rng.random((6, 9)).astype(np.float32)
    for psf, kind in [(makeBoxPsf(1, 1), K.Naive), (SparsePsf([(0, 0, 1.0)]), K.List), (makeDiscPsf(1), K.GenericBox),
                      (makeLinePsf(1), K.Box1dSliding), (makeBoxPsf(1, 1), K.Box2dSliding)]:
        assert np.array_equal(convolve(img, psf, kind), img)
    c = np.full((9, 13), 50.0, dtype=np.float32)
    for psf in [makeDiscPsf(9), makeDiagonalPsf(7), makeBoxPsf(5, 3), makeLinePsf(4), W.gaussian31()]:
        np.testing.assert_allclose(convolve(c, psf), c, rtol=2e-6)


def test_masked_semantics():
    # proj/tests/test_convolve.cpp:207-249
    rng = np.random.default_rng(37)
    img = rng.random((90, 120)).astype(np.float32)
    fb = rng.random((90, 120)).astype(np.float32)
    for psf, kind in [(W.gaussian31(), K.Naive), (makeDiagonalPsf(5), K.List), (makeDiscPsf(3), K.Naive)]:
        full = convolve(img, psf, kind)
        ones = np.ones(img.shape, np.uint8)
        assert np.array_equal(maskedConvolve(img, psf, kind, ones, fb), full)
        assert np.array_equal(maskedConvolve(img, psf, kind, np.zeros_like(ones), fb), fb)
        m = (rng.random(img.shape) < 0.5).astype(np.uint8)
        out = maskedConvolve(img, psf, kind, m, fb)
        assert np.array_equal(out, np.where(m == 1, full, fb))
    with pytest.raises(ValueError, match="does not support masked evaluation"):
        maskedConvolve(img, makeDiscPsf(3), K.GenericBox, np.ones(img.shape, np.uint8), fb)


def test_counters_on_device_plans():
    rng = np.random.default_rng(38)
    img = rng.random((32, 48))
    for psf, kind in [(makeLinePsf(9), K.List), (makeBoxPsf(17, 17), K.Box2dCumulated), (makeDiscPsf(9), K.Naive)]:
        c = ConvCounters()
        convolve(img, psf, kind, c)
        _, oc = O.convolve(img, psf, int(kind), counters=True)
        assert (c.pixels, c.perPixelOps, c.setupOps) == tuple(int(v) for v in oc)


def test_device_compaction_matches_run_walk():
    rng = np.random.default_rng(5)
    for h, w, p in [(1, 1, 0.5), (17, 33, 0.3), (64, 257, 0.7), (300, 100, 0.05)]:
        m = (rng.random((h, w)) < p).astype(np.uint8)
        idx, runs = maskRuns(m)
        assert np.array_equal(idx, O.active_list(m))
        assert np.array_equal(runs, O.mask_runs(m))


def test_engine_selection():
    assert ConvPlan(makeLinePsf(15), K.Box1dSliding).engine() == "box"
    assert ConvPlan(makeBoxPsf(15, 15), K.Box2dSliding).engine() == "box"
    assert ConvPlan(W.gaussian31(), K.Naive).engine() == "dense"
    assert ConvPlan(makeDiagonalPsf(9), K.List).engine() == "taps"
    assert ConvPlan(W.disc_r10(), K.GenericBox).engine() == "spans"
    assert ConvPlan(W.oblique_line(), K.GenericBox).engine() == "spans"
    assert ConvPlan(makeDiscPsf(9), K.GenericBox).engine() == "spans"  # runtime span table
    assert ConvPlan(convex_zoo()["wide65"], K.GenericBox).engine() == "taps"  # x extent 65 > 64
    assert ConvPlan(convex_zoo()["tall65"], K.GenericBox).engine() == "taps"  # 65 rows > 64


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", ["disc10", "oblique"])
def test_spans_kernels_both_paths(mode, name):
    """The span-table engine has a tile kernel (small images) and a marching
    kernel (large ones); force each on awkward sizes (width not a multiple of
    4, narrower than the halo, one row, several strips / bands)."""
    from paper_1304_7211_b200._lib import lib
    psf = psf_zoo()[name]
    prev = lib().fdg_set_option(b"spans", mode)
    try:
        rng = np.random.default_rng(11 + mode)
        for h, w in [(1, 7), (3, 130), (70, 9), (131, 259), (300, 513), (517, 1030)]:
            img = rng.random((h, w)).astype(np.float32).astype(np.float64)
            assert ConvPlan(psf, K.GenericBox).engine() == "spans"
            close(convolve(img, psf, K.GenericBox), O.convolve(img, psf, O.GENERIC_BOX))
    finally:
        lib().fdg_set_option(b"spans", prev)


def _oblique(length, angle_deg):
    """Row-convex rasterised line through the origin (the cfg1 rasteriser at
    another angle): UniformConvexPsf rows."""
    import math
    pts = set()
    t = -length / 2.0
    while t <= length / 2.0 + 1e-12:
        x = math.floor(t * math.cos(math.radians(angle_deg)) + 0.5)
        y = -math.floor(t * math.sin(math.radians(angle_deg)) + 0.5)
        pts.add((x, y))
        t += 0.125
    rows = {}
    for x, y in pts:
        lo, hi = rows.get(y, (x, x))
        rows[y] = (min(lo, x), max(hi, x))
    return UniformConvexPsf([(y, rows[y][0], rows[y][1]) for y in sorted(rows)])


def convex_zoo():
    """Row-convex uniform PSFs with no compile-time span table: the paper's
    discs and diagonals, lines at other angles, one-sided and wide / tall
    extremes of the runtime-table kernel (kernels_spanr.cu)."""
    z = {f"disc{d}": makeDiscPsf(d) for d in (2, 3, 5, 9, 17, 21, 31)}
    for m in (5, 9, 17):
        z[f"diag{m}"] = UniformConvexPsf([(dy, dy, dy) for dy in range(-(m // 2), m - m // 2)])
    z["anti9"] = UniformConvexPsf([(dy, -dy, -dy) for dy in range(-4, 5)])
    z["obl45_15"] = _oblique(15, 45.0)
    z["obl60_25"] = _oblique(25, 60.0)
    z["obl10_33"] = _oblique(33, 10.0)
    z["right_only"] = UniformConvexPsf([(2, 3, 7), (3, 1, 9), (4, 4, 4)])
    z["left_up"] = UniformConvexPsf([(-9, -12, -1), (-8, -20, -3)])
    z["wide64"] = UniformConvexPsf([(0, -32, 32), (1, -10, 5)])
    z["tall64"] = UniformConvexPsf([(dy, -1, 1) for dy in range(-32, 32)])
    z["wide65"] = UniformConvexPsf([(0, -32, 33)])
    z["tall65"] = UniformConvexPsf([(dy, 0, 0) for dy in range(-32, 33)])
    return z


@pytest.mark.parametrize("jit", [1, 0])
@pytest.mark.parametrize("name", sorted(set(convex_zoo()) - {"wide65", "tall65"}))
def test_runtime_span_table_kernel(name, jit):
    """GenericBox for any row-convex PSF: the tile kernel compiled for its
    table at plan time (NVRTC, spans_jit.cu) and the runtime-table kernel
    (kernels_spanr.cu), parity with the oracle (which restates
    genericBoxInto) on awkward sizes."""
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"spans_jit", jit)
    try:
        psf = convex_zoo()[name]
        assert ConvPlan(psf, K.GenericBox).engine() == "spans"
        rng = np.random.default_rng(abs(hash(name)) % 2**31)
        for h, w in [(1, 1), (1, 7), (5, 130), (70, 9), (33, 129), (131, 259), (300, 517)]:
            img = rng.random((h, w)).astype(np.float32).astype(np.float64)
            close(convolve(img, psf, K.GenericBox), O.convolve(img, psf, O.GENERIC_BOX))
    finally:
        lib().fdg_set_option(b"spans_jit", prev)


@pytest.mark.parametrize("name", ["disc10", "oblique"])
def test_runtime_span_table_forced_on_baseline_shapes(name):
    from paper_1304_7211_b200._lib import lib
    psf = psf_zoo()[name]
    prev = lib().fdg_set_option(b"spans", 3)
    try:
        rng = np.random.default_rng(21)
        for h, w in [(3, 130), (131, 259), (517, 1030)]:
            img = rng.random((h, w)).astype(np.float32).astype(np.float64)
            close(convolve(img, psf, K.GenericBox), O.convolve(img, psf, O.GENERIC_BOX))
    finally:
        lib().fdg_set_option(b"spans", prev)


@pytest.mark.parametrize("jit", [1, 0])
@pytest.mark.parametrize("name", ["disc9", "disc17", "obl60_25", "diag9"])
def test_runtime_span_table_rl(name, jit):
    """RL through the JIT tile kernel / the runtime-table kernel (fused
    quotient / update epilogues)."""
    from paper_1304_7211_b200 import RlConfig, rlDeconvolve
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"spans_jit", jit)
    try:
        _span_rl(name)
    finally:
        lib().fdg_set_option(b"spans_jit", prev)


def _span_rl(name):
    from paper_1304_7211_b200 import RlConfig, rlDeconvolve
    psf = convex_zoo()[name]
    g = W.scene(197, 143, 5, 8, 4) * 0.9 + 0.1
    f = np.maximum(O.convolve(g, psf, O.GENERIC_BOX), 1e-6).astype(np.float32)
    res = rlDeconvolve(f, psf, RlConfig(iterations=40, op=K.GenericBox))
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, 40, O.GENERIC_BOX)
    assert W.max_rel(res.image, ref) <= 1e-4
