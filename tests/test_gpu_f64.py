"""fdg_rl_deconvolve_f64: rlDeconvolve on the reference's own pixel type
(image.hpp: doubles).  The doubles are converted to the device's fp32 planes
chunk by chunk in the pinned staging buffers and rl.hpp:78-83 is checked on
them in the same pass, so: same result as the float call on the rounded image,
the reference's messages for the reference's cases (incl. doubles a float
check would miss), plain and strip-pipelined schedules.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve
from paper_1304_7211_b200 import workloads as W
from paper_1304_7211_b200 import _lib
from paper_1304_7211_b200._lib import Context

pytestmark = pytest.mark.gpu
MAX_REL = 1e-4


@pytest.fixture
def forced_pipeline():
    prev = _lib.lib().fdg_set_option(b"pipeline", 2)
    prev_f = _lib.lib().fdg_set_option(b"fused", 2)
    yield
    os.environ.pop("FDG_PIPE_STRIPS", None)
    _lib.lib().fdg_set_option(b"pipeline", prev)
    _lib.lib().fdg_set_option(b"fused", prev_f)


def _input64(w, h, seed, psf):
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.05, 1.0, size=(h, w))
    g[h // 3: h // 3 + max(1, h // 9), w // 4: w // 2] *= 3.0
    return np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape), 1e-6)


@pytest.mark.parametrize("name,op,oop,w,h,it", [
    ("cfg0", K.Box1dSliding, O.BOX1D_SLIDING, 300, 200, 12),
    ("cfg4", K.Box2dSliding, O.BOX2D_SLIDING, 520, 300, 9),
    ("cfg1", K.GenericBox, O.GENERIC_BOX, 257, 130, 10),
    ("cfg3", K.Naive, O.NAIVE, 96, 80, 6),
])
def test_f64_matches_oracle_and_the_float_call(name, op, oop, w, h, it):
    psf = W.make_psf(W.CONFIGS[name].psf)
    f = _input64(w, h, 3 + w, psf)
    assert f.dtype == np.float64
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=op))
    assert res.image.dtype == np.float64
    ref, mc, _ = O.rl_deconvolve(f, psf, it, oop)
    assert W.max_rel(res.image, ref) <= MAX_REL
    r32 = rlDeconvolve(f.astype(np.float32), psf, RlConfig(iterations=it, op=op))
    np.testing.assert_array_equal(res.image, r32.image.astype(np.float64))
    np.testing.assert_allclose([r.maxAbsChange for r in res.trace.records], mc, rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("w,h,it,strips", [(512, 700, 14, "100,200,300"), (2048, 9000, 3, "4500")])
def test_f64_strip_pipeline(forced_pipeline, w, h, it, strips):
    psf = W.make_psf(W.CONFIGS["cfg4"].psf)
    f = _input64(w, h, 17, psf)
    os.environ["FDG_PIPE_STRIPS"] = strips
    ctx = Context(0)
    out = np.zeros_like(f)
    rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding), ctx=ctx, out=out)
    assert ctx.last_schedule() == len(strips.split(",")) + 1
    ref, _, _ = O.rl_deconvolve(f, psf, it, O.BOX2D_SLIDING)
    assert W.max_rel(out, ref) <= MAX_REL


def test_f64_large_plain_path_uses_two_staging_chunks():
    psf = W.make_psf(W.CONFIGS["cfg0"].psf)
    f = _input64(4096, 2500, 5, psf)  # 41 MB of floats: two 32 MiB chunks each way
    res = rlDeconvolve(f, psf, RlConfig(iterations=3, op=K.Box1dSliding))
    ref, _, _ = O.rl_deconvolve(f, psf, 3, O.BOX1D_SLIDING)
    assert W.max_rel(res.image, ref) <= MAX_REL


CASES = [
    (-1e-50, "nonnegative"),       # rounds to -0.0f: a float check would let it through
    (-3.0, "nonnegative"),
    (np.nan, "non-finite"),
    (np.inf, "non-finite"),
    (1e39, "exceeds the fp32 range"),  # finite double, inf as a float
]


@pytest.mark.parametrize("bad,msg", CASES)
@pytest.mark.parametrize("pipelined", [False, True])
def test_f64_validation_on_the_doubles(forced_pipeline, bad, msg, pipelined):
    psf = W.make_psf(W.CONFIGS["cfg4"].psf)
    f = _input64(512, 600, 23, psf)
    f[577, 31] = bad
    if pipelined:
        os.environ["FDG_PIPE_STRIPS"] = "100,200"
    else:
        _lib.lib().fdg_set_option(b"pipeline", 0)
    with pytest.raises(_lib.FdgInvalidArgument, match=msg):
        rlDeconvolve(f, psf, RlConfig(iterations=3, op=K.Box2dSliding))


def test_f64_first_offender_decides():
    psf = W.make_psf(W.CONFIGS["cfg0"].psf)
    f = _input64(300, 200, 29, psf)
    f[150, 3] = np.nan
    f[20, 7] = -1e-300
    with pytest.raises(_lib.FdgInvalidArgument, match="nonnegative"):
        rlDeconvolve(f, psf, RlConfig(iterations=2, op=K.Box1dSliding))
    f[5, 5] = 1e300   # out of range, but a negative / non-finite pixel anywhere wins (rl.hpp:78-83 first)
    with pytest.raises(_lib.FdgInvalidArgument, match="nonnegative"):
        rlDeconvolve(f, psf, RlConfig(iterations=2, op=K.Box1dSliding))
    f[2, 2] = np.inf
    with pytest.raises(_lib.FdgInvalidArgument, match="non-finite"):
        rlDeconvolve(f, psf, RlConfig(iterations=2, op=K.Box1dSliding))


def test_f64_out_argument_must_be_float64():
    psf = W.make_psf(W.CONFIGS["cfg0"].psf)
    f = _input64(64, 48, 1, psf)
    with pytest.raises(_lib.FdgInvalidArgument, match="float64"):
        rlDeconvolve(f, psf, RlConfig(iterations=1, op=K.Box1dSliding), out=np.zeros(f.shape, np.float32))
