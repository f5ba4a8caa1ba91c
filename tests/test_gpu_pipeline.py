"""Time-skewed strip pipeline of the host-buffer rlDeconvolve (fdgpu.cu
rl_pipelined: page-locked buffers, fused engine): strip s runs all its
iterations before strip s + 1, its rows sliding up by the iteration's
dependency radius, so uploads / downloads overlap the loop.  The loop it must
reproduce is rl.hpp:153-177 (oracle/rl.c): every strip layout is checked
against the CPU oracle, including strips that shrink to nothing, boundaries
clipped at row 0, 1 / 2 iterations (first reads f, last writes the result
plane), the 9x9 / 17x17 boxes, input validation on late chunks and the
per-iteration trace.
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve
from paper_1304_7211_b200 import psf as P
from paper_1304_7211_b200 import workloads as W
from paper_1304_7211_b200 import _lib

pytestmark = pytest.mark.gpu
MAX_REL = 1e-4


@pytest.fixture(autouse=True)
def forced_pipeline():
    prev_f = _lib.lib().fdg_set_option(b"fused", 2)
    prev = _lib.lib().fdg_set_option(b"pipeline", 2)
    old = os.environ.pop("FDG_PIPE_STRIPS", None)
    yield
    os.environ.pop("FDG_PIPE_STRIPS", None)
    if old is not None:
        os.environ["FDG_PIPE_STRIPS"] = old
    _lib.lib().fdg_set_option(b"pipeline", prev)
    _lib.lib().fdg_set_option(b"fused", prev_f)


def _pinned(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


def _input(w, h, seed, psf=None):
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.05, 1.0, size=(h, w)).astype(np.float32)
    g[h // 3: h // 3 + max(1, h // 9), w // 4: w // 2] *= 3.0
    psf = psf if psf is not None else W.make_psf(W.CONFIGS["cfg4"].psf)
    f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape).astype(np.float32), 1e-6)
    return f.astype(np.float32), psf


def _run(f, psf, it, strips=None):
    if strips:
        os.environ["FDG_PIPE_STRIPS"] = strips
    else:
        os.environ.pop("FDG_PIPE_STRIPS", None)
    fp = _pinned(f)
    out = _pinned(np.zeros_like(f))
    res = rlDeconvolve(fp, psf, RlConfig(iterations=it, op=K.Box2dSliding), out=out)
    return out, res


# (w, h, iterations, strip heights): D = 14 rows per iteration for the 15x15 box
CASES = [
    (512, 700, 30, "100,200,300"),   # strips 0 and 1 shrink to nothing, strip 2 clipped at row 0
    (512, 700, 30, None),            # default layout
    (1024, 900, 25, "64,64,64,64"),  # many short strips, all vanish but the last
    (2000, 1500, 12, "500,500"),     # nothing vanishes; last column strip shifted (2000 = 4 * 496 + 16)
    (512, 300, 1, "100,100"),        # one iteration: f -> result plane
    (512, 300, 2, "100,100"),        # two: f -> plane 0 -> result plane
    (496, 64, 40, "16,16"),          # image shorter than the total shift
    (1536, 2200, 7, "1024"),
]


@pytest.mark.parametrize("w,h,it,strips", CASES)
def test_pipelined_matches_oracle(w, h, it, strips):
    f, psf = _input(w, h, w + 7 * h + it)
    out, res = _run(f, psf, it, strips)
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    err = W.max_rel(out, ref)
    assert err <= MAX_REL, f"{w}x{h} it={it} strips={strips}: max-rel {err:.3e}"
    gm = np.array([r.maxAbsChange for r in res.trace.records])
    np.testing.assert_allclose(gm, mc, rtol=1e-3, atol=1e-6)
    assert all(r.seconds > 0 for r in res.trace.records)


@pytest.mark.parametrize("m,my", [(3, 3), (5, 5), (9, 9), (17, 17), (15, 9), (5, 13)])
def test_pipelined_other_boxes(m, my):
    psf = P.makeBoxPsf(m, my)  # the strips slide by 2 x the vertical radius
    f, _ = _input(1024, 640, m + my, psf)
    out, _ = _run(f, psf, 15, "100,260")
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, 15, O.BOX2D_SLIDING)
    assert W.max_rel(out, ref) <= MAX_REL


def test_pipelined_is_the_path_taken_and_matches_plain():
    """Same call with the option off: the two schedules agree to rounding
    (running-sum segments differ), both are repeatable bit for bit, and the
    pipelined call launches one kernel per (strip, iteration)."""
    from paper_1304_7211_b200._lib import Context
    f, psf = _input(1024, 1200, 5)
    ctx = Context(0)
    os.environ["FDG_PIPE_STRIPS"] = "300,500"
    fp, o1, o2, o3 = _pinned(f), _pinned(np.zeros_like(f)), _pinned(np.zeros_like(f)), _pinned(np.zeros_like(f))
    cfg = RlConfig(iterations=10, op=K.Box2dSliding)
    n0 = ctx.launch_count()
    rlDeconvolve(fp, psf, cfg, ctx=ctx, out=o1)
    n1 = ctx.launch_count()
    rlDeconvolve(fp, psf, cfg, ctx=ctx, out=o2)
    assert np.array_equal(o1, o2)
    assert n1 - n0 >= 3 * 10  # 3 strips x 10 iterations (+ stamp, validation)
    assert ctx.last_schedule() == 3
    _lib.lib().fdg_set_option(b"pipeline", 0)
    rlDeconvolve(fp, psf, cfg, ctx=ctx, out=o3)
    assert ctx.last_schedule() == 0
    assert W.max_rel(o1, o3.astype(np.float64)) <= 2e-5


@pytest.mark.parametrize("w,h,it,strips,pin_in,pin_out", [
    (512, 400, 5, "100,150", False, False),     # small pageable arrays: plain copies inside the pipeline
    (2048, 9000, 3, "4500", False, False),      # > 32 MiB per strip: two staging chunks up and down
    (2048, 9000, 3, "3000,3000", True, False),  # page-locked in, pageable out
    (2048, 9000, 3, "3000,3000", False, True),
])
def test_pipelined_pageable_buffers(w, h, it, strips, pin_in, pin_out):
    """Pageable buffers go through the context's pinned staging chunks, strip
    by strip, behind the launches of the previous strip."""
    from paper_1304_7211_b200._lib import Context
    f, psf = _input(w, h, 11 + w + h)
    os.environ["FDG_PIPE_STRIPS"] = strips
    ctx = Context(0)
    fin = _pinned(f) if pin_in else f
    out = _pinned(np.zeros_like(f)) if pin_out else np.zeros_like(f)
    rlDeconvolve(fin, psf, RlConfig(iterations=it, op=K.Box2dSliding), ctx=ctx, out=out)
    assert ctx.last_schedule() == len(strips.split(",")) + 1
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    assert W.max_rel(out, ref) <= MAX_REL


@pytest.mark.parametrize("bad,msg", [(-1.0, "nonnegative"), (np.nan, "non-finite"), (np.inf, "non-finite")])
def test_pipelined_validates_late_chunks(bad, msg):
    """rl.hpp:78-83: a bad pixel in the last uploaded chunk is still reported
    (the verdict is read after the loop)."""
    f, psf = _input(512, 600, 13)
    f[590, 17] = bad
    with pytest.raises(_lib.FdgInvalidArgument, match=msg):
        _run(f, psf, 4, "100,200")


def test_pipelined_first_offender_decides_the_message():
    f, psf = _input(512, 600, 14)
    f[50, 3] = -2.0     # first chunk
    f[580, 3] = np.nan  # last chunk: later in row-major order
    with pytest.raises(_lib.FdgInvalidArgument, match="nonnegative"):
        _run(f, psf, 3, "100,200")
    f[10, 3] = np.nan
    with pytest.raises(_lib.FdgInvalidArgument, match="non-finite"):
        _run(f, psf, 3, "100,200")


def test_pipelined_in_place_call_takes_the_plain_path():
    from paper_1304_7211_b200._lib import Context
    f, psf = _input(512, 400, 21)
    ctx = Context(0)
    buf = _pinned(f)
    rlDeconvolve(buf, psf, RlConfig(iterations=5, op=K.Box2dSliding), ctx=ctx, out=buf)
    assert ctx.last_schedule() == 0
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, 5, O.BOX2D_SLIDING)
    assert W.max_rel(buf, ref) <= MAX_REL


def test_pipelined_late_born_last_strip():
    """FDG_PIPE_K0: the last boundary starts below the image, the last strip is
    empty until iteration k0 and grows afterwards."""
    f, psf = _input(512, 700, 31)
    os.environ["FDG_PIPE_K0"] = "6"
    try:
        out, _ = _run(f, psf, 14, "200,250")
    finally:
        os.environ.pop("FDG_PIPE_K0", None)
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, 14, O.BOX2D_SLIDING)
    assert W.max_rel(out, ref) <= MAX_REL


def test_pipelined_nan_in_iterate_reported():
    """rl.hpp:96-99,173 through the strip schedule: the NaN flag of an
    iteration accumulates over the strips' launches."""
    f = np.ones((700, 512), np.float32)
    f[450:520, 100:300] = 3.0e38  # overflows the fp32 window sums in a late strip
    with pytest.raises(_lib.FdgNaNError, match=r"rlDeconvolve: NaN in iterate at iteration \d+"):
        _run(f, W.make_psf(W.CONFIGS["cfg4"].psf), 8, "100,200")
