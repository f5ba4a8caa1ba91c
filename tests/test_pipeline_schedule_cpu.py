"""The time-skewed strip schedule of the host-buffer rlDeconvolve (fdgpu.cu
rl_pipelined), checked as a schedule -- no device: strip s runs
ALL its iterations before strip s + 1, iteration k of strip s writes rows
[a_s - D k, a_{s+1} - D k) of plane k % 2 and reads rows within D of them from
plane (k - 1) % 2 (iteration 0 reads f).  For the layouts the library chooses
(fdg_pipeline_layout) and for hand-made ones, replaying the launches in issue
order against a model of the two planes must find, for every row a launch
reads, exactly the previous iteration's value -- i.e. the loop of
rl.hpp:153-177 is evaluated with nothing recomputed, nothing stale and nothing
overwritten early.
"""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1304_7211_b200._lib import lib


def layout(height, shift, iters, width=16384):
    buf = (C.c_int * 64)()
    n = lib().fdg_pipeline_layout(width, height, shift, iters, buf, 64)
    assert 1 <= n <= 64
    return [buf[i] for i in range(n)]


def ranges(a, height, shift, k):
    """[lo, hi) of every strip at iteration k (rl_pipelined's clipping)."""
    n = len(a)
    out = []
    for s in range(n):
        lo = 0 if s == 0 else min(height, max(0, a[s] - shift * k))
        hi = height if s == n - 1 else min(height, max(0, a[s + 1] - shift * k))
        out.append((lo, hi))
    return out


def replay(a, height, shift, iters):
    """Issue order: strip 0's iterations, then strip 1's, ...  planes[p][r] =
    the iteration whose result row r of plane p currently holds (-1: nothing);
    the last iteration writes the result plane, iteration 0 reads f."""
    planes = [np.full(height, -1), np.full(height, -1)]
    result = np.full(height, -1)
    for s in range(len(a)):
        for k in range(iters):
            lo, hi = ranges(a, height, shift, k)[s]
            if hi <= lo:
                continue
            r0, r1 = max(0, lo - shift), min(height, hi + shift)
            if k > 0:
                src = planes[(k - 1) & 1][r0:r1]
                assert (src == k - 1).all(), (
                    f"strip {s} iteration {k} rows [{lo}, {hi}) reads rows [{r0}, {r1}) of plane {(k - 1) & 1}: "
                    f"found iterations {sorted(set(src.tolist()))}, need {k - 1}")
            dst = result if k == iters - 1 else planes[k & 1]
            dst[lo:hi] = k
    assert (result == iters - 1).all(), "every row must receive the last iteration exactly from its strip"


CASES = [(16384, 14, 100), (8192, 14, 100), (4096, 14, 37), (700, 14, 30), (300, 8, 50), (64, 16, 9), (20, 14, 5),
         (5000, 2, 200), (1, 14, 3), (4097, 16, 1), (4097, 16, 2)]


@pytest.mark.parametrize("height,shift,iters", CASES)
def test_library_layout_is_a_valid_schedule(height, shift, iters):
    os.environ.pop("FDG_PIPE_STRIPS", None)
    os.environ.pop("FDG_PIPE_K0", None)
    a = layout(height, shift, iters)
    assert a[0] == 0 and all(x < y for x, y in zip(a, a[1:]))
    for k in range(iters):
        r = ranges(a, height, shift, k)
        assert r[0][0] == 0 and r[-1][1] == height
        assert all(r[i][1] == r[i + 1][0] for i in range(len(r) - 1)), "strips tile the image at every iteration"
    replay(a, height, shift, iters)


def test_layouts_follow_the_timeline_model():
    """Few strips when launches are dear relative to the copies (many
    iterations, small images), more when the copies dominate."""
    os.environ.pop("FDG_PIPE_STRIPS", None)
    os.environ.pop("FDG_PIPE_K0", None)
    cfg4 = layout(16384, 14, 100)
    assert cfg4[0] == 0 and cfg4[-1] == 16384 - 64 and 4 <= len(cfg4) <= 6
    assert len(layout(8192, 14, 100, width=8192)) <= len(cfg4)
    assert len(layout(16384, 14, 1000)) <= len(cfg4)
    for w in (2048, 8192, 16384):
        replay(layout(8192, 14, 40, width=w), 8192, 14, 40)


@pytest.mark.parametrize("strips,k0", [("100,200,300", None), ("64,64,64,64", None), ("16,16", None),
                                       ("200,250", "6"), ("100", "1"), ("300,300", "29")])
def test_env_layouts_are_valid_schedules(strips, k0):
    os.environ["FDG_PIPE_STRIPS"] = strips
    if k0 is not None:
        os.environ["FDG_PIPE_K0"] = k0
    try:
        a = layout(700, 14, 30)
        if k0 is not None:
            assert a[-1] >= 700  # the last boundary starts at or below the image's end
        replay(a, 700, 14, 30)
    finally:
        os.environ.pop("FDG_PIPE_STRIPS", None)
        os.environ.pop("FDG_PIPE_K0", None)


def test_replay_catches_a_schedule_that_does_not_slide():
    """The model is a real check: strips that keep their rows (no skew) read
    rows their lower neighbour has not produced yet."""
    with pytest.raises(AssertionError):
        replay_fixed([0, 100, 200], 300, 14, 5)


def replay_fixed(a, height, shift, iters):
    planes = [np.full(height, -1), np.full(height, -1)]
    for s in range(len(a)):
        lo, hi = a[s], (a[s + 1] if s + 1 < len(a) else height)
        for k in range(iters):
            if k > 0:
                src = planes[(k - 1) & 1][max(0, lo - shift):min(height, hi + shift)]
                assert (src == k - 1).all()
            planes[k & 1][lo:hi] = k
