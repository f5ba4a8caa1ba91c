"""CPU-side checks of the product library (no GPU needed): the C ABI loads
and exports every symbol include/fdgpu.h declares; the plan logic
(dispatch, operatorAcceptsPsf, cost counters) agrees with the oracle /
reference rules; argument validation raises the reference's errors before
any device work; without a device, compute fails loudly (no fallback); the
BASELINE workload PSFs have the frozen geometry."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import (ConvCounters, OperatorKind as K, RlConfig, dispatch, operatorAcceptsPsf,
                                  operatorKindFromName, operatorName, rlDeconvolve, rlDeconvolveSelective,
                                  supportsMasking, workloads as W)
from paper_1304_7211_b200 import _lib
from paper_1304_7211_b200.convolve import ConvPlan, convolve
from paper_1304_7211_b200.psf import (DensePsf, SparsePsf, UniformConvexPsf, makeBoxPsf, makeDiagonalPsf,
                                      makeDiscPsf, makeLinePsf, adjoint, taps_of)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fdgpu.h")).read()
    return sorted(set(re.findall(r"\b(fdg_[a-z_0-9]+)\s*\(", src)))


def test_abi_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.lib_path())
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.fdg_abi_version() == 1


def psf_zoo():
    rng = np.random.default_rng(3)
    return [makeLinePsf(1), makeLinePsf(4), makeLinePsf(17), makeBoxPsf(9, 9), makeBoxPsf(5, 3), makeDiscPsf(9),
            makeDiscPsf(4), makeDiagonalPsf(9), SparsePsf([(0, 0, 1.0), (1, 0, 2.0)]),
            SparsePsf([(-1, 0, 1.0), (0, 0, 1.0), (1, 0, 1.0)]), DensePsf(3, 1, 1, 0, [1, 2, 1]),
            DensePsf(4, 3, 0, 2, rng.random(12)), W.disc_r10(), W.oblique_line(), W.gaussian31(),
            UniformConvexPsf([(0, -2, 2), (1, 0, 5)])]


def test_dispatch_and_acceptance_match_oracle():
    for psf in psf_zoo():
        for pref in K:
            o = O.dispatch(psf, int(pref))
            if o < 0:
                with pytest.raises(ValueError, match=operatorName(pref)):
                    dispatch(psf, pref)
                assert not operatorAcceptsPsf(pref, psf)
            else:
                assert int(dispatch(psf, pref)) == o
                assert operatorAcceptsPsf(pref, psf)


def test_reference_dispatch_table():
    # proj/tests/test_convolve.cpp:251-278 and SURVEY appendix A
    assert dispatch(makeDiscPsf(9)) == K.GenericBox
    assert dispatch(makeLinePsf(17)) == K.Box1dCumulated
    assert dispatch(makeBoxPsf(9, 9)) == K.Box2dCumulated
    assert dispatch(makeDiagonalPsf(9)) == K.List
    assert dispatch(DensePsf(3, 1, 1, 0, [1.0, 2.0, 1.0])) == K.Naive
    assert dispatch(W.disc_r10()) == K.GenericBox
    assert dispatch(W.gaussian31()) == K.Naive
    with pytest.raises(ValueError, match="box1d-sliding"):
        dispatch(makeBoxPsf(3, 3), K.Box1dSliding)


def test_names_and_masking():
    for k in K:
        assert operatorKindFromName(operatorName(k)) == k
    with pytest.raises(ValueError):
        operatorKindFromName("boxcar")
    assert supportsMasking(K.Naive) and supportsMasking(K.List) and not supportsMasking(K.GenericBox)


@pytest.mark.parametrize("w,h", [(48, 32), (17, 5)])
def test_counters_match_oracle(w, h):
    from paper_1304_7211_b200 import _lib as L
    import ctypes as C
    for psf in psf_zoo():
        for pref in K:
            if pref == K.Fourier or O.dispatch(psf, int(pref)) < 0:
                continue
            c = np.zeros(3, np.uint64)
            L.check(L.lib().fdg_op_counters(L.Desc(psf).ref, int(pref), w, h, c.ctypes.data_as(C.POINTER(C.c_uint64))))
            _, oc = O.convolve(np.ones((h, w)), psf, int(pref), counters=True)
            assert c.tolist() == oc.tolist(), (psf, pref)


def test_validation_without_device():
    f = np.ones((4, 4), np.float32)
    bad = f.copy()
    bad[1, 1] = -3
    with pytest.raises(ValueError, match="input image must be nonnegative"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    with pytest.raises(ValueError, match="epsilonDiv must be positive"):
        rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(epsilonDiv=0.0))
    with pytest.raises(ValueError, match="iterations must be >= 0"):
        rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(iterations=-1))
    with pytest.raises(ValueError, match="threshold must be >= 0"):
        rlDeconvolveSelective(f, makeBoxPsf(1, 1), RlConfig(), -0.1)
    with pytest.raises(ValueError, match="reactivation period"):
        rlDeconvolveSelective(f, makeBoxPsf(1, 1), RlConfig(), 0.1, 0)
    with pytest.raises(ValueError, match="does not support masked evaluation"):
        rlDeconvolveSelective(f, makeDiscPsf(3), RlConfig(op=K.GenericBox), 0.1)


def test_validation_in_double_before_fp32():
    """rl.hpp:78-83 on the caller's float64 values: a tiny negative that
    rounds to -0.0f is still rejected, the first offending pixel decides the
    message, and values beyond the fp32 range are refused explicitly."""
    f = np.ones((5, 7), np.float64)
    bad = f.copy()
    bad[2, 3] = -1e-46
    assert np.float32(bad[2, 3]) == 0.0
    with pytest.raises(ValueError, match="must be nonnegative"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    with pytest.raises(ValueError, match="must be nonnegative"):
        rlDeconvolveSelective(bad, makeBoxPsf(1, 1), RlConfig(), 0.1)
    bad[4, 0] = np.inf  # later in row-major order: the negative wins
    with pytest.raises(ValueError, match="must be nonnegative"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    bad[0, 1] = np.nan  # earlier: non-finite wins
    with pytest.raises(ValueError, match="non-finite"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    big = f.copy()
    big[1, 1] = 1e39
    with pytest.raises(ValueError, match="fp32 range"):
        rlDeconvolve(big, makeBoxPsf(1, 1))
    # config errors come first, like validateRlInputs
    with pytest.raises(ValueError, match="iterations must be >= 0"):
        rlDeconvolve(bad, makeBoxPsf(1, 1), RlConfig(iterations=-1))


def test_convplan_is_host_only_until_applied():
    from paper_1304_7211_b200 import ConvPlan
    p = ConvPlan(makeDiscPsf(9))
    assert p.kind() == K.GenericBox
    p = ConvPlan(makeBoxPsf(15, 15), K.Box2dSliding)
    assert p.kind() == K.Box2dSliding


@pytest.mark.skipif(_lib.device_available(), reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    with pytest.raises(_lib.FdgError, match="no CUDA"):
        rlDeconvolve(np.ones((8, 8), np.float32), makeDiscPsf(3))
    with pytest.raises(_lib.FdgError):
        convolve(np.ones((8, 8)), makeDiscPsf(3))


def test_psf_constructors_validate_like_the_reference():
    with pytest.raises(ValueError, match="anchor"):
        DensePsf(2, 2, 2, 0, [1, 1, 1, 1])
    with pytest.raises(ValueError, match="weight count"):
        DensePsf(2, 2, 0, 0, [1, 1, 1])
    with pytest.raises(ValueError, match="nonnegative"):
        DensePsf(2, 2, 0, 0, [1, -0.5, 0.2, 0.3])
    with pytest.raises(ValueError, match="positive"):
        DensePsf(2, 1, 0, 0, [0.0, 0.0])
    with pytest.raises(ValueError, match="duplicate"):
        SparsePsf([(0, 0, 1.0), (0, 0, 2.0)])
    with pytest.raises(ValueError, match="contiguous"):
        UniformConvexPsf([(0, 0, 1), (2, 0, 1)])
    # adjoint negates offsets (psf.hpp:280-308) and is an involution
    s = SparsePsf([(1, 2, 0.5), (0, 0, 0.5)])
    assert sorted((dx, dy) for dx, dy, _ in taps_of(adjoint(s))) == [(-1, -2), (0, 0)]
    d = makeDiscPsf(5)
    assert adjoint(adjoint(d)).rows == d.rows


def test_workload_psf_geometry():
    d = W.disc_r10()
    assert d.supportCount == 317 and len(d.rows) == 21
    assert [hi for _, _, hi in d.rows[:11]] == [0, 4, 6, 7, 8, 8, 9, 9, 9, 9, 10]
    o = W.oblique_line()
    assert o.supportCount == 29 and len(o.rows) == 11
    assert sorted((dx, dy) for dx, dy, _ in taps_of(o)) == sorted((-dx, -dy) for dx, dy, _ in taps_of(o))
    g = W.gaussian31()
    assert (g.width, g.height, g.anchorX, g.anchorY) == (31, 31, 15, 15)
    assert abs(sum(g.weights) - 1.0) < 1e-12
    assert not np.allclose(g.weights.reshape(31, 31), g.weights.reshape(31, 31)[::-1, ::-1])  # asymmetric


def test_scene_generator_is_seeded():
    a = W.make_input(W.CONFIGS["cfg0"], 64, 48)
    b = W.make_input(W.CONFIGS["cfg0"], 64, 48)
    assert np.array_equal(a[1], b[1]) and a[1].dtype == np.float32
    assert a[1].min() >= 1e-6
    assert 0.15 < float(np.median(a[0])) < 0.25  # background 0.2 dominates


def test_cpp_dropin_host_checks():
    exe = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/dropin_test not built (needs /root/reference headers at build time)")
    r = subprocess.run([exe, "--cpu-only"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
