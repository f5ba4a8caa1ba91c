"""Every engine's device loop on planes embedded in NaN guard bands: the image
planes (f and u) sit inside larger tensors whose surrounding rows and the
columns between the image width and the row pitch hold NaN.  A read outside
the image (beyond the replicate-clamped window) would poison the result, a
write outside it would change the guard; the result must still match the CPU
oracle (rl.hpp:153-177) and every guard element must still be the same NaN.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver
from paper_1304_7211_b200 import workloads as W
from paper_1304_7211_b200._lib import check, lib
from paper_1304_7211_b200.psf import makeBoxPsf, makeDiagonalPsf, makeDiscPsf, makeLinePsf

pytestmark = pytest.mark.gpu
GY = 9  # guard rows above / below


@pytest.fixture(autouse=True)
def every_qualifying_box_fused():
    prev = lib().fdg_set_option(b"fused", 2)  # the fused kernel on these small planes too
    yield
    lib().fdg_set_option(b"fused", prev)


def _cases():
    return [
        ("fused 15x15", makeBoxPsf(15, 15), K.Box2dSliding, O.BOX2D_SLIDING, 1024, 300, 5),
        ("fused 15x15 narrow", makeBoxPsf(15, 15), K.Box2dSliding, O.BOX2D_SLIDING, 500, 40, 4),
        ("fused 5x5 ragged", makeBoxPsf(5, 5), K.Box2dSliding, O.BOX2D_SLIDING, 1021, 77, 4),
        ("fused 17x17 short", makeBoxPsf(17, 17), K.Box2dSliding, O.BOX2D_SLIDING, 640, 11, 3),
        ("fused 15x9", makeBoxPsf(15, 9), K.Box2dSliding, O.BOX2D_SLIDING, 1000, 150, 4),
        ("fused 3x17 ragged", makeBoxPsf(3, 17), K.Box2dSliding, O.BOX2D_SLIDING, 509, 60, 3),
        ("fused vertical line 1x13", makeBoxPsf(1, 13), K.Box2dSliding, O.BOX2D_SLIDING, 640, 90, 4),
        ("box 31x3", makeBoxPsf(31, 3), K.Box2dSliding, O.BOX2D_SLIDING, 700, 130, 3),
        ("rowres line 15", makeLinePsf(15), K.Box1dSliding, O.BOX1D_SLIDING, 512, 96, 6),
        ("rowres line 31 ragged", makeLinePsf(31), K.Box1dSliding, O.BOX1D_SLIDING, 1022, 50, 4),
        ("spans disc r10", W.disc_r10(), K.GenericBox, O.GENERIC_BOX, 520, 200, 3),
        ("spans oblique", W.oblique_line(), K.GenericBox, O.GENERIC_BOX, 300, 131, 4),
        ("spans disc 9 (jit)", makeDiscPsf(9), K.GenericBox, O.GENERIC_BOX, 259, 140, 3),
        ("taps diagonal 9", makeDiagonalPsf(9), K.List, O.LIST, 260, 100, 3),
        ("dense gauss31", W.gaussian31(), K.Naive, O.NAIVE, 200, 90, 2),
    ]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_engine_stays_inside_its_planes(case):
    torch = pytest.importorskip("torch")
    name, psf, op, oop, w, h, it = case
    rng = np.random.default_rng(w * 3 + h)
    g = rng.uniform(0.05, 1.0, size=(h, w)).astype(np.float32)
    f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape), 1e-6).astype(np.float32)
    pitch = ((w + 3) // 4) * 4 + 32  # >= 32 guard columns right of every row
    dev = torch.device("cuda", 0)

    def guarded():
        t = torch.full((h + 2 * GY, pitch), float("nan"), dtype=torch.float32, device=dev)
        return t, t[GY:GY + h]

    fbuf, fview = guarded()
    ubuf, uview = guarded()
    fview[:, :w] = torch.from_numpy(f).to(dev)
    solver = RlSolver(psf, RlConfig(iterations=it, op=op), w, h)
    solver._bind()
    for _ in range(2):  # eager run, then the captured graph's replay
        uview[:, :w] = float("nan")
        check(lib().fdg_solver_run(solver.h, C.c_void_p(fview.data_ptr()), C.c_void_p(uview.data_ptr()), pitch,
                                   pitch * h, it))
        torch.cuda.synchronize()
        out = uview[:, :w].cpu().numpy()
        assert np.isfinite(out).all(), f"{name} ({solver.engine()}): a read outside the image reached the result"
        ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, oop)
        assert W.max_rel(out, ref) <= 1e-4, f"{name} ({solver.engine()})"
        for buf, what in ((ubuf, "u"), (fbuf, "f")):
            b = buf.cpu().numpy()
            assert np.isnan(b[:GY]).all() and np.isnan(b[GY + h:]).all(), f"{name}: guard rows of {what} written"
            assert np.isnan(b[GY:GY + h, w:]).all(), f"{name}: guard columns of {what} written"
