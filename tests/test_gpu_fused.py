"""Single-pass RL iteration engine (kernels_fused.cu, centred 15x15 box --
config 4's Box2dSliding PSF) against the CPU oracle (rl.hpp:153-177 restated
in oracle/rl.c): odd and even iteration counts (u ping-pongs between two
planes), images narrower / wider than one column strip, fewer rows than the
box, single rows and columns, several row bands, and batched solver runs.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve
from paper_1304_7211_b200 import workloads as W

pytestmark = pytest.mark.gpu
MAX_REL = 1e-4


@pytest.fixture(autouse=True)
def fused_engine():
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"fused", 2)  # every qualifying box, whatever the image size
    yield
    lib().fdg_set_option(b"fused", prev)


def _input(w, h, seed):
    cfg = W.CONFIGS["cfg4"]
    rng = np.random.default_rng(seed)
    g = rng.uniform(0.05, 1.0, size=(h, w)).astype(np.float32)
    psf = W.make_psf(cfg.psf)
    f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape).astype(np.float32), 1e-6)
    return f.astype(np.float32), psf


@pytest.mark.parametrize("w,h,it", [(1024, 768, 25), (1024, 768, 24), (37, 23, 7), (5, 3, 4), (513, 129, 10),
                                    (600, 1, 3), (1, 50, 3), (2050, 300, 1), (301, 2050, 2), (518, 40, 9),
                                    (4, 15, 6), (8192, 20, 3)])
def test_fused_matches_oracle(w, h, it):
    f, psf = _input(w, h, w * 131 + h)
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    err = W.max_rel(res.image, ref)
    assert err <= MAX_REL, f"{w}x{h} it={it}: max-rel {err:.3e}"
    gm = np.array([r.maxAbsChange for r in res.trace.records])
    np.testing.assert_allclose(gm, mc, rtol=1e-3, atol=1e-6)


def test_fused_zero_iterations_returns_input():
    f, psf = _input(100, 60, 3)
    res = rlDeconvolve(f, psf, RlConfig(iterations=0, op=K.Box2dSliding))
    assert np.array_equal(res.image, f)


def test_fused_batched_solver():
    import torch
    from paper_1304_7211_b200 import RlSolver
    w, h, b, it = 700, 260, 3, 11
    fs = [_input(w, h, 900 + i)[0] for i in range(b)]
    psf = _input(w, h, 0)[1]
    dev = torch.device("cuda", 0)
    pitch = 704
    fd = torch.zeros((b, h, pitch), device=dev)
    for i in range(b):
        fd[i, :, :w] = torch.from_numpy(fs[i])
    ud = torch.zeros_like(fd)
    solver = RlSolver(psf, RlConfig(iterations=it, op=K.Box2dSliding), w, h, batch=b)
    solver.use_stream(torch.cuda.current_stream(dev).cuda_stream)
    for rep in range(2):  # eager + captured graph
        solver.run(fd, ud)
        torch.cuda.synchronize()
        for i in range(b):
            ref, _, _ = O.rl_deconvolve(fs[i].astype(np.float64), psf, it, O.BOX2D_SLIDING)
            err = W.max_rel(ud[i, :, :w].cpu().numpy(), ref)
            assert err <= MAX_REL, f"image {i} rep {rep}: {err:.3e}"


def test_fused_strips_match_whole_image():
    """Row strips with a 2T-row u halo (the multi-GPU fused driver), the
    neighbour exchange emulated by local copies: gathered strips equal the
    whole-image run (vertical running sums restart per band: fp32 order)."""
    import torch
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200 import sharded as S
    w, h, it, nst = 700, 300, 9, 3
    f, psf = _input(w, h, 77)
    dev = torch.device("cuda", 0)
    pitch = 704
    rc = RlConfig(iterations=it, op=K.Box2dSliding)
    solver = RlSolver(psf, rc, w, h)
    assert solver.engine() == "fused"
    solver.use_stream(torch.cuda.current_stream(dev).cuda_stream)
    fw = torch.zeros((h, pitch), device=dev)
    fw[:, :w] = torch.from_numpy(f)
    uw = torch.empty_like(fw)
    solver.run(fw, uw)
    torch.cuda.synchronize()
    whole = uw[:, :w].cpu().numpy()

    T = S.fused_halo(psf)
    strips = [S.strip_of(h, nst, r, T) for r in range(nst)]
    fs = [S.load_strip(f, s, pitch, device=dev) for s in strips]

    def exchange(bufs):
        for r in range(nst - 1):
            a, b, c = bufs[r], bufs[r + 1], strips[r].core
            b[0:T] = a[c:c + T]
            a[T + c:2 * T + c] = b[T:2 * T]

    exchange(fs)
    run = S.GpuFused(solver)
    for split in (False, True):  # split: interior rows, then the two boundary bands (the overlapped driver)
        us = [x.clone() for x in fs]
        u2 = [torch.empty_like(x) for x in fs]
        for k in range(it):
            exchange(us)
            for r, s in enumerate(strips):
                if split:
                    for rows in ((T, s.core - T), (0, T), (s.core - T, s.core)):
                        run(fs[r], us[r], u2[r], s, k, rows=rows)
                else:
                    run(fs[r], us[r], u2[r], s, k)
            us, u2 = u2, us
        torch.cuda.synchronize()
        got = np.concatenate([us[r][T:T + s.core, :w].cpu().numpy() for r, s in enumerate(strips)])
        assert W.max_rel(got, whole) <= 1e-5
        ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
        assert W.max_rel(got, ref) <= MAX_REL


def test_fused_iterate_rejects_non_fused_solver():
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200._lib import FdgInvalidArgument
    from paper_1304_7211_b200.psf import makeBoxPsf
    s = RlSolver(makeBoxPsf(21, 3), RlConfig(iterations=2, op=K.Box2dSliding), 64, 64)
    assert s.engine() != "fused"
    with pytest.raises(FdgInvalidArgument):
        s.iterate(1, 2, 3, 64, 64 * 64, 0, 64, 0, 63, 0)


@pytest.mark.parametrize("psf_name,op,spans_mode", [("disc10", K.GenericBox, 1), ("disc10", K.GenericBox, 2),
                                                    ("oblique21", K.GenericBox, 0), ("gauss31", K.Naive, 0),
                                                    ("line31", K.Box1dSliding, 0), ("box15x15", K.Box2dSliding, 0)])
def test_two_pass_strips_match_whole_image(psf_name, op, spans_mode):
    """The multi-GPU two-pass strip driver (sharded.rl_strips + GpuPasses:
    T-row halos of u and q, row ranges and clamp ranges per strip) on one
    device, the exchange emulated by local copies, for every engine the
    strips can hit: gathered strips equal the whole-image run."""
    import torch
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200 import sharded as S
    from paper_1304_7211_b200._lib import lib
    w, h, it, nst = 333, 260, 6, 3
    psf = W.make_psf(psf_name)
    rng = np.random.default_rng(5)
    f = (rng.random((h, w)) * 0.9 + 0.1).astype(np.float32)
    dev = torch.device("cuda", 0)
    pitch = 336
    prev_f = lib().fdg_set_option(b"fused", 0)  # the box goes through its two-pass kernels here
    prev_s = lib().fdg_set_option(b"spans", spans_mode)
    try:
        solver = RlSolver(psf, RlConfig(iterations=it, op=op), w, h)
        solver.use_stream(torch.cuda.current_stream(dev).cuda_stream)
        fw = torch.zeros((h, pitch), device=dev)
        fw[:, :w] = torch.from_numpy(f)
        uw = torch.empty_like(fw)
        solver.run(fw, uw)
        torch.cuda.synchronize()
        whole = uw[:, :w].cpu().numpy()

        T = S.psf_halo(psf)
        strips = [S.strip_of(h, nst, r, T) for r in range(nst)]
        fs = [S.load_strip(f, s, pitch, device=dev) for s in strips]
        qs = [torch.zeros_like(x) for x in fs]

        def exchange(bufs):
            for r in range(nst - 1):
                a, b, c = bufs[r], bufs[r + 1], strips[r].core
                b[0:T] = a[c:c + T]
                a[T + c:2 * T + c] = b[T:2 * T]

        run = S.GpuPasses(solver)
        results = []
        for split in (False, True):  # split: interior rows, then the boundary bands (the overlapped driver)
            us = [x.clone() for x in fs]
            for k in range(it):
                for which, src, aux, dst in ((1, us, fs, qs), (2, qs, us, us)):
                    exchange(src)
                    for r, s in enumerate(strips):
                        if split and T > 0 and s.core > 2 * T:
                            for rows in ((T, s.core - T), (0, T), (s.core - T, s.core)):
                                run(which, src[r], aux[r], dst[r], s, k, rows=rows)
                        else:
                            run(which, src[r], aux[r], dst[r], s, k)
            torch.cuda.synchronize()
            results.append(np.concatenate([us[r][T:T + s.core, :w].cpu().numpy() for r, s in enumerate(strips)]))
    finally:
        lib().fdg_set_option(b"fused", prev_f)
        lib().fdg_set_option(b"spans", prev_s)
    for got in results:
        assert W.max_rel(got, whole) <= 1e-5  # same engine per strip; fp32 order differs only for box running sums


def test_fused_work_balanced_segments():
    """Images large enough for the work-balanced launch (CTAs take equal
    ranges of the strip-major (strip, row) sequence, crossing strips): odd
    sizes, against the oracle."""
    w, h, it = 4001, 3999, 3
    f, psf = _input(w, h, 91)
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    assert W.max_rel(res.image, ref) <= 2e-5
    np.testing.assert_allclose([r.maxAbsChange for r in res.trace.records], mc, rtol=2e-2, atol=1e-6)


@pytest.mark.parametrize("w", [5, 13, 1023, 1024, 1025, 2048])
def test_rowres_column_split_edges(w):
    """Row-resident RL around its 4 / 8 columns-per-thread switch (1024 px)
    and for widths that are not a multiple of 4, batch of rows."""
    from paper_1304_7211_b200.psf import makeLinePsf
    rng = np.random.default_rng(w)
    f = (rng.random((7, w)) * 0.9 + 0.1).astype(np.float32)
    psf = makeLinePsf(15)
    res = rlDeconvolve(f, psf, RlConfig(iterations=12, op=K.Box1dSliding))
    ref, _, _ = O.rl_deconvolve(f.astype(np.float64), psf, 12, O.BOX1D_SLIDING)
    assert W.max_rel(res.image, ref) <= 1e-5


@pytest.mark.parametrize("m", [3, 5, 7, 9, 11, 13, 17])
@pytest.mark.parametrize("w,h,it", [(1024, 768, 12), (37, 23, 5), (5, 3, 4), (513, 129, 7), (2050, 300, 2),
                                    (600, 1, 3), (8192, 20, 3)])
def test_fused_other_boxes_match_oracle(m, w, h, it):
    """The one-launch iteration for every other centred odd square box up to
    17 x 17 (generic window sums, m-row vertical rings)."""
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200.psf import makeBoxPsf
    psf = makeBoxPsf(m, m)
    rng = np.random.default_rng(w * 7 + h + m)
    g = rng.uniform(0.05, 1.0, size=(h, w)).astype(np.float32)
    f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape), 1e-6).astype(np.float32)
    assert RlSolver(psf, RlConfig(iterations=it, op=K.Box2dSliding), w, h).engine() == "fused"
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    assert W.max_rel(res.image, ref) <= MAX_REL
    np.testing.assert_allclose([r.maxAbsChange for r in res.trace.records], mc, rtol=1e-3, atol=1e-6)


def test_fused_repeat_calls_are_bit_identical():
    """Work-balanced segments with the last column strip shifted to end at the
    image edge (2000 = 4 x 496 + 16): the overlapped columns have one writer,
    so the result does not depend on which CTA finishes last."""
    f, psf = _input(2000, 8000, 77)
    cfg = RlConfig(iterations=6, op=K.Box2dSliding)
    a = rlDeconvolve(f, psf, cfg).image
    for _ in range(3):
        assert np.array_equal(a, rlDeconvolve(f, psf, cfg).image)


@pytest.mark.parametrize("m", [5, 6, 7, 8, 9, 10, 12, 21, 22, 30, 31])
@pytest.mark.parametrize("w,h", [(700, 9), (3, 4), (1500, 5)])
def test_rowres_every_line_length(m, w, h):
    """The row-resident engine for every anchor-centred horizontal line of
    5 .. 31 px (odd and even lengths; rows wider than 1024 px use 8 columns
    per thread and need a window of at least 9), against the oracle."""
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200.psf import makeLinePsf
    rng = np.random.default_rng(m * 100 + w)
    f = (rng.random((h, w)) * 0.9 + 0.1).astype(np.float32)
    psf = makeLinePsf(m)
    expect = "rowres" if (w <= 1024 or m >= 9) else "box"
    assert RlSolver(psf, RlConfig(iterations=9, op=K.Box1dSliding), w, h).engine() == expect
    res = rlDeconvolve(f, psf, RlConfig(iterations=9, op=K.Box1dSliding))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, 9, O.BOX1D_SLIDING)
    assert W.max_rel(res.image, ref) <= 1e-5
    np.testing.assert_allclose([r.maxAbsChange for r in res.trace.records], mc, rtol=1e-3, atol=1e-6)


@pytest.mark.parametrize("mx,my", [(15, 9), (9, 15), (3, 17), (17, 3), (5, 7), (13, 11), (7, 15), (15, 3),
                                   (1, 3), (1, 9), (1, 15), (1, 17)])
@pytest.mark.parametrize("w,h,it", [(1024, 768, 9), (37, 23, 5), (513, 129, 6), (2050, 300, 2), (600, 1, 3),
                                    (8192, 20, 3)])
def test_fused_rectangular_boxes_match_oracle(mx, my, w, h, it):
    """Centred odd boxes with different extents (and vertical lines, mx = 1):
    one instantiation per horizontal radius, the vertical radius (ring height,
    halo rows) at run time."""
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200.psf import makeBoxPsf
    psf = makeBoxPsf(mx, my)
    rng = np.random.default_rng(w * 7 + h + 31 * mx + my)
    g = rng.uniform(0.05, 1.0, size=(h, w)).astype(np.float32)
    f = np.maximum(W.blur_replicate(g, psf) + rng.normal(0, 0.01, size=g.shape), 1e-6).astype(np.float32)
    assert RlSolver(psf, RlConfig(iterations=it, op=K.Box2dSliding), w, h).engine() == "fused"
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=K.Box2dSliding))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, O.BOX2D_SLIDING)
    assert W.max_rel(res.image, ref) <= MAX_REL
    np.testing.assert_allclose([r.maxAbsChange for r in res.trace.records], mc, rtol=1e-3, atol=1e-6)


def test_fused_engine_is_chosen_by_launch_size():
    """Option "fused" = 1 (the default): small launches stay on the two-pass
    path (its span-tile kernels win there: up to ~3 Mpx, ~12 Mpx for boxes of
    at most 9 px), larger ones take the one-launch iteration."""
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200._lib import lib
    from paper_1304_7211_b200.psf import makeBoxPsf
    prev = lib().fdg_set_option(b"fused", 1)
    try:
        cfg = RlConfig(iterations=3, op=K.Box2dSliding)
        assert RlSolver(makeBoxPsf(15, 15), cfg, 512, 512).engine() != "fused"
        assert RlSolver(makeBoxPsf(15, 15), cfg, 1536, 1536).engine() != "fused"
        assert RlSolver(makeBoxPsf(15, 15), cfg, 2048, 2048).engine() == "fused"
        assert RlSolver(makeBoxPsf(15, 15), cfg, 256, 256, batch=64).engine() == "fused"
        assert RlSolver(makeBoxPsf(5, 5), cfg, 3072, 3072).engine() != "fused"
        assert RlSolver(makeBoxPsf(5, 5), cfg, 4096, 4096).engine() == "fused"
        f, psf = _input(640, 480, 5)
        a = rlDeconvolve(f, psf, cfg).image
        lib().fdg_set_option(b"fused", 2)
        b = rlDeconvolve(f, psf, cfg).image
        assert W.max_rel(a, b.astype(np.float64)) <= 1e-5
    finally:
        lib().fdg_set_option(b"fused", prev)
