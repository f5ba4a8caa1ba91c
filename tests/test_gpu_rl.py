"""GPU Richardson-Lucy parity against the CPU oracle on the BASELINE
configurations (full size where the oracle finishes in seconds, the same
seeded generator at reduced size otherwise) -- the north-star bound:
max-rel <= 1e-4 after the configured iteration count and
|PSNR(u_gpu, g) - PSNR(u_ref, g)| <= 0.01 dB (peak 1).
Also the RL invariants of proj/tests/test_rl.cpp.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import (OperatorKind as K, RlConfig, rlDeconvolve, rlDeconvolveSelective, rlStep,
                                  workloads as W)
from paper_1304_7211_b200.convolve import convolve, maskRuns
from paper_1304_7211_b200.psf import makeBoxPsf, makeDiagonalPsf, makeDiscPsf, makeLinePsf

pytestmark = pytest.mark.gpu
MAX_REL = 1e-4
DPSNR = 0.01

OPS = {"box1d-sliding": K.Box1dSliding, "box2d-sliding": K.Box2dSliding, "generic-box": K.GenericBox,
       "naive": K.Naive}


def run_config(name, w=None, h=None, iterations=None):
    cfg = W.CONFIGS[name]
    g, f = W.make_input(cfg, w, h)
    psf = W.make_psf(cfg.psf)
    it = iterations or cfg.iterations
    op = OPS[cfg.op]
    res = rlDeconvolve(f, psf, RlConfig(iterations=it, op=op))
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, int(op))
    err = W.max_rel(res.image, ref)
    dp = abs(W.psnr(res.image, g) - W.psnr(ref, g))
    assert err <= MAX_REL, f"{name}: max-rel {err:.3e}"
    assert dp <= DPSNR, f"{name}: dPSNR {dp:.4f} dB"
    # per-iteration max|du| trace tracks the oracle's
    gm = np.array([r.maxAbsChange for r in res.trace.records])
    assert len(gm) == it
    np.testing.assert_allclose(gm, mc, rtol=2e-2, atol=1e-6)
    return err, dp


def test_cfg0_full():
    run_config("cfg0")


def test_cfg1_full():
    run_config("cfg1")


def test_cfg2_reduced():
    run_config("cfg2", 512, 512)


def test_cfg3_unthinned_reduced():
    run_config("cfg3", 192, 160)


def test_cfg4_reduced():
    run_config("cfg4", 1024, 768)


def test_cfg4b_one_image_reduced():
    run_config("cfg4b", 2048, 96)


def test_identity_fixed_point_bit_identical():
    rng = np.random.default_rng(51)
    f = rng.integers(0, 256, size=(10, 14)).astype(np.float32)
    r = rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(iterations=5))
    assert np.array_equal(r.image, f)
    assert len(r.trace.records) == 5


def test_constant_stays_constant():
    f = np.full((12, 16), 100.0, np.float32)
    for psf in [makeDiscPsf(5), makeBoxPsf(3, 3), makeDiagonalPsf(5), W.gaussian31()]:
        r = rlDeconvolve(f, psf, RlConfig(iterations=20))
        np.testing.assert_allclose(r.image, f, rtol=1e-5)


def test_exact_reblur_fixed_point():
    g = W.scene(48, 48, 42, 4, 2) * 0.9 + 0.1
    for psf in [W.gaussian31(), makeBoxPsf(3, 3), makeDiscPsf(5)]:
        f = convolve(g, psf, K.Naive)
        u = g.astype(np.float32)
        for _ in range(10):
            u = rlStep(u, f, psf, RlConfig(op=K.Naive))
        assert W.max_rel(u, g) < 1e-4


def test_nonnegative():
    rng = np.random.default_rng(52)
    g = rng.integers(0, 256, size=(20, 20)).astype(np.float64)
    f = convolve(g, makeDiscPsf(3))
    r = rlDeconvolve(f, makeDiscPsf(3), RlConfig(iterations=15))
    assert (r.image >= 0).all()


def test_selective_threshold_zero_equals_standard():
    # proj/tests/test_rl.cpp:81-101, on the device: same kernels, same bits
    _, f = W.make_input(W.CONFIGS["cfg3"], 96, 80)
    psf = W.gaussian31()
    std = rlDeconvolve(f, psf, RlConfig(iterations=12, op=K.Naive)).image
    sel = rlDeconvolveSelective(f, psf, RlConfig(iterations=12, op=K.Naive), 0.0)
    assert np.array_equal(std, sel.image)
    assert sel.trace.omittedPercent() == 0.0


def test_selective_infinite_threshold_schedule():
    # proj/tests/test_rl.cpp:103-127
    _, f = W.make_input(W.CONFIGS["cfg3"], 64, 48)
    psf = makeDiscPsf(3)
    r = rlDeconvolveSelective(f, psf, RlConfig(iterations=25, op=K.Naive), float("inf"), 10)
    u = f.copy()
    for _ in range(3):
        u = rlStep(u, f, psf, RlConfig(op=K.Naive))
    np.testing.assert_allclose(r.image, u, rtol=1e-6)
    assert abs(r.trace.omittedPercent() - 88.0) < 1e-9
    assert r.trace.records[0].inactiveFraction == 0.0
    assert r.trace.records[1].inactiveFraction == 1.0
    assert r.trace.records[10].inactiveFraction == 0.0


@pytest.mark.parametrize("psf_name,op", [("gauss31", K.Naive), ("diag9", K.List)])
def test_selective_mask_replay_parity(psf_name, op):
    """Config-3 semantics at reduced size: thinning from iteration 20 on, the
    oracle's per-iteration active masks replayed on the device; compaction
    lists / runs bit-exact, the image within tolerance."""
    _, f = W.make_input(W.CONFIGS["cfg3"], 160, 128)
    psf = W.gaussian31() if psf_name == "gauss31" else makeDiagonalPsf(9)
    it, thr = 60, 2e-4
    ref, inact, mc, masks = O.rl_selective(f.astype(np.float64), psf, it, thr, 10, 20, int(op), record_masks=True)
    assert 0.05 < inact[20:].mean() < 0.95  # the threshold actually thins
    res = rlDeconvolveSelective(f, psf, RlConfig(iterations=it, op=op), thr, 10, thin_start=20,
                                mask_replay=masks, record_masks=True)
    assert np.array_equal(res.masks, masks)
    np.testing.assert_allclose([r.inactiveFraction for r in res.trace.records], inact, atol=0)
    assert W.max_rel(res.image, ref) <= MAX_REL
    for k in (20, 35, 59):
        idx, runs = maskRuns(masks[k])
        assert np.array_equal(idx, O.active_list(masks[k]))
        assert np.array_equal(runs, O.mask_runs(masks[k]))


def test_selective_free_running_close_to_replay():
    _, f = W.make_input(W.CONFIGS["cfg3"], 128, 128)
    psf = W.gaussian31()
    it, thr = 50, 2e-4
    ref, inact, _, masks = O.rl_selective(f.astype(np.float64), psf, it, thr, 10, 20, O.NAIVE, record_masks=True)
    res = rlDeconvolveSelective(f, psf, RlConfig(iterations=it, op=K.Naive), thr, 10, thin_start=20,
                                record_masks=True)
    inter = np.logical_and(res.masks[20:], masks[20:]).sum()
    union = np.logical_or(res.masks[20:], masks[20:]).sum()
    assert inter / max(union, 1) > 0.97  # mask Jaccard of the free-running device
    # fp32 flips decisions near the threshold, so the free-running image is
    # compared loosely (the replay test above is the parity gate)
    assert W.max_rel(res.image, ref) <= 1e-2
    assert W.psnr(res.image, ref) > 70


def test_validation_messages():
    f = np.ones((4, 4), np.float32)
    bad = f.copy()
    bad[1, 1] = -3
    with pytest.raises(ValueError, match="nonnegative"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    bad[1, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        rlDeconvolve(bad, makeBoxPsf(1, 1))
    with pytest.raises(ValueError, match="epsilonDiv"):
        rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(epsilonDiv=0.0))
    with pytest.raises(ValueError, match="threshold"):
        rlDeconvolveSelective(f, makeBoxPsf(1, 1), RlConfig(), -0.1)
    with pytest.raises(ValueError, match="period"):
        rlDeconvolveSelective(f, makeBoxPsf(1, 1), RlConfig(), 0.1, 0)
    with pytest.raises(ValueError, match="masked evaluation"):
        rlDeconvolveSelective(f, makeDiscPsf(3), RlConfig(op=K.GenericBox), 0.1)


def test_device_solver_graph_replay_matches_host_api():
    import torch
    from paper_1304_7211_b200 import RlSolver
    from paper_1304_7211_b200 import sharded as S
    cfg = W.CONFIGS["cfg4"]
    _, f = W.make_input(cfg, 768, 320)
    psf = W.make_psf(cfg.psf)
    rc = RlConfig(iterations=25, op=K.Box2dSliding)
    host = rlDeconvolve(f, psf, rc).image
    dev = torch.device("cuda", 0)
    fd = torch.from_numpy(f).to(dev)
    ud = torch.empty_like(fd)
    solver = RlSolver(psf, rc, 768, 320)
    solver.use_stream(torch.cuda.current_stream(dev).cuda_stream)
    for _ in range(3):  # eager, capture, replay
        solver.run(fd, ud)
        torch.cuda.synchronize()
        assert np.array_equal(ud.cpu().numpy(), host)
    # the row-strip driver with a single rank (no exchange) runs the two-pass
    # engine (the solver's run() fuses each iteration into one pass)
    s = S.strip_of(320, 1, 0, 0)
    u2 = S.rl_strips(fd.clone(), s, 25, S.GpuPasses(solver))
    torch.cuda.synchronize()
    assert W.max_rel(u2.cpu().numpy(), host) <= 1e-5
    mc = [m for m, _ in solver.trace(25)]
    assert all(m > 0 for m in mc)


@pytest.mark.parametrize("name,w,h", [("cfg1", 640, 480), ("cfg2", 512, 512)])
def test_spans_marching_kernel_rl(name, w, h):
    """RL on the marching span kernel (the default for images > 4.5 Mpx),
    forced on a reduced config; the tile kernel runs these sizes by default."""
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"spans", 2)
    try:
        run_config(name, w, h, iterations=60)
    finally:
        lib().fdg_set_option(b"spans", prev)


@pytest.mark.parametrize("w,h", [(1, 1), (5, 3), (7, 9), (130, 67), (1027, 515)])
def test_validation_first_bad_pixel_order(w, h):
    """rl.hpp:78-83: the first offending pixel in row-major order decides the
    message (non-finite before negative at the same pixel); the device scan
    runs float4 chunks with a scalar tail, so probe heads, tails and both
    orders."""
    rng = np.random.default_rng(w * 1000 + h)
    for _ in range(6):
        f = np.ones((h, w), np.float32)
        i_neg, i_nan = rng.integers(0, w * h, 2)
        f.flat[i_neg] = -1.0
        f.flat[i_nan] = np.inf if rng.random() < 0.5 else np.nan
        msg = "non-finite" if i_nan <= i_neg else "nonnegative"
        with pytest.raises(ValueError, match=msg):
            rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(iterations=1))
    f = np.ones((h, w), np.float32)
    f.flat[w * h - 1] = -0.5  # the very last pixel (tail chunk)
    with pytest.raises(ValueError, match="nonnegative"):
        rlDeconvolve(f, makeBoxPsf(1, 1), RlConfig(iterations=1))


def test_concurrent_calls_from_threads():
    """The reference API is reentrant (independent calls may run concurrently,
    SPEC.md:314): each thread gets its own default context (stream, scratch,
    cached solver), so concurrent calls give the sequential results."""
    import threading
    from paper_1304_7211_b200.psf import makeLinePsf
    rng = np.random.default_rng(21)
    jobs = [(rng.random((96 + 8 * i, 120 + 4 * i)).astype(np.float32) + 0.05, psf, op)
            for i, (psf, op) in enumerate([(W.disc_r10(), K.GenericBox), (makeLinePsf(15), K.Box1dSliding),
                                           (makeBoxPsf(15, 15), K.Box2dSliding), (W.oblique_line(), K.GenericBox),
                                           (W.gaussian31(seed=3, size=9), K.Naive), (makeDiscPsf(3), K.GenericBox)])]
    seq = [rlDeconvolve(f, psf, RlConfig(iterations=15, op=op)).image for f, psf, op in jobs]
    out = [None] * len(jobs)
    errs = []

    def work(i):
        try:
            for _ in range(3):
                f, psf, op = jobs[i]
                out[i] = rlDeconvolve(f, psf, RlConfig(iterations=15, op=op)).image
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a, b in zip(out, seq):
        np.testing.assert_array_equal(a, b)


def test_batch_api_matches_per_image_calls():
    """fdg_rl_deconvolve_batch (chunked, copies overlapping the iterations
    with page-locked buffers; pageable ones one chunk at a time) == one
    rlDeconvolve per image, bit for bit (same engine, same arithmetic)."""
    torch = pytest.importorskip("torch")
    from paper_1304_7211_b200 import rlDeconvolveBatch
    cfg = W.CONFIGS["cfg4b"]
    psf = W.make_psf(cfg.psf)
    imgs = np.stack([W.make_input(cfg, 512, 200, image=i)[1] for i in range(7)])
    rc = RlConfig(iterations=12, op=K.Box1dSliding)
    ref = np.stack([rlDeconvolve(x, psf, rc).image for x in imgs])
    res = rlDeconvolveBatch(imgs, psf, rc)  # pageable
    assert np.array_equal(res.image, ref)
    fp = torch.from_numpy(imgs).pin_memory().numpy()
    up = torch.empty(imgs.shape, dtype=torch.float32).pin_memory().numpy()
    res2 = rlDeconvolveBatch(fp, psf, rc, out=up)
    assert np.array_equal(up, ref) and res2.image is up
    mc = np.max([[r.maxAbsChange for r in rlDeconvolve(x, psf, rc).trace.records] for x in imgs], axis=0)
    np.testing.assert_allclose([r.maxAbsChange for r in res2.trace.records], mc, rtol=1e-6)
    bad = imgs.copy()
    bad[5, 3, 4] = -1.0
    with pytest.raises(Exception, match="nonnegative"):
        rlDeconvolveBatch(bad.astype(np.float32), psf, rc)
