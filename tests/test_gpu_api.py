"""API contract of the GPU path beyond numerics: reentrancy (plans shared
across threads, plans outliving their creating thread, concurrent calls on
images large enough for the pinned staging path), the NaN-in-iterate
failure of rl.hpp:96-99/173, per-iteration trace seconds (rl.hpp:154,172),
device / stream hygiene of the contexts and the device solver."""
import threading

import numpy as np
import pytest

from paper_1304_7211_b200 import OperatorKind as K, RlConfig, RlSolver, rlDeconvolve, workloads as W
from paper_1304_7211_b200 import _lib
from paper_1304_7211_b200.convolve import ConvPlan, convolve
from paper_1304_7211_b200.psf import makeBoxPsf, makeDiscPsf, makeLinePsf

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    errs = []

    def wrap(fn):
        try:
            fn()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=wrap, args=(fn,)) for fn in fns]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs


def test_one_plan_shared_by_threads():
    """ConvPlan is immutable (convolve.hpp:650-753): applications from
    several threads run on each thread's own context (scratch, stream)."""
    rng = np.random.default_rng(5)
    for psf in (makeDiscPsf(9), W.gaussian31(seed=2, size=11), makeBoxPsf(7, 5)):
        plan = ConvPlan(psf)
        imgs = [rng.random((300 + 40 * i, 260 + 24 * i)).astype(np.float32) for i in range(6)]
        seq = [plan.apply(a) for a in imgs]
        out = [None] * len(imgs)

        def job(i):
            def run():
                for _ in range(4):
                    out[i] = plan.apply(imgs[i])
            return run

        _run_threads([job(i) for i in range(len(imgs))])
        for a, b in zip(out, seq):
            np.testing.assert_array_equal(a, b)


def test_plan_outlives_its_creating_thread():
    box = {}

    def make():
        p = ConvPlan(makeDiscPsf(7))
        p.engine()  # device representation built on this thread's context
        box["p"] = p

    t = threading.Thread(target=make)
    t.start()
    t.join()
    import gc
    gc.collect()
    img = np.random.default_rng(6).random((120, 90)).astype(np.float32)
    np.testing.assert_array_equal(box["p"].apply(img), ConvPlan(makeDiscPsf(7)).apply(img))


def test_concurrent_large_calls_staging():
    """Pageable host images >= 4 MiB go through the pinned staging chunks:
    concurrent calls (per-thread contexts) must not share them."""
    rng = np.random.default_rng(7)
    jobs = [(rng.random((1100 + 16 * i, 1024)).astype(np.float32) + 0.05, psf, op) for i, (psf, op) in
            enumerate([(makeLinePsf(15), K.Box1dSliding), (makeBoxPsf(15, 15), K.Box2dSliding),
                       (W.disc_r10(), K.GenericBox), (makeBoxPsf(5, 5), K.Box2dSliding)])]
    assert all(f.nbytes >= 4 << 20 for f, _, _ in jobs)
    seq = [rlDeconvolve(f, psf, RlConfig(iterations=6, op=op)).image for f, psf, op in jobs]
    out = [None] * len(jobs)

    def job(i):
        def run():
            f, psf, op = jobs[i]
            for _ in range(3):
                out[i] = rlDeconvolve(f, psf, RlConfig(iterations=6, op=op)).image
        return run

    _run_threads([job(i) for i in range(len(jobs))])
    for a, b in zip(out, seq):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("psf,op", [(makeBoxPsf(15, 15), K.Box2dSliding), (makeLinePsf(15), K.Box1dSliding),
                                    (W.disc_r10(), K.GenericBox), (makeBoxPsf(5, 3), K.Box2dSliding)])
def test_nan_in_iterate_reported(psf, op):
    """rl.hpp:96-99,173: a NaN in the iterate stops the run with
    "rlDeconvolve: NaN in iterate at iteration k".  Pixels near FLT_MAX
    overflow the fp32 window sums (inf), the next quotient divides by
    max(0, eps) and inf * 0 appears: every engine must flag it."""
    f = np.ones((96, 128), np.float32)
    f[30:60, 40:90] = 3.0e38
    with pytest.raises(_lib.FdgNaNError, match=r"rlDeconvolve: NaN in iterate at iteration \d+"):
        rlDeconvolve(f, psf, RlConfig(iterations=30, op=op))


def test_trace_seconds_are_per_iteration():
    """rl.hpp:154,172: the trace carries each iteration's own time, also when
    the loop is one replayed CUDA graph (device %globaltimer stamps)."""
    cfg = W.CONFIGS["cfg4"]
    _, f = W.make_input(cfg, 1024, 1024)
    for psf, op in ((W.make_psf("box15x15"), K.Box2dSliding), (makeLinePsf(15), K.Box1dSliding),
                    (W.disc_r10(), K.GenericBox)):
        for _ in range(2):  # first call captures, second replays
            r = rlDeconvolve(f, psf, RlConfig(iterations=20, op=op))
        sec = np.array([x.seconds for x in r.trace.records])
        assert (sec > 0).all(), (op, sec)
        assert r.trace.totalSeconds() == pytest.approx(sec.sum())
        # a steady loop: no iteration is an outlier of the whole-run average
        assert sec.max() < 20 * np.median(sec), (op, sec)


def test_entry_points_restore_the_current_device():
    import torch
    torch.cuda.set_device(0)
    rlDeconvolve(np.ones((32, 32), np.float32), makeDiscPsf(3), RlConfig(iterations=2))
    assert torch.cuda.current_device() == 0
    assert _lib.current_device() == 0


def test_solver_follows_torchs_current_stream():
    """RlSolver issues on torch's current stream at call time, so a torch op
    queued before it on a side stream is ordered with it."""
    import torch
    dev = torch.device("cuda", 0)
    cfg = W.CONFIGS["cfg4"]
    _, f = W.make_input(cfg, 512, 384)
    psf = W.make_psf("box15x15")
    rc = RlConfig(iterations=8, op=K.Box2dSliding)
    want = rlDeconvolve(f, psf, rc).image
    solver = RlSolver(psf, rc, 512, 384)
    side = torch.cuda.Stream(dev)
    with torch.cuda.stream(side):
        fd = torch.from_numpy(f).to(dev, non_blocking=False)
        torch.cuda._sleep(2_000_000)  # a long kernel before the input is final on this stream
        fd.mul_(1.0)
        ud = torch.empty_like(fd)
        solver.run(fd, ud)
    side.synchronize()
    np.testing.assert_array_equal(ud.cpu().numpy(), want)
