"""Row-strip sharded RL inside libfdgpu (fdg_shard_*) on one GPU.

A ShardGroup runs `world` strips of one image in one process with the
production schedule, row ranges and kernels (interior launch, both boundary
bands in one launch, halo rows from the neighbours), the NCCL send/recv
replaced by device copies between the strips' planes.  The gathered result
must equal the single-image GPU run (the strips read exactly the rows the
whole-image launch reads) and the CPU oracle (rl.hpp:153-177) within the
north-star bound.  ShardedRl with world 1 exercises the per-rank entry
point without a communicator.  The NCCL exchange itself needs >= 2 GPUs
(the driver's scaling run); its host logic is mirrored by the gloo tests
of tests/test_sharded_cpu.py.
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_1304_7211_b200 import OperatorKind as K, RlConfig, rlDeconvolve, workloads as W
from paper_1304_7211_b200._lib import FdgInvalidArgument
from paper_1304_7211_b200.psf import makeBoxPsf, makeDiagonalPsf, makeLinePsf
from paper_1304_7211_b200.sharded import ShardedRl, ShardGroup

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _input(w, h, seed, psf, op):
    g = W.scene(w, h, seed, max(2, w * h // 16384), max(1, w * h // 32768)) * 0.9 + 0.05
    f = np.maximum(O.convolve(g, psf, int(op)), 1e-6).astype(np.float32)
    return g, f


CASES = [
    # name, psf, op, engine, width, height, iterations
    ("box15-fused", makeBoxPsf(15, 15), K.Box2dSliding, "fused", 640, 700, 12),
    ("box15-fused-narrow", makeBoxPsf(15, 15), K.Box2dSliding, "fused", 516, 301, 7),
    ("box5x3-rect", makeBoxPsf(5, 3), K.Box2dSliding, "box", 300, 257, 9),
    ("disc10-spans", W.disc_r10(), K.GenericBox, "spans", 333, 410, 8),
    ("gauss31-dense", W.gaussian31(), K.Naive, "dense", 260, 300, 5),
    ("diag9-taps", makeDiagonalPsf(9), K.List, "taps", 250, 199, 8),
    ("line31-rowres", makeLinePsf(31), K.Box1dSliding, "rowres", 1000, 120, 10),
]


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_group_equals_single_image_and_oracle(case, world):
    name, psf, op, engine, w, h, it = case
    g, f = _input(w, h, 17 + world, psf, op)
    cfg = RlConfig(iterations=it, op=op)
    grp = ShardGroup(psf, cfg, w, h, world)
    assert grp.infos[0]["engine"] == engine
    assert sum(i["core"] for i in grp.infos) == h
    u = np.empty_like(f)
    tr = grp.run(f, u, trace=True)
    single = rlDeconvolve(f, psf, cfg)
    scale = float(np.abs(single.image).max())
    assert float(np.abs(u - single.image).max()) <= 2e-6 * scale, name
    ref, mc, _ = O.rl_deconvolve(f.astype(np.float64), psf, it, int(op))
    assert W.max_rel(u, ref) <= 1e-4
    np.testing.assert_allclose([r.maxAbsChange for r in tr], mc, rtol=2e-2, atol=1e-6)


def test_group_device_buffers_and_exchange_geometry():
    psf = makeBoxPsf(15, 15)
    w, h, world = 1024, 2048, 8
    _, f = _input(w, h, 3, psf, K.Box2dSliding)
    cfg = RlConfig(iterations=6, op=K.Box2dSliding)
    grp = ShardGroup(psf, cfg, w, h, world)
    for r, info in enumerate(grp.infos):
        assert info["r0"] == r * h // world and info["halo"] == 14
        assert info["exchanges_per_iteration"] == 1
        nb = (r > 0) + (r < world - 1)
        assert info["halo_bytes_per_iteration"] == nb * 14 * (info["halo_bytes_per_iteration"] // max(nb * 14, 1))
    df = torch.from_numpy(f).cuda()
    du = torch.empty_like(df)
    grp.run(df, du)
    torch.cuda.synchronize()
    single = rlDeconvolve(f, psf, cfg).image
    np.testing.assert_allclose(du.cpu().numpy(), single, rtol=2e-6, atol=1e-7)
    t = grp.timing(3)
    assert t["interior_ms"] > 0 and t["bands_ms"] > 0


def test_world1_shard_entry_point_host_and_device():
    psf = makeBoxPsf(15, 15)
    w, h = 700, 333
    _, f = _input(w, h, 5, psf, K.Box2dSliding)
    cfg = RlConfig(iterations=10, op=K.Box2dSliding)
    sh = ShardedRl(psf, cfg, w, h, 0, 1)
    assert sh.info["engine"] == "fused" and sh.info["exchanges_per_iteration"] == 0
    u = np.empty_like(f)
    tr = sh.run(f, u, trace=True)
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"fused", 2)  # the same engine for the 0.23 Mpx single-image run
    try:
        single = rlDeconvolve(f, psf, cfg)
    finally:
        lib().fdg_set_option(b"fused", prev)
    np.testing.assert_allclose(u, single.image, rtol=1e-6, atol=1e-7)
    assert len(tr) == 10 and all(r.seconds > 0 for r in tr)
    df = torch.from_numpy(f).cuda()
    du = torch.empty_like(df)
    sh.run(df, du)
    torch.cuda.synchronize()
    assert np.array_equal(du.cpu().numpy(), u)


def test_shard_validation():
    psf = makeBoxPsf(15, 15)
    cfg = RlConfig(iterations=2, op=K.Box2dSliding)
    with pytest.raises(FdgInvalidArgument, match="thinner than"):
        ShardGroup(psf, cfg, 600, 100, 8)  # 12-row strips < the 14-row halo
    with pytest.raises(FdgInvalidArgument, match="communicator"):
        ShardedRl(psf, cfg, 600, 100, 0, 2, None)


@pytest.mark.parametrize("psf,op", [(makeBoxPsf(15, 15), K.Box2dSliding), (makeBoxPsf(3, 3), K.Box2dSliding)])
def test_nan_in_iterate_reported_by_the_group(psf, op):
    """rl.hpp:96-99,173 over the strips (fused and two-pass engines): pixels
    near FLT_MAX overflow the window sums, the iterate turns NaN."""
    from paper_1304_7211_b200._lib import FdgNaNError
    f = np.ones((192, 256), np.float32)
    f[60:120, 40:90] = 3.0e38
    grp = ShardGroup(psf, RlConfig(iterations=30, op=op), 256, 192, 2)
    with pytest.raises(FdgNaNError, match=r"NaN in iterate at iteration \d+"):
        grp.run(f, np.empty_like(f), trace=True)


def test_world1_with_nccl_communicator():
    """A one-rank NCCL communicator (libnccl.so.2 loaded with dlopen, comm
    init, the trace all-reduce) on the real GPU: the NCCL plumbing of the
    sharded runner executes; the result equals the plain run."""
    from paper_1304_7211_b200.sharded import comm_unique_id
    psf = makeBoxPsf(15, 15)
    w, h = 640, 300
    _, f = _input(w, h, 9, psf, K.Box2dSliding)
    cfg = RlConfig(iterations=8, op=K.Box2dSliding)
    sh = ShardedRl(psf, cfg, w, h, 0, 1, comm_unique_id())
    u = np.empty_like(f)
    tr = sh.run(f, u, trace=True)
    from paper_1304_7211_b200._lib import lib
    prev = lib().fdg_set_option(b"fused", 2)  # the same engine for the 0.23 Mpx single-image run
    try:
        single = rlDeconvolve(f, psf, cfg)
    finally:
        lib().fdg_set_option(b"fused", prev)
    np.testing.assert_allclose(u, single.image, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose([r.maxAbsChange for r in tr], [r.maxAbsChange for r in single.trace.records],
                               rtol=1e-5)
