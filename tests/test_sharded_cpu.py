"""Row-strip sharding host logic on CPU: world_size 2 over gloo, the fused
passes evaluated by the oracle on each rank's strip + halo.  The gathered
result must equal the single-image oracle run (the halo exchange and the
clamp ranges are exactly right iff this holds; SURVEY 8c strip-parallel
oracle).  The GPU executor (GpuPasses) runs the same driver on the box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as O
from paper_1304_7211_b200 import sharded as S
from paper_1304_7211_b200.psf import adjoint, makeBoxPsf, makeDiscPsf, makeLinePsf
from paper_1304_7211_b200 import workloads as W


class OraclePasses:
    def __init__(self, psf, op, eps=1e-8):
        self.psf, self.adj, self.op, self.eps = psf, adjoint(psf), op, eps

    def __call__(self, which, src, aux, out, s, k, rows=None):
        """Output rows [y0, y1) of the core; reads only src rows within T of them."""
        T, w = s.halo, self.width
        y0, y1 = rows if rows is not None else (0, s.core)
        rlo, rhi = max(s.ylo, y0 - T), min(s.yhi, y1 - 1 + T)
        img = src[T + rlo:T + rhi + 1, :w].numpy()
        conv = O.convolve(img, self.psf if which == 1 else self.adj, self.op)
        v = conv[y0 - rlo:y1 - rlo]
        a = aux[T + y0:T + y1, :w].numpy()
        if which == 1:
            res = a / np.where(v < self.eps, self.eps, v)
        else:
            res = np.maximum(v * a, 0.0)
        out[T + y0:T + y1, :w] = torch.from_numpy(res)


class OracleFused:
    """One whole RL iteration on a strip with a 2T-row u halo (the fused
    engine's contract): q on rows [-T, core + T) clamped to the readable
    range, then the adjoint over the core."""

    def __init__(self, psf, op, eps=1e-8):
        self.psf, self.adj, self.op, self.eps = psf, adjoint(psf), op, eps

    def __call__(self, f, u_in, u_out, s, k, rows=None):
        """Output rows [y0, y1) of the core; reads only u rows within 2T of
        them (so the interior pass never touches halo rows in flight)."""
        T2, w = s.halo, self.width
        T = T2 // 2
        y0, y1 = rows if rows is not None else (0, s.core)
        rlo, rhi = max(s.ylo, y0 - T2), min(s.yhi, y1 - 1 + T2)   # u rows read
        img = u_in[T2 + rlo:T2 + rhi + 1, :w].numpy()
        v = O.convolve(img, self.psf, self.op)   # replicate-clamped at rlo / rhi
        qlo, qhi = max(s.ylo, y0 - T), min(s.yhi, y1 - 1 + T)     # q rows needed
        vq = v[qlo - rlo:qhi - rlo + 1]
        fq = f[T2 + qlo:T2 + qhi + 1, :w].numpy()
        qb = fq / np.where(vq < self.eps, self.eps, vq)
        c = O.convolve(qb, self.adj, self.op)[y0 - qlo:y1 - qlo]
        uc = u_in[T2 + y0:T2 + y1, :w].numpy()
        u_out[T2 + y0:T2 + y1, :w] = torch.from_numpy(np.maximum(c * uc, 0.0))


def _worker(rank, world, port, case, H, W_, it, q, fused=False, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        psf, op = CASES[case]()
        rng = np.random.default_rng(9)
        f = rng.random((H, W_)) + 0.05
        s = S.strip_of(H, world, rank, S.fused_halo(psf) if fused else S.psf_halo(psf))
        fl = S.load_strip(f, s, W_ + 3, dtype=torch.float64)
        ex = OracleFused(psf, op) if fused else OraclePasses(psf, op)
        ex.width = W_
        u = S.rl_strips_fused(fl, s, it, ex, overlap=overlap) if fused else S.rl_strips(fl, s, it, ex, overlap=overlap)
        full = S.gather_strips(u, s, W_)
        if rank == 0:
            ref, _, _ = O.rl_deconvolve(f, psf, it, op)
            q.put(float(np.max(np.abs(full.numpy() - ref) / ref)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


CASES = {
    "disc5-generic": lambda: (makeDiscPsf(5), O.GENERIC_BOX),
    "box3x5-box2d": lambda: (makeBoxPsf(3, 5), O.BOX2D_SLIDING),
    "gauss-naive": lambda: (W.gaussian31(seed=5, size=7), O.NAIVE),
    "line9-box1d": lambda: (makeLinePsf(9), O.BOX1D_SLIDING),
}


@pytest.mark.parametrize("name,overlap", [(n, True) for n in sorted(CASES)] + [("disc5-generic", False)])
def test_two_rank_strips_equal_single_image(name, overlap):
    """Two-pass strip driver (u and q halo exchanges), with and without the
    exchanges overlapped by the interior rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, 37, 23, 6, q, False, overlap)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err < 1e-12, err


@pytest.mark.parametrize("world,overlap", [(2, True), (3, True), (2, False)])
def test_fused_strips_equal_single_image(world, overlap):
    """The fused strip driver (2T-row u halo, one exchange per iteration,
    q recomputed next to the core) gives the single-image result -- also
    with the exchange overlapped by the interior rows (boundary bands after
    it lands)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "box3x5-box2d", 61, 23, 6, q, True, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err < 1e-12, err


def test_strip_geometry():
    s0, s1, s2 = (S.strip_of(100, 3, r, 7) for r in range(3))
    assert (s0.r0, s0.core, s0.ylo, s0.yhi) == (0, 33, 0, 39)
    assert (s1.r0, s1.core, s1.ylo, s1.yhi) == (33, 33, -7, 39)
    assert (s2.r0, s2.core, s2.ylo, s2.yhi) == (66, 34, -7, 33)
    assert list(S.batch_share(64, 8, 3)) == list(range(24, 32))
    with pytest.raises(ValueError):
        S.strip_of(10, 4, 0, 7)


# ---- the native sharded runner's host plumbing (libfdgpu fdg_shard_*)
def _id_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cid = S.comm_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, cid)
        if rank == 0:
            q.put((len(cid), all(i == ids[0] for i in ids)))
    finally:
        dist.destroy_process_group()


def test_comm_unique_id_reaches_every_rank():
    """Rank 0's NCCL unique id (fdg_comm_unique_id) is what every rank
    passes to fdg_shard_create (bench.py --gpus N)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    n, same = q.get(timeout=5)
    assert n == 128 and same


def test_shard_create_validation_before_device():
    """Argument errors surface as the reference's exception class even without
    a GPU; the compute entry point itself then refuses (no CPU fallback)."""
    import ctypes as C

    from paper_1304_7211_b200._lib import Desc, FdgError, FdgInvalidArgument, check, lib
    from paper_1304_7211_b200.rl import RlConfig
    h = C.c_void_p()
    cfg = RlConfig(iterations=2).c()
    psf = makeBoxPsf(15, 15)
    with pytest.raises(FdgInvalidArgument, match="communicator"):
        check(lib().fdg_shard_create(None, Desc(psf).ref, C.byref(cfg), 64, 64, 0, 2, None, C.byref(h)))
    with pytest.raises(FdgError):
        check(lib().fdg_shard_create(None, Desc(psf).ref, C.byref(cfg), 64, 64, 0, 1, None, C.byref(h)))
