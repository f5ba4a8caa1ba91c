"""Multi-GPU Richardson-Lucy: row-strip sharding of one large image with a
per-iteration PSF-radius halo exchange, and by-image sharding of batches
(SURVEY 8e).  One process per GPU, torch.distributed for the plumbing
(NCCL over NVLink on the B200 box; gloo on CPU for the tests).

Row strips.  Rank r owns rows [r*H/P, (r+1)*H/P).  Every plane (f, u, q)
is stored with T halo rows above and below the core (T = the PSF's
vertical radius), the device pointer addressing core row 0.  Per iteration:

    exchange(u)   top/bottom T core rows <-> neighbours' halos
    pass 1        q = f / max(h (x) u, eps)       rows [0, core), reads [ylo, yhi]
    exchange(q)
    pass 2        u = max(h* (x) q * u, 0)

With the fused engine (rl_strips_fused) the halo is 2T rows of u and each
iteration is one exchange + one fused launch that recomputes the q rows
next to the core.

Replicate clamping happens only at the global first/last row (ylo = 0 on
rank 0, yhi = core-1 on the last rank); interior strip edges read the
neighbour's rows, so the sharded result equals the single-GPU one (up to
the box2d vertical running-sum order).  The halo exchange is the path's
only collective; batches need none.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import torch
import torch.distributed as dist


@dataclass
class Strip:
    rank: int
    world: int
    height: int      # global rows
    r0: int          # first global row of the core
    core: int        # core rows
    halo: int        # T

    @property
    def ylo(self) -> int:
        return -self.halo if self.rank > 0 else 0

    @property
    def yhi(self) -> int:
        return self.core - 1 + (self.halo if self.rank < self.world - 1 else 0)

    @property
    def rows(self) -> int:
        return self.core + 2 * self.halo


def strip_of(height: int, world: int, rank: int, halo: int) -> Strip:
    r0 = rank * height // world
    r1 = (rank + 1) * height // world
    if world > 1 and r1 - r0 < halo:
        raise ValueError(f"strip of {r1 - r0} rows is thinner than the {halo}-row halo")
    return Strip(rank, world, height, r0, r1 - r0, halo)


def psf_halo(psf) -> int:
    from .psf import taps_of
    dys = [t[1] for t in taps_of(psf)]
    return max(0, -min(dys), max(dys))


def exchange(buf: torch.Tensor, s: Strip, group=None):
    """Swap T boundary core rows with rank-1 / rank+1 (no wrap-around).
    buf: (rows, pitch) with the core at rows [T, T + core)."""
    for r in exchange_async(buf, s, group):
        r.wait()


def exchange_async(buf: torch.Tensor, s: Strip, group=None) -> list:
    """Post the halo exchange of `exchange` and return the pending works
    (NCCL runs them on its own stream; ``work.wait()`` orders the caller's
    current stream after them)."""
    if s.world == 1 or s.halo == 0:
        return []
    T, c = s.halo, s.core
    ops = []
    if s.rank > 0:
        ops.append(dist.P2POp(dist.isend, buf[T:2 * T], s.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[0:T], s.rank - 1, group))
    if s.rank < s.world - 1:
        ops.append(dist.P2POp(dist.isend, buf[c:c + T], s.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, buf[T + c:T + c + T], s.rank + 1, group))
    return dist.batch_isend_irecv(ops)


class GpuPasses:
    """Fused passes on the device through libfdgpu (RlSolver.pass_)."""

    def __init__(self, solver):
        self.solver = solver

    def __call__(self, which: int, src: torch.Tensor, aux: torch.Tensor, out: torch.Tensor, s: Strip, k: int,
                 rows: Optional[Tuple[int, int]] = None):
        pitch = src.shape[-1]
        off = s.halo * pitch * 4
        y0, y1 = rows if rows is not None else (0, s.core)
        self.solver.pass_(which, src.data_ptr() + off, aux.data_ptr() + off, out.data_ptr() + off, pitch,
                          s.rows * pitch, y0, y1, s.ylo, s.yhi, k)


class GpuFused:
    """Whole fused RL iterations on the device through libfdgpu
    (RlSolver.iterate; the solver's engine must be "fused")."""

    def __init__(self, solver):
        self.solver = solver

    def __call__(self, f: torch.Tensor, u_in: torch.Tensor, u_out: torch.Tensor, s: Strip, k: int,
                 rows: Optional[Tuple[int, int]] = None):
        pitch = f.shape[-1]
        off = s.halo * pitch * 4
        y0, y1 = rows if rows is not None else (0, s.core)
        self.solver.iterate(f.data_ptr() + off, u_in.data_ptr() + off, u_out.data_ptr() + off, pitch,
                            s.rows * pitch, y0, y1, s.ylo, s.yhi, k)


def fused_halo(psf) -> int:
    """Halo rows of the fused strip driver: q rows up to the PSF's vertical
    radius outside the core are recomputed from u, so u needs twice that."""
    return 2 * psf_halo(psf)


def rl_strips_fused(f_local: torch.Tensor, s: Strip, iterations: int, fused: Callable, group=None,
                    u: Optional[torch.Tensor] = None, u2: Optional[torch.Tensor] = None,
                    overlap: bool = True) -> torch.Tensor:
    """RL on this rank's strip with one exchange per iteration: the 2T-row
    u halo (s.halo = fused_halo(psf)), then one fused iteration that
    recomputes the q rows next to the core ("exchange 14 rows of
    u once and recompute v and q on the halo rows").  f's halo rows are
    filled once (the q rows beyond the core read them).  u ping-pongs
    between two buffers; returns the one holding the result.

    overlap: the exchange is posted first and the interior rows
    [halo, core - halo) -- whose windows stay inside the core -- are computed
    while it is in flight; the two boundary bands follow once it has landed
    (the executor takes an output row range)."""
    if u is None:
        u = torch.empty_like(f_local)
    if u2 is None:
        u2 = torch.empty_like(f_local)
    exchange(f_local, s, group)
    u.copy_(f_local)
    H = s.halo
    split = overlap and s.world > 1 and H > 0 and s.core > 2 * H
    for k in range(iterations):
        if split:
            works = exchange_async(u, s, group)
            fused(f_local, u, u2, s, k, rows=(H, s.core - H))
            for w in works:
                w.wait()
            fused(f_local, u, u2, s, k, rows=(0, H))
            fused(f_local, u, u2, s, k, rows=(s.core - H, s.core))
        else:
            exchange(u, s, group)
            fused(f_local, u, u2, s, k)
        u, u2 = u2, u
    return u


def rl_strips(f_local: torch.Tensor, s: Strip, iterations: int, passes: Callable, group=None,
              u: Optional[torch.Tensor] = None, q: Optional[torch.Tensor] = None,
              overlap: bool = True) -> torch.Tensor:
    """RL on this rank's strip.  f_local: (rows, pitch) with halos (f's halo
    rows are never read).  Returns u (same layout).

    overlap: each pass posts its halo exchange (u before pass 1, q before
    pass 2), runs the interior rows [T, core - T) -- whose windows stay
    inside the core -- while it is in flight, then the two T-row boundary
    bands (the executor takes an output row range)."""
    if u is None:
        u = torch.empty_like(f_local)
    if q is None:
        q = torch.empty_like(f_local)
    u.copy_(f_local)
    T = s.halo
    split = overlap and s.world > 1 and T > 0 and s.core > 2 * T

    def run(which, src, aux, out, k):
        if not split:
            exchange(src, s, group)
            passes(which, src, aux, out, s, k)
            return
        works = exchange_async(src, s, group)
        passes(which, src, aux, out, s, k, rows=(T, s.core - T))
        for w in works:
            w.wait()
        passes(which, src, aux, out, s, k, rows=(0, T))
        passes(which, src, aux, out, s, k, rows=(s.core - T, s.core))

    for k in range(iterations):
        run(1, u, f_local, q, k)
        run(2, q, u, u, k)
    return u


def load_strip(f_global, s: Strip, pitch: int, device=None, dtype=torch.float32) -> torch.Tensor:
    """This rank's rows of a (H, W) host array into a (rows, pitch) buffer."""
    import numpy as np
    buf = torch.zeros((s.rows, pitch), dtype=dtype)
    w = f_global.shape[1]
    buf[s.halo:s.halo + s.core, :w] = torch.from_numpy(np.ascontiguousarray(f_global[s.r0:s.r0 + s.core]))
    return buf.to(device) if device is not None else buf


def gather_strips(u: torch.Tensor, s: Strip, width: int, group=None) -> Optional[torch.Tensor]:
    """Concatenate every rank's core rows on rank 0 (tests / validation)."""
    core = u[s.halo:s.halo + s.core, :width].contiguous()
    sizes = [None] * s.world
    dist.all_gather_object(sizes, core.shape[0], group=group)
    mx = max(sizes)
    pad = torch.zeros((mx, width), dtype=u.dtype, device=u.device)
    pad[:core.shape[0]] = core
    out = [torch.zeros_like(pad) for _ in range(s.world)]
    dist.all_gather(out, pad, group=group)
    if s.rank != 0:
        return None
    return torch.cat([o[:n] for o, n in zip(out, sizes)], dim=0)


def batch_share(batch: int, world: int, rank: int) -> range:
    """Images of a batch owned by `rank` (by-image sharding, no collective)."""
    return range(rank * batch // world, (rank + 1) * batch // world)


# ------------------------------------------------------------------------
# Native sharded loop (libfdgpu fdg_shard_*): the schedule above -- halo
# exchange on a communication stream overlapping the strip interior, both
# boundary bands in one launch -- with NCCL send/recv issued from C++
# (include/fdgpu.h, csrc/shard.cuh).  torch.distributed only carries the
# 128-byte NCCL unique id to the ranks.

ENGINES = {0: "fused", 1: "two-pass", 2: "rowres"}


def comm_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id, every rank receives it (without an
    initialised process group: this process's own id, for a one-rank
    communicator)."""
    import ctypes as C

    from ._lib import check, lib
    if not dist.is_available() or not dist.is_initialized():
        buf = (C.c_ubyte * 128)()
        check(lib().fdg_comm_unique_id(buf))
        return bytes(buf)
    obj = [None]
    if dist.get_rank(group) == 0:
        buf = (C.c_ubyte * 128)()
        check(lib().fdg_comm_unique_id(buf))
        obj[0] = bytes(buf)
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def _ptr_pitch(a, width):
    """(pointer, pitch, host) of a torch CUDA tensor or a host numpy array."""
    import numpy as np
    if isinstance(a, np.ndarray):
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            raise TypeError("host images must be C-contiguous float32")
        return a.ctypes.data, a.shape[-1], 1
    if not a.is_cuda or a.dtype != torch.float32 or a.stride(-1) != 1:
        raise TypeError("device images must be float32 CUDA tensors with unit column stride")
    return a.data_ptr(), a.stride(0), 0


class _ShardBase:
    def _info(self, h):
        import ctypes as C

        from ._lib import check, lib
        v = (C.c_longlong * 6)()
        check(lib().fdg_shard_info(h, v))
        return {"r0": v[0], "core": v[1], "halo": v[2], "exchanges_per_iteration": v[3],
                "halo_bytes_per_iteration": v[4], "engine": lib().fdg_shard_engine(h).decode()}

    def _timing(self, h):
        import ctypes as C

        from ._lib import check, lib
        ms = (C.c_double * 3)()
        check(lib().fdg_shard_timing(h, ms))
        return {"interior_ms": ms[0], "bands_ms": ms[1], "exchange_ms": ms[2]}

    @staticmethod
    def _records(trace, n):
        if not trace:
            return None
        from ._lib import RlRecordC
        return (RlRecordC * max(n, 1))()

    @staticmethod
    def _trace(recs, n):
        if recs is None:
            return None
        from .rl import RlIterationRecord
        return [RlIterationRecord(recs[i].iteration, recs[i].inactive_fraction, recs[i].max_abs_change,
                                  recs[i].seconds) for i in range(n)]


class ShardedRl(_ShardBase):
    """This rank's row strip of one image (fdg_shard_create / _run)."""

    def __init__(self, psf, cfg, width: int, height: int, rank: int, world: int, comm_id: Optional[bytes] = None,
                 ctx=None):
        import ctypes as C

        from ._lib import Context, Desc, check, lib
        self.ctx = ctx or Context.default()
        self.cfg = cfg
        self.width, self.height = width, height
        idp = None
        if comm_id is not None:
            idp = (C.c_ubyte * 128).from_buffer_copy(comm_id)
        h = C.c_void_p()
        c = cfg.c()
        check(lib().fdg_shard_create(self.ctx.h, Desc(psf).ref, C.byref(c), width, height, rank, world, idp,
                                     C.byref(h)))
        self.h = h
        self.info = self._info(h)

    def run(self, f, u, iterations: Optional[int] = None, trace: bool = False):
        """f / u: this rank's core rows (host float32 arrays or CUDA
        tensors).  Device buffers without trace: asynchronous on the
        context's stream."""
        from ._lib import check, lib
        it = self.cfg.iterations if iterations is None else iterations
        pf, pitch, host = _ptr_pitch(f, self.width)
        pu, pitch_u, host_u = _ptr_pitch(u, self.width)
        if (pitch, host) != (pitch_u, host_u):
            raise ValueError("f and u need the same pitch and memory kind")
        recs = self._records(trace, it)
        check(lib().fdg_shard_run(self.h, pf, pu, pitch, host, it, recs))
        return self._trace(recs, it)

    def timing(self):
        return self._timing(self.h)

    def __del__(self):
        try:
            from ._lib import lib
            if self.h:
                lib().fdg_shard_destroy(self.h)
        except Exception:
            pass


class ShardGroup(_ShardBase):
    """`world` strips of one image in this process on one device, exchanging
    halos by device copies (fdg_shard_group_*): the sharded schedule and row
    ranges, checkable against the single-image run on one GPU."""

    def __init__(self, psf, cfg, width: int, height: int, world: int, ctx=None):
        import ctypes as C

        from ._lib import Context, Desc, check, lib
        self.ctx = ctx or Context.default()
        self.cfg = cfg
        self.width, self.height, self.world = width, height, world
        arr = (C.c_void_p * world)()
        c = cfg.c()
        check(lib().fdg_shard_group_create(self.ctx.h, Desc(psf).ref, C.byref(c), width, height, world, arr))
        self.arr = arr
        self.infos = [self._info(arr[r]) for r in range(world)]

    def run(self, f, u, iterations: Optional[int] = None, trace: bool = False):
        from ._lib import check, lib
        it = self.cfg.iterations if iterations is None else iterations
        pf, pitch, host = _ptr_pitch(f, self.width)
        pu, pitch_u, host_u = _ptr_pitch(u, self.width)
        if (pitch, host) != (pitch_u, host_u):
            raise ValueError("f and u need the same pitch and memory kind")
        recs = self._records(trace, it)
        check(lib().fdg_shard_group_run(self.arr, self.world, pf, pu, pitch, host, it, recs))
        return self._trace(recs, it)

    def timing(self, rank: int):
        return self._timing(self.arr[rank])

    def __del__(self):
        try:
            from ._lib import lib
            for r in range(self.world):
                if self.arr[r]:
                    lib().fdg_shard_destroy(self.arr[r])
        except Exception:
            pass
