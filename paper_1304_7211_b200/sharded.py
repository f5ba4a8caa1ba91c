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
