"""Richardson-Lucy drivers on the B200 -- Python face of
/root/reference/proj/include/fastdeconv/rl.hpp.

``rlDeconvolve`` / ``rlDeconvolveSelective`` / ``rlStep`` keep the reference
signatures and error behaviour; the whole iteration loop runs inside
libfdgpu with u, f and q resident in HBM (two fused passes per iteration,
see paper_1304_7211_b200/csrc/fdgpu.cu).  ``RlSolver`` is the device-resident
form used by bench.py and the row-strip sharding (torch tensors in, no host
copies inside the loop).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import Context, Desc, RlConfigC, RlRecordC, check, f32, fptr, lib, u8ptr
from .convolve import OperatorKind, convolve


@dataclass
class RlConfig:
    """rl.hpp:18-23"""

    iterations: int = 100
    op: OperatorKind = OperatorKind.Auto
    epsilonDiv: float = 1e-8
    clampNonNegative: bool = True

    def c(self) -> RlConfigC:
        return RlConfigC(int(self.iterations), int(self.op), float(self.epsilonDiv), int(bool(self.clampNonNegative)))


@dataclass
class RlIterationRecord:
    """rl.hpp:25-30"""

    iteration: int = 0
    inactiveFraction: float = 0.0
    maxAbsChange: float = 0.0
    seconds: float = 0.0


@dataclass
class RlTrace:
    """rl.hpp:32-50"""

    records: List[RlIterationRecord] = field(default_factory=list)

    def omittedPercent(self) -> float:
        if not self.records:
            return 0.0
        s = 0.0
        for r in self.records:
            s += r.inactiveFraction
        return 100.0 * s / len(self.records)

    def totalSeconds(self) -> float:
        s = 0.0
        for r in self.records:
            s += r.seconds
        return s


@dataclass
class RlResult:
    """rl.hpp:52-55 (+ the recorded masks of a selective run when asked)"""

    image: np.ndarray
    trace: RlTrace
    masks: Optional[np.ndarray] = None


class BoundaryMode(enum.IntEnum):
    """rl.hpp:67"""

    Cyclic = 0
    Replicate = 1


def _image(f) -> np.ndarray:
    a = np.asarray(f)
    if a.ndim != 2:
        raise _lib.FdgInvalidArgument("empty input image")
    return a


def _validate_cfg(a: np.ndarray, cfg: RlConfig, where: str):
    """rl.hpp:71-77: the checks that come before the pixels"""
    if a.size == 0:
        raise _lib.FdgInvalidArgument(f"{where}: empty input image")
    if cfg.iterations < 0:
        raise _lib.FdgInvalidArgument(f"{where}: iterations must be >= 0")
    if not (cfg.epsilonDiv > 0.0):
        raise _lib.FdgInvalidArgument(f"{where}: epsilonDiv must be positive")


def _validate(a: np.ndarray, cfg: RlConfig, where: str):
    """rl.hpp:71-84 in the reference's order (config first, then pixels) on
    the caller's own values; float32 input is validated on the device."""
    _validate_cfg(a, cfg, where)
    _lib.validate_image(a, where)


_REC_DTYPE = np.dtype([("iteration", "<i4"), ("_pad", "<i4"), ("inactive", "<f8"), ("maxc", "<f8"),
                       ("sec", "<f8")])


def _trace(recs, n) -> RlTrace:
    if n <= 0:
        return RlTrace([])
    # one numpy view of the C records (per-field ctypes access costs ~1 us each)
    a = np.frombuffer(recs, dtype=_REC_DTYPE, count=n)
    return RlTrace([RlIterationRecord(int(i), float(f), float(m), float(t))
                    for i, f, m, t in zip(a["iteration"], a["inactive"], a["maxc"], a["sec"])])


def _out(a, u32):
    return u32.astype(a.dtype if a.dtype in (np.float32, np.float64) else np.float64, copy=False)


def rlDeconvolve(f, h, cfg: RlConfig = RlConfig(), ctx: Optional[Context] = None,
                 out: Optional[np.ndarray] = None) -> RlResult:
    """Standard RL from u0 = f (rl.hpp:140-179).  ``out``: optional
    C-contiguous (H, W) array of the image's dtype that receives the result
    (e.g. page-locked memory: the device -> host copy then runs at full DMA
    speed instead of through the pinned staging chunks).  float64 images (the
    reference's pixel type) go to fdg_rl_deconvolve_f64: converted and checked
    (rl.hpp:78-83, on the doubles) chunk by chunk on their way to the device,
    the result converted back the same way."""
    a = _image(f)
    n = max(cfg.iterations, 0)
    recs = (RlRecordC * max(n, 1))()
    c = cfg.c()
    if a.dtype == np.float64 and a.size:
        _validate_cfg(a, cfg, "rlDeconvolve")
        src = np.ascontiguousarray(a)
        hh, w = src.shape
        if out is not None:
            if out.dtype != np.float64 or out.shape != src.shape or not out.flags.c_contiguous:
                raise _lib.FdgInvalidArgument(
                    "rlDeconvolve: out must be a C-contiguous float64 array of the image's shape")
            u = out
        else:
            u = np.empty_like(src)
        check(lib().fdg_rl_deconvolve_f64(Context.handle_or_null(ctx), Desc(h).ref, C.byref(c), _lib.dptr(src), w, hh,
                                          _lib.dptr(u), recs))
        return RlResult(u, _trace(recs, n))
    _validate(a, cfg, "rlDeconvolve")
    src = f32(a)
    hh, w = src.shape if src.size else (0, 0)
    if out is not None:
        if out.dtype != np.float32 or out.shape != src.shape or not out.flags.c_contiguous:
            raise _lib.FdgInvalidArgument("rlDeconvolve: out must be a C-contiguous float32 array of the image's shape")
        u = out
    else:
        u = np.empty_like(src)
    check(lib().fdg_rl_deconvolve(Context.handle_or_null(ctx), Desc(h).ref, C.byref(c), fptr(src), w, hh, fptr(u), recs))
    return RlResult(_out(a, u), _trace(recs, n))


def rlDeconvolveBatch(fs, h, cfg: RlConfig = RlConfig(), ctx: Optional[Context] = None,
                      out: Optional[np.ndarray] = None) -> RlResult:
    """rlDeconvolve (rl.hpp:140-179) over a (batch, H, W) stack of independent
    images in one call (fdg_rl_deconvolve_batch): with page-locked input /
    output the uploads and downloads of neighbouring chunks overlap the
    iterations.  trace: per iteration, max|du| over the batch."""
    a = np.asarray(fs)
    if a.ndim != 3 or a.size == 0:
        raise _lib.FdgInvalidArgument("rlDeconvolve: empty input image")
    _validate(a, cfg, "rlDeconvolve")
    src = f32(a)
    b, hh, w = src.shape
    if out is not None:
        if out.dtype != np.float32 or out.shape != src.shape or not out.flags.c_contiguous:
            raise _lib.FdgInvalidArgument("rlDeconvolve: out must be a C-contiguous float32 array of the batch's shape")
        u = out
    else:
        u = np.empty_like(src)
    n = max(cfg.iterations, 0)
    recs = (RlRecordC * max(n, 1))()
    c = cfg.c()
    check(lib().fdg_rl_deconvolve_batch(Context.handle_or_null(ctx), Desc(h).ref, C.byref(c), fptr(src), w, hh, b,
                                        fptr(u), recs))
    return RlResult(_out(a, u), _trace(recs, n))


def rlDeconvolveSelective(f, h, cfg: RlConfig, threshold: float, period: int = 10, thin_start: int = 0,
                          mask_replay: Optional[np.ndarray] = None, record_masks: bool = False,
                          ctx: Optional[Context] = None) -> RlResult:
    """Selective (thinned) RL, rl.hpp:187-257.  ``thin_start`` holds the
    deactivation off for 0-based iterations k < thin_start (0 = reference);
    ``mask_replay`` (iterations x H x W uint8) replays recorded active masks."""
    a = _image(f)
    _validate(a, cfg, "rlDeconvolveSelective")
    src = f32(a)
    hh, w = src.shape
    u = np.empty_like(src)
    n = max(cfg.iterations, 0)
    recs = (RlRecordC * max(n, 1))()
    rep = None
    if mask_replay is not None:
        rep = np.ascontiguousarray(mask_replay, dtype=np.uint8)
        if rep.shape != (n, hh, w):
            raise _lib.FdgInvalidArgument("mask_replay must be iterations x height x width")
    rec = np.zeros((n, hh, w), dtype=np.uint8) if record_masks else None
    c = cfg.c()
    check(lib().fdg_rl_deconvolve_selective(Context.handle_or_null(ctx), Desc(h).ref, C.byref(c), float(threshold), int(period),
                                            int(thin_start), u8ptr(rep), u8ptr(rec), fptr(src), w, hh,
                                            fptr(u), recs))
    return RlResult(_out(a, u), _trace(recs, n), rec)


def rlStep(u, f, h, cfg: RlConfig = RlConfig(), ctx: Optional[Context] = None) -> np.ndarray:
    """One multiplicative update (rl.hpp:131-137)."""
    ua, fa = _image(u), _image(f)
    if ua.shape != fa.shape:
        raise _lib.FdgInvalidArgument("rlStep: image dimensions differ")
    u32, f32_ = f32(ua), f32(fa)
    out = np.empty_like(u32)
    hh, w = u32.shape
    c = cfg.c()
    mc = C.c_double(0)
    check(lib().fdg_rl_step(Context.handle_or_null(ctx), Desc(h).ref, C.byref(c), fptr(u32), fptr(f32_), w, hh, fptr(out), C.byref(mc)))
    return _out(ua, out)


def blurImage(g, h, mode: BoundaryMode) -> np.ndarray:
    """rl.hpp:261-265: cyclic = the Fourier operator's wrap-around contract,
    replicate = the auto-dispatched spatial operator."""
    if BoundaryMode(mode) == BoundaryMode.Cyclic:
        return convolve(g, h, OperatorKind.Fourier)
    return convolve(g, h, OperatorKind.Auto)


class RlSolver:
    """Device-resident RL for ``batch`` images of ``height`` x ``width``
    (fdg_solver_*).  Buffers are torch CUDA tensors (float32, last dim =
    pitch, pitch % 4 == 0).  Work is issued on torch's current stream of the
    solver's device at the time of each call (so it is ordered with torch
    ops and the NCCL halo exchanges torch.distributed posts there), unless
    use_stream() pinned an explicit stream."""

    def __init__(self, h, cfg: RlConfig, width: int, height: int, batch: int = 1, device: int = 0,
                 ctx: Optional[Context] = None):
        self.ctx = ctx or Context(device)
        self.device = self.ctx.device
        self.cfg = cfg
        self.width, self.height, self.batch = width, height, batch
        self._pinned_stream = None
        self._bound = None
        s = C.c_void_p()
        c = cfg.c()
        check(lib().fdg_solver_create(self.ctx.h, Desc(h).ref, C.byref(c), width, height, batch, C.byref(s)))
        self.h = s

    def use_stream(self, stream_ptr: int):
        """Pin every later call to this cudaStream_t."""
        self._pinned_stream = stream_ptr
        self._bind()

    def _bind(self):
        sp = self._pinned_stream
        if sp is None:
            import torch
            sp = torch.cuda.current_stream(self.device).cuda_stream
        if sp != self._bound:
            self.ctx.set_stream(sp)
            self._bound = sp

    def run(self, f, u, iterations: Optional[int] = None):
        """u <- f, then `iterations` RL iterations in place (device tensors)."""
        self._bind()
        it = self.cfg.iterations if iterations is None else iterations
        pitch = f.shape[-1]
        stride = f.stride(0) if f.dim() == 3 else pitch * self.height
        check(lib().fdg_solver_run(self.h, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), pitch, stride, it))

    def pass_(self, which: int, d_in: int, d_aux: int, d_out: int, pitch: int, image_stride: int, y0: int,
              y1: int, ylo: int, yhi: int, iteration: int):
        """One fused pass on raw device pointers (row-strip sharding)."""
        self._bind()
        check(lib().fdg_solver_pass(self.h, which, C.c_void_p(d_in), C.c_void_p(d_aux), C.c_void_p(d_out), pitch,
                                    image_stride, y0, y1, ylo, yhi, iteration))

    def iterate(self, d_f: int, d_u_in: int, d_u_out: int, pitch: int, image_stride: int, y0: int, y1: int,
                ylo: int, yhi: int, iteration: int):
        """One whole fused RL iteration on raw device pointers (row strips;
        engine() must be "fused")."""
        self._bind()
        check(lib().fdg_solver_iterate(self.h, C.c_void_p(d_f), C.c_void_p(d_u_in), C.c_void_p(d_u_out), pitch,
                                       image_stride, y0, y1, ylo, yhi, iteration))

    def trace(self, n: Optional[int] = None):
        """[(max|du|, nan_flag)] per iteration (synchronises)."""
        self._bind()
        n = n or max(self.cfg.iterations, 1)
        recs = (RlRecordC * n)()
        check(lib().fdg_solver_trace(self.h, recs, n))
        return [(recs[i].max_abs_change, bool(recs[i].inactive_fraction)) for i in range(n)]

    def reset_trace(self):
        self._bind()
        check(lib().fdg_solver_reset_trace(self.h))

    def launches(self) -> int:
        return self.ctx.launch_count()

    def engine(self) -> str:
        """Engine of run(): "fused", "rowres" or the two-pass plan engine."""
        return lib().fdg_solver_engine(self.h).decode()

    def __del__(self):
        try:
            if self.h:
                lib().fdg_solver_destroy(self.h)
        except Exception:
            pass
