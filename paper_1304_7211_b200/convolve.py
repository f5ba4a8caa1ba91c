"""Spatial convolution operators on the B200 -- Python face of
/root/reference/proj/include/fastdeconv/convolve.hpp.

Same contract (convolve.hpp:17-21): ``out(x,y) = sum w(dx,dy) * in(x+dx, y+dy)``
with replicate continuation (correlation; the adjoint negates offsets).  The
operator kind is resolved exactly like ``dispatch`` (convolve.hpp:627-643) by
the native plan logic, then served by one of the sm_100a engines ("box",
"taps", "dense", "spans", "cyclic").  Images are 2-D numpy arrays (H, W);
device arithmetic is fp32.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import Context, Desc, check, f32, fptr, lib, u8ptr
from .psf import SparsePsf


class OperatorKind(enum.IntEnum):
    """convolve.hpp:22-32 (same numbering as the C ABI's fdg_op)."""

    Naive = 0
    List = 1
    GenericBox = 2
    Box2dSliding = 3
    Box2dCumulated = 4
    Box1dSliding = 5
    Box1dCumulated = 6
    Fourier = 7
    Auto = 8


_NAMES = {
    OperatorKind.Naive: "naive", OperatorKind.List: "list", OperatorKind.GenericBox: "generic-box",
    OperatorKind.Box2dSliding: "box2d-sliding", OperatorKind.Box2dCumulated: "box2d-cumul",
    OperatorKind.Box1dSliding: "box1d-sliding", OperatorKind.Box1dCumulated: "box1d-cumul",
    OperatorKind.Fourier: "fourier", OperatorKind.Auto: "auto",
}


def operatorName(kind) -> str:
    """convolve.hpp:34-47"""
    return _NAMES.get(OperatorKind(kind), "unknown")


def operatorKindFromName(name: str) -> OperatorKind:
    """convolve.hpp:49-56"""
    for k, n in _NAMES.items():
        if n == name:
            return k
    raise ValueError(f"unknown operator name: {name}")


def supportsMasking(kind) -> bool:
    """convolve.hpp:59-61"""
    return OperatorKind(kind) in (OperatorKind.Naive, OperatorKind.List)


@dataclass
class ConvCounters:
    """convolve.hpp:66-70; filled analytically from the reference cost model."""

    pixels: int = 0
    perPixelOps: int = 0
    setupOps: int = 0

    def _add(self, c):
        self.pixels += int(c[0])
        self.perPixelOps += int(c[1])
        self.setupOps += int(c[2])


def dispatch(psf, preference=OperatorKind.Auto) -> OperatorKind:
    """convolve.hpp:627-643 (host-only; raises ValueError naming the operator)."""
    d = Desc(psf)
    k = C.c_int(-1)
    check(lib().fdg_dispatch(d.ref, int(preference), C.byref(k)))
    return OperatorKind(k.value)


def operatorAcceptsPsf(kind, psf) -> bool:
    """convolve.hpp:607-625"""
    d = Desc(psf)
    a = C.c_int(0)
    check(lib().fdg_operator_accepts(int(kind), d.ref, C.byref(a)))
    return bool(a.value)


def _as_image(img) -> np.ndarray:
    a = np.asarray(img)
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("Image: dimensions must be at least 1x1")
    return a


def _out_dtype(a):
    return a.dtype if a.dtype in (np.float32, np.float64) else np.float64


class ConvPlan:
    """convolve.hpp:650-753: a PSF bound to its resolved operator.  The
    device plan (uploaded taps / weights) is created on first use."""

    def __init__(self, psf, preference=OperatorKind.Auto, ctx: Optional[Context] = None):
        self._psf = psf
        self._kind = dispatch(psf, preference)  # host-only: no device needed
        self._ctx = ctx      # explicit context (else: the calling thread's)
        self._home = None    # context the device representation was built on
        self._h = None
        self._lock = threading.Lock()

    def kind(self) -> OperatorKind:
        return self._kind

    def _plan(self):
        """The immutable device plan (built once, on first use)."""
        if self._h is None:
            with self._lock:
                if self._h is None:
                    ctx = self._ctx or Context.default()
                    h = C.c_void_p()
                    d = Desc(self._psf)
                    check(lib().fdg_plan_create(ctx.h, d.ref, int(self._kind), C.byref(h)))
                    self._home, self._h = ctx, h
        return self._h

    def _caller_ctx(self):
        """Scratch and stream of this call: the explicit context, else the
        calling thread's default context on the plan's device (concurrent
        applications from several threads share nothing but the plan)."""
        plan = self._plan()
        if self._ctx is not None:
            return self._ctx.h, plan
        return Context.default(lib().fdg_plan_device(plan)).h, plan

    def engine(self) -> str:
        return lib().fdg_plan_engine(self._plan()).decode()

    def _count(self, counters, w, h):
        if counters is not None:
            c = np.zeros(3, dtype=np.uint64)
            check(lib().fdg_op_counters(Desc(self._psf).ref, int(self._kind), w, h,
                                        c.ctypes.data_as(C.POINTER(C.c_uint64))))
            counters._add(c)

    def apply(self, img, counters: Optional[ConvCounters] = None) -> np.ndarray:
        """ConvPlan::apply / applyInto (convolve.hpp:680-722)."""
        a = _as_image(img)
        src = f32(a)
        out = np.empty_like(src)
        h, w = src.shape
        ctx, plan = self._caller_ctx()
        check(lib().fdg_conv_apply_ctx(ctx, plan, fptr(src), w, h, fptr(out)))
        self._count(counters, w, h)
        return out.astype(_out_dtype(a), copy=False)

    applyInto = apply

    def applyMasked(self, img, active, fallback, counters: Optional[ConvCounters] = None) -> np.ndarray:
        """ConvPlan::applyMasked (convolve.hpp:724-744): value where active,
        fallback elsewhere; Naive and List only."""
        if not supportsMasking(self._kind):
            raise _lib.FdgInvalidArgument("operator does not support masked evaluation")
        a = _as_image(img)
        fb = np.asarray(fallback)
        act = np.ascontiguousarray(active, dtype=np.uint8)
        if fb.shape != a.shape:
            raise _lib.FdgInvalidArgument("maskedConvolve: fallback dimensions differ from input")
        if act.size != a.size:
            raise _lib.FdgInvalidArgument("maskedConvolve: mask size differs from input")
        src, fb32 = f32(a), f32(fb)
        out = np.empty_like(src)
        h, w = src.shape
        ctx, plan = self._caller_ctx()
        check(lib().fdg_conv_apply_masked_ctx(ctx, plan, fptr(src), w, h, u8ptr(act.reshape(h, w)),
                                              fptr(fb32), fptr(out)))
        if counters is not None:
            c = np.zeros(3, dtype=np.uint64)
            check(lib().fdg_op_counters(Desc(self._psf).ref, int(self._kind), w, h,
                                        c.ctypes.data_as(C.POINTER(C.c_uint64))))
            visited = int(np.count_nonzero(act))
            per_px = int(c[1]) // max(w * h, 1)
            counters.pixels += visited
            counters.perPixelOps += visited * per_px
        return out.astype(_out_dtype(a), copy=False)

    applyMaskedInto = applyMasked

    def apply_device(self, d_in, d_out, width, height, pitch):
        """device-resident apply on raw device pointers (ints), ctx stream."""
        check(lib().fdg_conv_apply_device(self._plan(), C.c_void_p(d_in), C.c_void_p(d_out), width, height,
                                          pitch))

    def __del__(self):
        try:
            if self._h is not None:
                lib().fdg_plan_destroy(self._h)
        except Exception:
            pass


def convolve(img, psf, kind=OperatorKind.Auto, counters: Optional[ConvCounters] = None) -> np.ndarray:
    """convolve.hpp:756-759"""
    return ConvPlan(psf, kind).apply(img, counters)


def maskedConvolve(img, psf, kind, active, fallback, counters: Optional[ConvCounters] = None) -> np.ndarray:
    """convolve.hpp:762-770: Auto resolves to List for a SparsePsf, else Naive."""
    kind = OperatorKind(kind)
    if kind == OperatorKind.Auto:
        kind = OperatorKind.List if isinstance(psf, SparsePsf) else OperatorKind.Naive
    if not supportsMasking(kind):
        raise _lib.FdgInvalidArgument("operator does not support masked evaluation")
    return ConvPlan(psf, kind).applyMasked(img, active, fallback, counters)


# one-shot operators, convolve.hpp:517-601
def naiveConvolve(img, psf, counters=None):
    return convolve(img, psf, OperatorKind.Naive, counters)


def listConvolve(img, psf, counters=None):
    return convolve(img, psf, OperatorKind.List, counters)


def genericBoxConvolve(img, psf, counters=None):
    return convolve(img, psf, OperatorKind.GenericBox, counters)


def fourierConvolve(img, psf):
    return convolve(img, psf, OperatorKind.Fourier)


def box1dSlidingConvolve(img, length, counters=None):
    from .psf import makeLinePsf
    if length < 1:
        raise ValueError("box1dSlidingConvolve: length must be >= 1")
    return convolve(img, makeLinePsf(length), OperatorKind.Box1dSliding, counters)


def box1dCumulatedConvolve(img, length, counters=None):
    from .psf import makeLinePsf
    if length < 1:
        raise ValueError("box1dCumulatedConvolve: length must be >= 1")
    return convolve(img, makeLinePsf(length), OperatorKind.Box1dCumulated, counters)


def box2dSlidingConvolve(img, mx, my, counters=None):
    from .psf import makeBoxPsf
    if mx < 1 or my < 1:
        raise ValueError("box2dSlidingConvolve: sizes must be >= 1")
    return convolve(img, makeBoxPsf(mx, my), OperatorKind.Box2dSliding, counters)


def box2dCumulatedConvolve(img, mx, my, counters=None):
    from .psf import makeBoxPsf
    if mx < 1 or my < 1:
        raise ValueError("box2dCumulatedConvolve: sizes must be >= 1")
    return convolve(img, makeBoxPsf(mx, my), OperatorKind.Box2dCumulated, counters)


def maskedNaiveConvolve(img, psf, active, fallback, counters=None):
    return maskedConvolve(img, psf, OperatorKind.Naive, active, fallback, counters)


def maskedListConvolve(img, psf, active, fallback, counters=None):
    return maskedConvolve(img, psf, OperatorKind.List, active, fallback, counters)


def maskRuns(active, ctx: Optional[Context] = None):
    """Device stream compaction of a mask: (ordered active index list,
    (y, x0, len) runs) in the order of the reference run walk
    (convolve.hpp:450-465)."""
    act = np.ascontiguousarray(active, dtype=np.uint8)
    h, w = act.shape
    ctx = ctx or Context.default()
    na, nr = C.c_int64(0), C.c_int64(0)
    L = lib()
    check(L.fdg_mask_compact(ctx.h, u8ptr(act), w, h, None, 0, C.byref(na), None, 0, C.byref(nr)))
    idx = np.zeros(max(na.value, 1), dtype=np.int64)
    runs = np.zeros((max(nr.value, 1), 3), dtype=np.int32)
    check(L.fdg_mask_compact(ctx.h, u8ptr(act), w, h, idx.ctypes.data_as(C.POINTER(C.c_int64)), na.value,
                             C.byref(na), runs.ctypes.data_as(C.POINTER(C.c_int32)), nr.value, C.byref(nr)))
    return idx[:na.value], runs[:nr.value]
