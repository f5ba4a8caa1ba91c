"""ctypes binding of libfdgpu.so (the C ABI declared in include/fdgpu.h).

The library is built in-tree by ``make lib`` / ``__graft_entry__.build()``.
Plan logic (dispatch, counters) works without a GPU; every compute entry
point raises :class:`FdgError` when no CUDA device is present -- there is no
CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import psf as _psf

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libfdgpu.so"

FDG_OK, FDG_EINVAL, FDG_ENAN, FDG_ELOGIC, FDG_ECUDA = range(5)


class FdgError(RuntimeError):
    """Base error of the GPU path (std::runtime_error of the reference)."""

    code = FDG_ECUDA


class FdgInvalidArgument(FdgError, ValueError):
    """std::invalid_argument: validation, dispatch, masked-evaluation refusals."""

    code = FDG_EINVAL


class FdgNaNError(FdgError):
    """std::runtime_error("...: NaN in iterate at iteration k")."""

    code = FDG_ENAN


class FdgLogicError(FdgError):
    code = FDG_ELOGIC


_ERR = {FDG_EINVAL: FdgInvalidArgument, FDG_ENAN: FdgNaNError, FDG_ELOGIC: FdgLogicError}


class PsfDesc(C.Structure):
    _fields_ = [("repr", C.c_int), ("width", C.c_int), ("height", C.c_int), ("anchor_x", C.c_int),
                ("anchor_y", C.c_int), ("weights", C.POINTER(C.c_double)), ("n_rows", C.c_int),
                ("row_dy", C.POINTER(C.c_int)), ("row_xmin", C.POINTER(C.c_int)),
                ("row_xmax", C.POINTER(C.c_int)), ("n_taps", C.c_int), ("tap_dx", C.POINTER(C.c_int)),
                ("tap_dy", C.POINTER(C.c_int)), ("tap_w", C.POINTER(C.c_double))]


class RlConfigC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("op", C.c_int), ("epsilon_div", C.c_double),
                ("clamp_nonnegative", C.c_int)]


class RlRecordC(C.Structure):
    _fields_ = [("iteration", C.c_int), ("inactive_fraction", C.c_double),
                ("max_abs_change", C.c_double), ("seconds", C.c_double)]


_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    # FDG_LIB_PATH: A/B experiments against another in-tree build
    return os.environ.get("FDG_LIB_PATH") or os.path.join(HERE, LIB_NAME)


def lib():
    """The loaded libfdgpu.so (raises FdgError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not os.path.exists(path):
            raise FdgError(f"{path} is not built: run `make lib` (or __graft_entry__.build()); "
                           "the B200 path has no CPU fallback")
        L = C.CDLL(path)
        vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
        u8p, u64p = C.POINTER(C.c_uint8), C.POINTER(C.c_uint64)
        fp = C.POINTER(C.c_float)
        D = C.POINTER(PsfDesc)
        sig = {
            "fdg_abi_version": (C.c_int, []),
            "fdg_last_error": (C.c_char_p, []),
            "fdg_device_available": (C.c_int, []),
            "fdg_get_device": (C.c_int, [ip]),
            "fdg_plan_device": (C.c_int, [vp]),
            "fdg_conv_apply_ctx": (C.c_int, [vp, vp, fp, C.c_int, C.c_int, fp]),
            "fdg_conv_apply_masked_ctx": (C.c_int, [vp, vp, fp, C.c_int, C.c_int, u8p, fp, fp]),
            "fdg_rl_step_planned": (C.c_int, [vp, vp, vp, C.POINTER(RlConfigC), fp, fp, C.c_int, C.c_int, fp, dp]),
            "fdg_set_option": (C.c_int, [C.c_char_p, C.c_int]),
            "fdg_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "fdg_ctx_destroy": (None, [vp]),
            "fdg_ctx_set_stream": (C.c_int, [vp, vp]),
            "fdg_ctx_synchronize": (C.c_int, [vp]),
            "fdg_ctx_launch_count": (C.c_uint64, [vp]),
            "fdg_ctx_last_schedule": (C.c_int, [vp]),
            "fdg_pipeline_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int]),
            "fdg_dispatch": (C.c_int, [D, C.c_int, ip]),
            "fdg_operator_accepts": (C.c_int, [C.c_int, D, ip]),
            "fdg_plan_create": (C.c_int, [vp, D, C.c_int, C.POINTER(vp)]),
            "fdg_plan_destroy": (None, [vp]),
            "fdg_plan_kind": (C.c_int, [vp]),
            "fdg_plan_counters": (C.c_int, [vp, C.c_int, C.c_int, u64p]),
            "fdg_op_counters": (C.c_int, [D, C.c_int, C.c_int, C.c_int, u64p]),
            "fdg_plan_engine": (C.c_char_p, [vp]),
            "fdg_solver_engine": (C.c_char_p, [vp]),
            "fdg_solver_iterate": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_longlong, C.c_int, C.c_int, C.c_int,
                                             C.c_int, C.c_int]),
            "fdg_conv_apply": (C.c_int, [vp, fp, C.c_int, C.c_int, fp]),
            "fdg_conv_apply_masked": (C.c_int, [vp, fp, C.c_int, C.c_int, u8p, fp, fp]),
            "fdg_conv_apply_device": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int]),
            "fdg_rl_deconvolve": (C.c_int, [vp, D, C.POINTER(RlConfigC), fp, C.c_int, C.c_int, fp,
                                            C.POINTER(RlRecordC)]),
            "fdg_rl_deconvolve_f64": (C.c_int, [vp, D, C.POINTER(RlConfigC), C.POINTER(C.c_double), C.c_int, C.c_int,
                                                C.POINTER(C.c_double), C.POINTER(RlRecordC)]),
            "fdg_rl_deconvolve_selective": (C.c_int, [vp, D, C.POINTER(RlConfigC), C.c_double, C.c_int,
                                                      C.c_int, u8p, u8p, fp, C.c_int, C.c_int, fp,
                                                      C.POINTER(RlRecordC)]),
            "fdg_rl_deconvolve_batch": (C.c_int, [vp, D, C.POINTER(RlConfigC), fp, C.c_int, C.c_int, C.c_int, fp,
                                                  C.POINTER(RlRecordC)]),
            "fdg_rl_step": (C.c_int, [vp, D, C.POINTER(RlConfigC), fp, fp, C.c_int, C.c_int, fp, dp]),
            "fdg_solver_create": (C.c_int, [vp, D, C.POINTER(RlConfigC), C.c_int, C.c_int, C.c_int,
                                            C.POINTER(vp)]),
            "fdg_solver_destroy": (None, [vp]),
            "fdg_solver_run": (C.c_int, [vp, vp, vp, C.c_int, C.c_longlong, C.c_int]),
            "fdg_solver_pass": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int, C.c_longlong, C.c_int, C.c_int,
                                          C.c_int, C.c_int, C.c_int]),
            "fdg_solver_trace": (C.c_int, [vp, C.POINTER(RlRecordC), C.c_int]),
            "fdg_solver_reset_trace": (C.c_int, [vp]),
            "fdg_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
            "fdg_shard_create": (C.c_int, [vp, D, C.POINTER(RlConfigC), C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_ubyte), C.POINTER(vp)]),
            "fdg_shard_group_create": (C.c_int, [vp, D, C.POINTER(RlConfigC), C.c_int, C.c_int, C.c_int,
                                                 C.POINTER(vp)]),
            "fdg_shard_destroy": (None, [vp]),
            "fdg_shard_info": (C.c_int, [vp, C.POINTER(C.c_longlong)]),
            "fdg_shard_engine": (C.c_char_p, [vp]),
            "fdg_shard_run": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(RlRecordC)]),
            "fdg_shard_group_run": (C.c_int, [C.POINTER(vp), C.c_int, vp, vp, C.c_int, C.c_int, C.c_int,
                                              C.POINTER(RlRecordC)]),
            "fdg_shard_timing": (C.c_int, [vp, dp]),
            "fdg_mask_compact": (C.c_int, [vp, u8p, C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_int64,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int64,
                                           C.POINTER(C.c_int64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def check(status: int):
    if status != FDG_OK:
        msg = lib().fdg_last_error().decode(errors="replace")
        raise _ERR.get(status, FdgError)(msg)


def device_available() -> bool:
    return bool(lib().fdg_device_available())


class Desc:
    """fdg_psf_desc for a PSF object (keeps its arrays alive)."""

    def __init__(self, psf):
        d = PsfDesc()
        self._keep = []
        if isinstance(psf, _psf.DensePsf):
            w = np.ascontiguousarray(psf.weights, dtype=np.float64)
            self._keep.append(w)
            d.repr = 0
            d.width, d.height, d.anchor_x, d.anchor_y = psf.width, psf.height, psf.anchorX, psf.anchorY
            d.weights = w.ctypes.data_as(C.POINTER(C.c_double))
        elif isinstance(psf, _psf.UniformConvexPsf):
            a = np.array(psf.rows, dtype=np.int32).reshape(-1, 3)
            cols = [np.ascontiguousarray(a[:, i]) for i in range(3)]
            self._keep += cols
            d.repr = 1
            d.n_rows = len(a)
            d.row_dy, d.row_xmin, d.row_xmax = (c.ctypes.data_as(C.POINTER(C.c_int)) for c in cols)
        elif isinstance(psf, _psf.SparsePsf):
            dx = np.array([t[0] for t in psf.taps], dtype=np.int32)
            dy = np.array([t[1] for t in psf.taps], dtype=np.int32)
            w = np.array([t[2] for t in psf.taps], dtype=np.float64)
            self._keep += [dx, dy, w]
            d.repr = 2
            d.n_taps = len(dx)
            d.tap_dx = dx.ctypes.data_as(C.POINTER(C.c_int))
            d.tap_dy = dy.ctypes.data_as(C.POINTER(C.c_int))
            d.tap_w = w.ctypes.data_as(C.POINTER(C.c_double))
        else:
            raise TypeError(f"not a PSF: {type(psf).__name__}")
        d._arrays = self._keep  # byref(d) keeps the arrays alive for temporaries
        self.s = d

    @property
    def ref(self):
        return C.byref(self.s)


class Context:
    """fdg_ctx: a device + stream + scratch.  One default context per device
    and thread: calls from different threads never share buffers or streams
    (the reference API is reentrant)."""

    _tls = threading.local()

    def __init__(self, device: int = 0):
        L = lib()
        h = C.c_void_p()
        check(L.fdg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def handle_or_null(cls, ctx=None):
        """ctx handle, the default context's, or NULL when no device exists
        (argument validation still runs in the library; compute then fails
        with FdgError)."""
        if ctx is not None:
            return ctx.h
        if not lib().fdg_device_available():
            return None
        return cls.default().h

    @classmethod
    def default(cls, device: int = None) -> "Context":
        """The calling thread's context on `device` (default: the thread's
        current CUDA device)."""
        if device is None:
            device = current_device()
        per_thread = getattr(cls._tls, "ctx", None)
        if per_thread is None:
            per_thread = cls._tls.ctx = {}
        ctx = per_thread.get(device)
        if ctx is None:
            ctx = per_thread[device] = cls(device)
        return ctx

    def set_stream(self, stream_ptr: int):
        check(lib().fdg_ctx_set_stream(self.h, C.c_void_p(stream_ptr)))

    def synchronize(self):
        check(lib().fdg_ctx_synchronize(self.h))

    def launch_count(self) -> int:
        return int(lib().fdg_ctx_launch_count(self.h))

    def last_schedule(self) -> int:
        """0: the last rlDeconvolve uploaded, iterated, downloaded; n >= 2: it
        ran as a time-skewed pipeline over n row strips."""
        return int(lib().fdg_ctx_last_schedule(self.h))

    def __del__(self):
        try:
            if self.h:
                lib().fdg_ctx_destroy(self.h)
        except Exception:
            pass


def current_device() -> int:
    """The calling thread's current CUDA device (0 when none is usable)."""
    d = C.c_int(0)
    if lib().fdg_get_device(C.byref(d)) != FDG_OK:
        return 0
    return d.value


_FLT_MAX = float(np.finfo(np.float32).max)


def validate_image(a: np.ndarray, where: str):
    """rl.hpp:78-83 on the caller's own values (before the fp32 conversion of
    the GPU path): the first non-finite or negative pixel in row-major order
    decides the message (non-finite first at the same pixel).  Finite values
    beyond the fp32 range cannot be represented on the device and are
    refused with their own message (the reference would accept them)."""
    if a.dtype == np.float32 or a.size == 0:
        return  # exactly what the device sees; validated there
    v = np.asarray(a, dtype=np.float64).ravel()
    bad_nf = np.flatnonzero(~np.isfinite(v))
    bad_neg = np.flatnonzero(v < 0)
    i_nf = bad_nf[0] if bad_nf.size else None
    i_neg = bad_neg[0] if bad_neg.size else None
    if i_nf is not None and (i_neg is None or i_nf <= i_neg):
        raise FdgInvalidArgument(f"{where}: input image has non-finite pixels")
    if i_neg is not None:
        raise FdgInvalidArgument(f"{where}: input image must be nonnegative")
    if v.size and float(v.max()) > _FLT_MAX:
        raise FdgInvalidArgument(f"{where}: input pixel exceeds the fp32 range of the GPU path")


def f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def u8ptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_uint8))
