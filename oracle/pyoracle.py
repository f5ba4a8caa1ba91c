"""ctypes face of the CPU oracle (oracle/liboracle.so) and of the compiled
reference (oracle/_ref/libfdref.so).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs -- never from the
product package.  PSF arguments are duck-typed: any object with ``raw()``
returning the constructor inputs (see paper_1304_7211_b200.psf) works.

Operator kinds use the reference numbering (convolve.hpp:22-32).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NAIVE, LIST, GENERIC_BOX, BOX2D_SLIDING, BOX2D_CUMUL, BOX1D_SLIDING, BOX1D_CUMUL, FOURIER, AUTO = range(9)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


class OracleError(RuntimeError):
    pass


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _u8(a):
    return a.ctypes.data_as(_u8p) if a is not None else None


def _load(path):
    if not os.path.exists(path):
        raise OracleError(f"{path} not built (run `make oracle ref` or __graft_entry__.build())")
    return C.CDLL(path)


# --------------------------------------------------------------- the oracle
_orc = None


class _OrcPsf(C.Structure):
    _fields_ = [("repr", C.c_int), ("width", C.c_int), ("height", C.c_int), ("anchor_x", C.c_int),
                ("anchor_y", C.c_int), ("weights", _dp), ("n_rows", C.c_int), ("row_dy", _ip),
                ("row_xmin", _ip), ("row_xmax", _ip), ("support", C.c_int), ("uniform_w", C.c_double),
                ("n_taps", C.c_int), ("tap_dx", _ip), ("tap_dy", _ip), ("tap_w", _dp)]


def orc():
    global _orc
    if _orc is None:
        L = _load(os.path.join(HERE, "liboracle.so"))
        P = C.POINTER(_OrcPsf)
        L.orc_psf_dense.restype = P
        L.orc_psf_dense.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.orc_psf_convex.restype = P
        L.orc_psf_convex.argtypes = [C.c_int, _ip, _ip, _ip]
        L.orc_psf_sparse.restype = P
        L.orc_psf_sparse.argtypes = [C.c_int, _ip, _ip, _dp]
        L.orc_psf_free.argtypes = [P]
        L.orc_psf_adjoint.restype = P
        L.orc_psf_adjoint.argtypes = [P]
        L.orc_psf_to_sparse.restype = P
        L.orc_psf_to_sparse.argtypes = [P]
        L.orc_dispatch.argtypes = [P, C.c_int]
        L.orc_convolve.argtypes = [_dp, C.c_int, C.c_int, P, C.c_int, _dp, _u64p]
        L.orc_masked_convolve.argtypes = [_dp, C.c_int, C.c_int, P, C.c_int, _u8p, _dp, _dp, _u64p]
        L.orc_rl_deconvolve.argtypes = [_dp, C.c_int, C.c_int, P, C.c_int, C.c_int, C.c_double, C.c_int,
                                        _dp, _dp, _dp, _ip]
        L.orc_rl_selective.argtypes = [_dp, C.c_int, C.c_int, P, C.c_int, C.c_int, C.c_double, C.c_int,
                                       C.c_double, C.c_int, C.c_int, _dp, _dp, _dp, _u8p, _ip]
        L.orc_rl_step.argtypes = [_dp, _dp, C.c_int, C.c_int, P, C.c_int, C.c_double, C.c_int, _dp, _dp]
        L.orc_mask_runs.restype = C.c_int64
        L.orc_mask_runs.argtypes = [_u8p, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int64]
        L.orc_active_list.restype = C.c_int64
        L.orc_active_list.argtypes = [_u8p, C.c_int64, C.POINTER(C.c_int64), C.c_int64]
        L.orc_num_threads.restype = C.c_int
        _orc = L
    return _orc


class OPsf:
    """Owned oracle PSF built from a duck-typed PSF's ``raw()`` inputs."""

    def __init__(self, psf):
        r = psf.raw() if hasattr(psf, "raw") else psf
        L = orc()
        self._keep = []
        if r["repr"] == 0:
            w = np.ascontiguousarray(r["weights"], dtype=np.float64)
            self.p = L.orc_psf_dense(r["width"], r["height"], r["anchor_x"], r["anchor_y"], _d(w))
        elif r["repr"] == 1:
            dy, lo, hi = (np.ascontiguousarray(a, dtype=np.int32) for a in r["rows"])
            self.p = L.orc_psf_convex(len(dy), _i(dy), _i(lo), _i(hi))
        else:
            dx, dy = (np.ascontiguousarray(a, dtype=np.int32) for a in r["taps"][:2])
            w = np.ascontiguousarray(r["taps"][2], dtype=np.float64)
            self.p = L.orc_psf_sparse(len(dx), _i(dx), _i(dy), _d(w))
        if not self.p:
            raise OracleError("invalid PSF")
        self.repr = r["repr"]

    def __del__(self):
        try:
            orc().orc_psf_free(self.p)
        except Exception:
            pass

    def taps(self, adjoint=False):
        """normalised tap list of toSparse(psf) (psf.hpp:314-332)."""
        L = orc()
        src = L.orc_psf_adjoint(self.p) if adjoint else self.p
        s = L.orc_psf_to_sparse(src)
        n = s.contents.n_taps
        out = (np.array(s.contents.tap_dx[:n]), np.array(s.contents.tap_dy[:n]),
               np.array(s.contents.tap_w[:n]))
        L.orc_psf_free(s)
        if adjoint:
            L.orc_psf_free(src)
        return out


def _img(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def dispatch(psf, preference=AUTO):
    _op = OPsf(psf)
    return orc().orc_dispatch(_op.p, preference)


def convolve(img, psf, kind=AUTO, counters=False):
    _op = OPsf(psf)
    img = _img(img)
    h, w = img.shape
    out = np.empty_like(img)
    cnt = np.zeros(3, dtype=np.uint64)
    st = orc().orc_convolve(_d(img), w, h, _op.p, kind, _d(out), cnt.ctypes.data_as(_u64p))
    if st:
        raise OracleError(f"orc_convolve status {st}")
    return (out, cnt) if counters else out


def masked_convolve(img, psf, kind, active, fallback, counters=False):
    _op = OPsf(psf)
    img = _img(img)
    h, w = img.shape
    act = np.ascontiguousarray(active, dtype=np.uint8)
    fb = _img(fallback)
    out = np.empty_like(img)
    cnt = np.zeros(3, dtype=np.uint64)
    st = orc().orc_masked_convolve(_d(img), w, h, _op.p, kind, _u8(act), _d(fb), _d(out),
                                   cnt.ctypes.data_as(_u64p))
    if st:
        raise OracleError(f"orc_masked_convolve status {st}")
    return (out, cnt) if counters else out


def rl_deconvolve(f, psf, iterations=100, op=AUTO, eps=1e-8, clamp=True):
    """rlDeconvolve; returns (u, max_change[iterations], seconds[iterations])."""
    _op = OPsf(psf)
    f = _img(f)
    h, w = f.shape
    u = np.empty_like(f)
    mc = np.zeros(max(iterations, 1))
    sec = np.zeros(max(iterations, 1))
    nan_it = C.c_int(0)
    st = orc().orc_rl_deconvolve(_d(f), w, h, _op.p, iterations, op, eps, int(clamp), _d(u),
                                 _d(mc), _d(sec), C.byref(nan_it))
    if st == 2:
        raise OracleError(f"NaN in iterate at iteration {nan_it.value}")
    if st:
        raise OracleError(f"orc_rl_deconvolve status {st}")
    return u, mc[:iterations], sec[:iterations]


def rl_selective(f, psf, iterations, threshold, period=10, thin_start=0, op=AUTO, eps=1e-8,
                 clamp=True, record_masks=False):
    """rlDeconvolveSelective (+thin_start); returns (u, inactive, max_change, masks|None)."""
    _op = OPsf(psf)
    f = _img(f)
    h, w = f.shape
    u = np.empty_like(f)
    inact = np.zeros(max(iterations, 1))
    mc = np.zeros(max(iterations, 1))
    masks = np.zeros((iterations, h, w), dtype=np.uint8) if record_masks else None
    nan_it = C.c_int(0)
    st = orc().orc_rl_selective(_d(f), w, h, _op.p, iterations, op, eps, int(clamp),
                                threshold, period, thin_start, _d(u), _d(inact), _d(mc),
                                _u8(masks), C.byref(nan_it))
    if st == 2:
        raise OracleError(f"NaN in iterate at iteration {nan_it.value}")
    if st:
        raise OracleError(f"orc_rl_selective status {st}")
    return u, inact[:iterations], mc[:iterations], masks


def rl_step(u, f, psf, op=AUTO, eps=1e-8, clamp=True):
    _op = OPsf(psf)
    u = _img(u)
    f = _img(f)
    h, w = f.shape
    out = np.empty_like(f)
    mc = C.c_double(0)
    st = orc().orc_rl_step(_d(u), _d(f), w, h, _op.p, op, eps, int(clamp), _d(out), C.byref(mc))
    if st:
        raise OracleError(f"orc_rl_step status {st}")
    return out


def mask_runs(active):
    """(y, x0, len) active runs in the row-major order of convolve.hpp:450-465."""
    act = np.ascontiguousarray(active, dtype=np.uint8)
    h, w = act.shape
    n = orc().orc_mask_runs(_u8(act), w, h, None, 0)
    runs = np.zeros((max(n, 1), 3), dtype=np.int32)
    orc().orc_mask_runs(_u8(act), w, h, runs.ctypes.data_as(C.POINTER(C.c_int32)), n)
    return runs[:n]


def active_list(active):
    act = np.ascontiguousarray(active, dtype=np.uint8).ravel()
    n = orc().orc_active_list(_u8(act), act.size, None, 0)
    idx = np.zeros(max(n, 1), dtype=np.int64)
    orc().orc_active_list(_u8(act), act.size, idx.ctypes.data_as(C.POINTER(C.c_int64)), n)
    return idx[:n]


def num_threads():
    return orc().orc_num_threads()


# ------------------------------------------------- the compiled reference
_ref = None


class _RefPsf(C.Structure):
    _fields_ = [("repr", C.c_int), ("width", C.c_int), ("height", C.c_int), ("anchor_x", C.c_int),
                ("anchor_y", C.c_int), ("weights", _dp), ("n_rows", C.c_int), ("row_dy", _ip),
                ("row_xmin", _ip), ("row_xmax", _ip), ("n_taps", C.c_int), ("tap_dx", _ip),
                ("tap_dy", _ip), ("tap_w", _dp)]


def ref_available():
    return os.path.exists(os.path.join(HERE, "_ref", "libfdref.so"))


def ref():
    global _ref
    if _ref is None:
        L = _load(os.path.join(HERE, "_ref", "libfdref.so"))
        P = C.POINTER(_RefPsf)
        L.fdref_last_error.restype = C.c_char_p
        L.fdref_dispatch.argtypes = [P, C.c_int]
        L.fdref_psf_taps.argtypes = [P, C.c_int, _ip, _ip, _dp, C.c_int]
        L.fdref_convolve.argtypes = [P, C.c_int, _dp, C.c_int, C.c_int, _dp, _u64p]
        L.fdref_masked_convolve.argtypes = [P, C.c_int, _dp, C.c_int, C.c_int, _u8p, _dp, _dp, _u64p]
        L.fdref_rl_deconvolve.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_int, _dp, C.c_int, C.c_int,
                                          _dp, _dp, _dp]
        L.fdref_rl_selective.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                         _dp, C.c_int, C.c_int, _dp, _dp, _dp]
        L.fdref_rl_selective_from.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double,
                                              C.c_int, C.c_int, _dp, C.c_int, C.c_int, _dp, _dp, _dp, _u8p]
        L.fdref_rl_step.argtypes = [P, C.c_int, C.c_double, C.c_int, _dp, _dp, C.c_int, C.c_int, _dp]
        L.fdref_bench_strips.restype = C.c_double
        L.fdref_bench_strips.argtypes = [P, C.c_int, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.POINTER(C.c_double)]
        _ref = L
    return _ref


class RPsf:
    def __init__(self, psf):
        r = psf.raw() if hasattr(psf, "raw") else psf
        self.s = _RefPsf()
        self.s.repr = r["repr"]
        self._keep = []
        if r["repr"] == 0:
            w = np.ascontiguousarray(r["weights"], dtype=np.float64)
            self._keep.append(w)
            self.s.width, self.s.height = r["width"], r["height"]
            self.s.anchor_x, self.s.anchor_y = r["anchor_x"], r["anchor_y"]
            self.s.weights = _d(w)
        elif r["repr"] == 1:
            arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in r["rows"]]
            self._keep += arrs
            self.s.n_rows = len(arrs[0])
            self.s.row_dy, self.s.row_xmin, self.s.row_xmax = (_i(a) for a in arrs)
        else:
            dx, dy = (np.ascontiguousarray(a, dtype=np.int32) for a in r["taps"][:2])
            w = np.ascontiguousarray(r["taps"][2], dtype=np.float64)
            self._keep += [dx, dy, w]
            self.s.n_taps = len(dx)
            self.s.tap_dx, self.s.tap_dy, self.s.tap_w = _i(dx), _i(dy), _d(w)

    @property
    def p(self):
        return C.byref(self.s)


def _ref_check(st):
    if st:
        raise OracleError(ref().fdref_last_error().decode())


def ref_dispatch(psf, preference=AUTO):
    _rp = RPsf(psf)
    return ref().fdref_dispatch(_rp.p, preference)


def ref_taps(psf, adjoint=False):
    rp = RPsf(psf)
    n = ref().fdref_psf_taps(rp.p, int(adjoint), None, None, None, 0)
    dx = np.zeros(n, np.int32)
    dy = np.zeros(n, np.int32)
    w = np.zeros(n)
    ref().fdref_psf_taps(rp.p, int(adjoint), _i(dx), _i(dy), _d(w), n)
    return dx, dy, w


def ref_convolve(img, psf, kind=AUTO, counters=False):
    _rp = RPsf(psf)
    img = _img(img)
    h, w = img.shape
    out = np.empty_like(img)
    cnt = np.zeros(3, dtype=np.uint64)
    _ref_check(ref().fdref_convolve(_rp.p, kind, _d(img), w, h, _d(out), cnt.ctypes.data_as(_u64p)))
    return (out, cnt) if counters else out


def ref_masked_convolve(img, psf, kind, active, fallback, counters=False):
    _rp = RPsf(psf)
    img = _img(img)
    h, w = img.shape
    act = np.ascontiguousarray(active, dtype=np.uint8)
    fb = _img(fallback)
    out = np.empty_like(img)
    cnt = np.zeros(3, dtype=np.uint64)
    _ref_check(ref().fdref_masked_convolve(_rp.p, kind, _d(img), w, h, _u8(act), _d(fb), _d(out),
                                           cnt.ctypes.data_as(_u64p)))
    return (out, cnt) if counters else out


def ref_rl_deconvolve(f, psf, iterations=100, op=AUTO, eps=1e-8, clamp=True):
    _rp = RPsf(psf)
    f = _img(f)
    h, w = f.shape
    u = np.empty_like(f)
    mc = np.zeros(max(iterations, 1))
    sec = np.zeros(max(iterations, 1))
    _ref_check(ref().fdref_rl_deconvolve(_rp.p, iterations, op, eps, int(clamp), _d(f), w, h,
                                         _d(u), _d(mc), _d(sec)))
    return u, mc[:iterations], sec[:iterations]


def ref_rl_selective(f, psf, iterations, threshold, period=10, op=AUTO, eps=1e-8, clamp=True):
    _rp = RPsf(psf)
    f = _img(f)
    h, w = f.shape
    u = np.empty_like(f)
    inact = np.zeros(max(iterations, 1))
    mc = np.zeros(max(iterations, 1))
    _ref_check(ref().fdref_rl_selective(_rp.p, iterations, op, eps, int(clamp), threshold, period,
                                        _d(f), w, h, _d(u), _d(inact), _d(mc)))
    return u, inact[:iterations], mc[:iterations]


def ref_rl_selective_from(f, psf, iterations, threshold, period=10, thin_start=0, op=AUTO, eps=1e-8,
                          clamp=True, record_masks=False):
    _rp = RPsf(psf)
    f = _img(f)
    h, w = f.shape
    u = np.empty_like(f)
    inact = np.zeros(max(iterations, 1))
    mc = np.zeros(max(iterations, 1))
    masks = np.zeros((iterations, h, w), dtype=np.uint8) if record_masks else None
    _ref_check(ref().fdref_rl_selective_from(_rp.p, iterations, op, eps, int(clamp), threshold,
                                             period, thin_start, _d(f), w, h, _d(u), _d(inact), _d(mc),
                                             _u8(masks)))
    return u, inact[:iterations], mc[:iterations], masks


def ref_rl_step(u, f, psf, op=AUTO, eps=1e-8, clamp=True):
    _rp = RPsf(psf)
    u = _img(u)
    f = _img(f)
    h, w = f.shape
    out = np.empty_like(f)
    _ref_check(ref().fdref_rl_step(_rp.p, op, eps, int(clamp), _d(u), _d(f), w, h, _d(out)))
    return out


def ref_bench_strips(f, psf, op, iterations, threads, strip_rows):
    """Wall seconds and px*it of `threads` independent reference rlDeconvolve
    runs on strips of f (the reference is single-threaded by design)."""
    _rp = RPsf(psf)
    f = _img(f)
    h, w = f.shape
    pxit = C.c_double(0)
    secs = ref().fdref_bench_strips(_rp.p, op, _d(f), w, h, iterations, threads, strip_rows,
                                    C.byref(pxit))
    return secs, pxit.value
