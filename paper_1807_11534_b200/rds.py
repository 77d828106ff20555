"""Thin Python binding of librds (include/rds.h) via ctypes -- argument marshalling only.

Every computation runs in the CUDA kernels of ``librds.so``; this module only converts
numpy arrays (host, ``on_device=0``) or torch CUDA tensors (device, ``on_device=1``) to
pointers and checks return codes.  There is no CPU fallback: if the library is missing this
module raises at import time.

Function names mirror the C ABI (``rds_create``, ``rds_solve``, ...).  ``Solver`` is a small
convenience wrapper around a handle.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "librds.so")

RDS_OK, RDS_EINVAL, RDS_ESTATE, RDS_ECUDA, RDS_ENOMEM = 0, -1, -2, -3, -4
RDS_LABEL_BG, RDS_LABEL_FG, RDS_LABEL_RD = 0, 1, 2
RDS_OPT_KFUSE, RDS_OPT_ITEM_ROWS, RDS_OPT_TIMING, RDS_OPT_SKIP, RDS_OPT_GRAPH = 1, 2, 3, 4, 5
RDS_OPT_CTAS_PER_SM = 6
RDS_OPT_STOP_NORM = 7  # 0 Euclidean over pixels (default), 1 RMS
RDS_OPT_COMPACT = 8    # f3: 0 dense stencil, 1 compacted RD iteration, 2 auto (default)
RDS_OPT_WAVE = 9       # temporal wavefront for fixed-K solves: 0 off (default), 1 on, 2 auto
RDS_OPT_RESIDENT = 10  # small images as one resident cluster: 0 off, 1 / 2 (default) on
RDS_OPT_PROLOGUE = 14  # plain stencil launches in the prologue form: 0 off, 1 on, 2 auto (default)
RDS_OPT_WS = 13        # full-depth launches on the warp-specialised stencil: 0 off (default), 1 on
RDS_OPT_PERSIST = 11   # fixed-K loop as one persistent launch: 0 off (default), 1 on, 2 auto
RDS_OPT_RDC_SPLIT = 15 # compact fixed-K solves: 1 decoupled RD pixels iterate alone, 2 (default) also small connected components inside one warp / CTA, 0 off
RDS_OPT_GRID = 12      # mid-size images resident on the whole GPU: 0 off (default), 1 / 2 on

EXPORTS = (
    "rds_create", "rds_create_batch", "rds_destroy", "rds_set_stream", "rds_set_option",
    "rds_set_image",
    "rds_set_fitting", "rds_set_state", "rds_fitting_absmax", "rds_solve", "rds_get_u",
    "rds_get_mask", "rds_get_v", "rds_get_p", "rds_get_fitting", "rds_get_labels",
    "rds_get_active_tiles", "rds_tile_shape", "rds_energy", "rds_get_stats",
    "rds_kfuse_supported", "rds_last_error", "rds_version", "rds_band_for_fraction",
    "rds_solve_q", "rds_solve_tol", "rds_solve_gt", "rds_get_u_gt", "rds_compare_gt",
    "rds_check_frame", "rds_solve_continue", "rds_get_state_rows", "rds_set_state_rows",
    "rds_set_energy_rows", "rds_continue_check", "rds_abs_histogram",
    "rds3_create", "rds3_destroy", "rds3_set_stream", "rds3_set_kz", "rds3_set_kfuse",
    "rds3_set_image",
    "rds3_set_fitting",
    "rds3_fitting_absmax", "rds3_solve", "rds3_get_u", "rds3_get_v", "rds3_get_p",
    "rds3_get_mask", "rds3_get_labels", "rds3_get_stats", "rds3_last_error",
)


class RdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rds error {code}: {msg}")
        self.code = code


class rds_energy_t(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("E_v", "E_u", "D_p", "gap", "TV_v", "fit_v",
                                                "F_rd")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class rds_gt_t(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("residual", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class rds_stats_t(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int64), ("W", ctypes.c_int64), ("n_rd", ctypes.c_int64),
                ("n_tiles", ctypes.c_int64), ("n_active_tiles", ctypes.c_int64),
                ("n_items", ctypes.c_int64), ("n_active_items", ctypes.c_int64),
                ("n_active_cells", ctypes.c_int64),
                ("iters", ctypes.c_int32), ("k_fuse", ctypes.c_int32),
                ("launches", ctypes.c_int32), ("item_rows", ctypes.c_int32),
                ("item_cols", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("setup_ms", ctypes.c_float), ("loop_ms", ctypes.c_float),
                ("residual", ctypes.c_float), ("check_every", ctypes.c_int32),
                ("compact", ctypes.c_int32), ("wave", ctypes.c_int32),
                ("resident", ctypes.c_int32), ("persist", ctypes.c_int32),
                ("rdc_decoupled", ctypes.c_int32),
                ("rdc_grouped", ctypes.c_int32),
                ("rdc_label_rounds", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (no CPU fallback exists)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i64, i32, f, i = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_int
    sig = {
        "rds_create": [i64, i64, ctypes.POINTER(P)],
        "rds_create_batch": [i64, i64, i64, ctypes.POINTER(P)],
        "rds_destroy": [P],
        "rds_set_stream": [P, P],
        "rds_set_option": [P, i, i64],
        "rds_set_image": [P, P, i],
        "rds_set_fitting": [P, f, f, f, P, i],
        "rds_set_state": [P, P, P, P, i],
        "rds_fitting_absmax": [P, ctypes.POINTER(f)],
        "rds_solve": [P, f, f, f, f, i32],
        "rds_get_u": [P, P, i],
        "rds_get_mask": [P, P, i],
        "rds_get_v": [P, P, i],
        "rds_get_p": [P, P, P, i],
        "rds_get_fitting": [P, P, i],
        "rds_get_labels": [P, P, i],
        "rds_get_active_tiles": [P, P, i64, ctypes.POINTER(i64)],
        "rds_tile_shape": [ctypes.POINTER(i), ctypes.POINTER(i)],
        "rds_energy": [P, ctypes.POINTER(rds_energy_t)],
        "rds_get_stats": [P, ctypes.POINTER(rds_stats_t)],
        "rds_kfuse_supported": [ctypes.POINTER(i32), i],
        "rds_last_error": [P],
        "rds_version": [],
        "rds_band_for_fraction": [P, ctypes.c_double, ctypes.POINTER(f)],
        "rds_solve_q": [P, f, f, f, ctypes.c_double, i32],
        "rds_solve_tol": [P, f, f, f, f, i32, f, i32],
        "rds_solve_gt": [P, f, f, f, f, i32, ctypes.c_double, i32, ctypes.POINTER(rds_gt_t)],
        "rds_get_u_gt": [P, P, i],
        "rds_compare_gt": [P, f, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
        "rds_check_frame": [P, ctypes.POINTER(i64)],
        "rds_solve_continue": [P, i32],
        "rds_get_state_rows": [P, i64, i64, P, i],
        "rds_set_state_rows": [P, i64, i64, P, i],
        "rds_set_energy_rows": [P, i64, i64],
        "rds_continue_check": [P, i32, i64, i64, ctypes.POINTER(ctypes.c_double)],
        "rds_abs_histogram": [P, i64, i64, ctypes.c_uint32, ctypes.c_uint32, i32,
                              ctypes.POINTER(ctypes.c_uint32)],
        "rds3_create": [i64, i64, i64, ctypes.POINTER(P)],
        "rds3_destroy": [P],
        "rds3_set_stream": [P, P],
        "rds3_set_kz": [P, i32],
        "rds3_set_kfuse": [P, i32],
        "rds3_set_image": [P, P, i],
        "rds3_set_fitting": [P, f, f, f, P, i],
        "rds3_fitting_absmax": [P, ctypes.POINTER(f)],
        "rds3_solve": [P, f, f, f, f, i32],
        "rds3_get_u": [P, P, i],
        "rds3_get_v": [P, P, i],
        "rds3_get_p": [P, P, P, P, i],
        "rds3_get_mask": [P, P, i],
        "rds3_get_labels": [P, P, i],
        "rds3_get_stats": [P, ctypes.POINTER(i64), ctypes.POINTER(i32), ctypes.POINTER(i32),
                           ctypes.POINTER(f)],
        "rds3_last_error": [P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.rds_last_error.restype = ctypes.c_char_p
    lib.rds3_last_error.restype = ctypes.c_char_p
    lib.rds_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


def _check(rc, h=None):
    if rc != RDS_OK:
        raise RdsError(rc, _lib.rds_last_error(h).decode())
    return rc


def _buf(a, dtype, shape, writable=False):
    """(pointer, on_device, keepalive) for a numpy array or torch tensor of `dtype`/`shape`."""
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):  # torch tensor
        import torch

        tdt = {np.float32: torch.float32, np.uint8: torch.uint8, np.int32: torch.int32,
               np.float64: torch.float64}[dtype]
        if a.dtype != tdt or tuple(a.shape) != tuple(shape) or not a.is_contiguous():
            raise ValueError(f"expected contiguous {tdt} tensor of shape {shape}")
        return ctypes.c_void_p(a.data_ptr()), int(a.is_cuda), a
    arr = np.asarray(a)
    if arr.dtype != dtype or arr.shape != tuple(shape) or not arr.flags.c_contiguous or \
            (writable and not arr.flags.writeable):
        raise ValueError(f"expected C-contiguous {np.dtype(dtype)} array of shape {shape}")
    return ctypes.c_void_p(arr.ctypes.data), 0, arr


# ------------------------------------------------------------------------------------------
# C-ABI mirror
# ------------------------------------------------------------------------------------------

def rds_create(H, W):
    h = ctypes.c_void_p()
    _check(_lib.rds_create(int(H), int(W), ctypes.byref(h)))
    return h


def rds_destroy(h):
    _check(_lib.rds_destroy(h))


CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: what torch's default stream (cuda_stream 0) is


def _stream_arg(stream_ptr):
    """None -> NULL (the handle's private stream); 0 (torch's default stream) ->
    cudaStreamLegacy, so that `torch.cuda.current_stream().cuda_stream` always means the
    stream torch is using; anything else is a cudaStream_t."""
    if stream_ptr is None:
        return ctypes.c_void_p(None)
    return ctypes.c_void_p(int(stream_ptr) or CUDA_STREAM_LEGACY)


def rds_set_stream(h, stream_ptr):
    _check(_lib.rds_set_stream(h, _stream_arg(stream_ptr)), h)


def rds_set_option(h, key, value):
    _check(_lib.rds_set_option(h, int(key), int(value)), h)


def rds_set_image(h, z, shape):
    p, dev, _keep = _buf(z, np.float32, shape)
    _check(_lib.rds_set_image(h, p, dev), h)


def rds_set_fitting(h, c1, c2, gamma, P, shape):
    if P is None:
        p, dev = None, 0
    else:
        p, dev, _keep = _buf(P, np.float32, shape)
    _check(_lib.rds_set_fitting(h, float(c1), float(c2), float(gamma), p, dev), h)


def rds_set_state(h, v, rho1, rho2, shape):
    pv, dev, _k1 = _buf(v, np.float32, shape)
    p1, dev1, _k2 = _buf(rho1, np.float32, shape)
    p2, dev2, _k3 = _buf(rho2, np.float32, shape)
    if not (dev == dev1 == dev2):
        raise ValueError("v, rho1, rho2 must all be host or all device")
    _check(_lib.rds_set_state(h, pv, p1, p2, dev), h)


def rds_fitting_absmax(h):
    out = ctypes.c_float()
    _check(_lib.rds_fitting_absmax(h, ctypes.byref(out)), h)
    return np.float32(out.value)


def rds_band_for_fraction(h, q):
    out = ctypes.c_float()
    _check(_lib.rds_band_for_fraction(h, float(q), ctypes.byref(out)), h)
    return np.float32(out.value)


def rds_solve_q(h, lam, theta, tau, q, iters):
    _check(_lib.rds_solve_q(h, float(lam), float(theta), float(tau), float(q), int(iters)), h)


def rds_solve(h, lam, theta, tau, delta, iters):
    _check(_lib.rds_solve(h, float(lam), float(theta), float(tau), float(delta), int(iters)), h)


def rds_solve_tol(h, lam, theta, tau, delta, max_iters, tol, check_every=0):
    _check(_lib.rds_solve_tol(h, float(lam), float(theta), float(tau), float(delta),
                              int(max_iters), float(tol), int(check_every)), h)


def rds_solve_gt(h, lam, theta, tau, delta, max_iters, tol, check_every):
    r = rds_gt_t()
    _check(_lib.rds_solve_gt(h, float(lam), float(theta), float(tau), float(delta),
                             int(max_iters), float(tol), int(check_every), ctypes.byref(r)), h)
    return r.as_dict()


def rds_compare_gt(h, eps=0.5):
    e1, e2 = ctypes.c_double(), ctypes.c_double()
    _check(_lib.rds_compare_gt(h, float(eps), ctypes.byref(e1), ctypes.byref(e2)), h)
    return e1.value, e2.value


def rds_solve_continue(h, iters):
    _check(_lib.rds_solve_continue(h, int(iters)), h)


def rds_get_state_rows(h, row0, nrows, out, W):
    """rows [row0, row0 + nrows) of (v, rho1, rho2) into out (3, nrows, W) float32."""
    p, dev, _keep = _buf(out, np.float32, (3, nrows, W), writable=True)
    _check(_lib.rds_get_state_rows(h, int(row0), int(nrows), p, dev), h)
    return out


def rds_set_state_rows(h, row0, buf, W):
    nrows = int(buf.shape[1])
    p, dev, _keep = _buf(buf, np.float32, (3, nrows, W))
    _check(_lib.rds_set_state_rows(h, int(row0), nrows, p, dev), h)


def rds_set_energy_rows(h, row0, row1):
    _check(_lib.rds_set_energy_rows(h, int(row0), int(row1)), h)


def rds_continue_check(h, iters, row0, row1):
    """(sum du^2, sum dv^2) of the last of `iters` continued iterations over rows [row0, row1)."""
    out = (ctypes.c_double * 2)()
    _check(_lib.rds_continue_check(h, int(iters), int(row0), int(row1), out), h)
    return out[0], out[1]


def rds_abs_histogram(h, row0, row1, prefix, mask, shift):
    """256 counts of byte `shift` of |f|'s bit pattern over rows [row0, row1) (radix pass)."""
    out = (ctypes.c_uint32 * 256)()
    _check(_lib.rds_abs_histogram(h, int(row0), int(row1), int(prefix), int(mask), int(shift),
                                  out), h)
    return np.frombuffer(out, dtype=np.uint32).copy()


def _get(fn, h, out, dtype, shape):
    p, dev, _keep = _buf(out, dtype, shape, writable=True)
    _check(fn(h, p, dev), h)
    return out


def rds_get_u(h, out, shape):
    return _get(_lib.rds_get_u, h, out, np.float32, shape)


def rds_get_mask(h, out, shape):
    return _get(_lib.rds_get_mask, h, out, np.uint8, shape)


def rds_get_v(h, out, shape):
    return _get(_lib.rds_get_v, h, out, np.float32, shape)


def rds_get_fitting(h, out, shape):
    return _get(_lib.rds_get_fitting, h, out, np.float32, shape)


def rds_get_labels(h, out, shape):
    return _get(_lib.rds_get_labels, h, out, np.uint8, shape)


def rds_get_p(h, rho1, rho2, shape):
    p1, dev1, _k1 = _buf(rho1, np.float32, shape, writable=True)
    p2, dev2, _k2 = _buf(rho2, np.float32, shape, writable=True)
    if dev1 != dev2:
        raise ValueError("rho1 and rho2 must both be host or both device")
    _check(_lib.rds_get_p(h, p1, p2, dev1), h)
    return rho1, rho2


def rds_get_active_tiles(h):
    cnt = ctypes.c_int64()
    rc = _lib.rds_get_active_tiles(h, None, 0, ctypes.byref(cnt))
    if rc not in (RDS_OK, RDS_EINVAL):
        _check(rc, h)
    out = np.empty(max(cnt.value, 1), dtype=np.int32)
    _check(_lib.rds_get_active_tiles(h, ctypes.c_void_p(out.ctypes.data), out.size,
                                     ctypes.byref(cnt)), h)
    return out[: cnt.value].copy()


def rds_tile_shape():
    th, tw = ctypes.c_int(), ctypes.c_int()
    _check(_lib.rds_tile_shape(ctypes.byref(th), ctypes.byref(tw)))
    return th.value, tw.value


def rds_energy(h):
    e = rds_energy_t()
    _check(_lib.rds_energy(h, ctypes.byref(e)), h)
    return e.as_dict()


def rds_get_stats(h):
    s = rds_stats_t()
    _check(_lib.rds_get_stats(h, ctypes.byref(s)), h)
    return s.as_dict()


def rds_kfuse_supported():
    buf = (ctypes.c_int32 * 64)()
    n = _lib.rds_kfuse_supported(buf, 64)
    return [buf[i] for i in range(min(n, 64))]


def rds_last_error(h=None):
    return _lib.rds_last_error(h).decode()


def rds_version():
    return _lib.rds_version().decode()


# ------------------------------------------------------------------------------------------
# convenience wrapper
# ------------------------------------------------------------------------------------------

class Solver:
    """One librds handle for an H x W image.  Host (numpy) or device (torch) buffers."""

    def __init__(self, H, W, stream=None, k_fuse=0, item_rows=0, timing=False, skip=True,
                 graph=True, batch=None, compact=None, wave=None, resident=None,
                 persist=None, grid=None, ws=None, prologue=None, rdc_split=None):
        self.shape = (int(H) * (int(batch) if batch else 1), int(W))
        if batch is not None:
            h = ctypes.c_void_p()
            _check(_lib.rds_create_batch(int(batch), int(H), int(W), ctypes.byref(h)))
            self.h = h
        else:
            self.h = rds_create(H, W)
        if stream is not None:
            rds_set_stream(self.h, stream)
        if k_fuse:
            rds_set_option(self.h, RDS_OPT_KFUSE, k_fuse)
        if item_rows:
            rds_set_option(self.h, RDS_OPT_ITEM_ROWS, item_rows)
        rds_set_option(self.h, RDS_OPT_TIMING, int(timing))
        rds_set_option(self.h, RDS_OPT_SKIP, int(skip))
        rds_set_option(self.h, RDS_OPT_GRAPH, int(graph))
        if compact is not None:  # None: the library default (2, auto)
            rds_set_option(self.h, RDS_OPT_COMPACT, int(compact))
        if wave is not None:
            rds_set_option(self.h, RDS_OPT_WAVE, int(wave))
        if resident is not None:
            rds_set_option(self.h, RDS_OPT_RESIDENT, int(resident))
        if persist is not None:
            rds_set_option(self.h, RDS_OPT_PERSIST, int(persist))
        if grid is not None:
            rds_set_option(self.h, RDS_OPT_GRID, int(grid))
        if ws is not None:
            rds_set_option(self.h, RDS_OPT_WS, int(ws))
        if prologue is not None:
            rds_set_option(self.h, RDS_OPT_PROLOGUE, int(prologue))
        if rdc_split is not None:
            rds_set_option(self.h, RDS_OPT_RDC_SPLIT, int(rdc_split))

    def close(self):
        if self.h is not None:
            rds_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream_ptr):
        rds_set_stream(self.h, stream_ptr)

    def set_option(self, key, value):
        rds_set_option(self.h, key, value)

    def set_image(self, z):
        rds_set_image(self.h, z, self.shape)

    def set_fitting(self, c1, c2, gamma=0.0, P=None):
        rds_set_fitting(self.h, c1, c2, gamma, P, self.shape)

    def set_state(self, v, rho1, rho2):
        rds_set_state(self.h, v, rho1, rho2, self.shape)

    def absmax(self):
        return rds_fitting_absmax(self.h)

    def band_for_fraction(self, q):
        return rds_band_for_fraction(self.h, q)

    def solve_q(self, lam, theta, tau, q, iters):
        rds_solve_q(self.h, lam, theta, tau, q, iters)

    def solve(self, lam, theta, tau, delta, iters):
        rds_solve(self.h, lam, theta, tau, math.inf if delta is None else delta, iters)

    def solve_continue(self, iters):
        """`iters` more iterations from the current state (parameters of the last solve)."""
        rds_solve_continue(self.h, iters)

    def state_rows(self, row0, nrows, out=None):
        """(3, nrows, W) float32: v, rho1, rho2 on rows [row0, row0 + nrows)."""
        W = self.shape[1]
        out = np.empty((3, nrows, W), np.float32) if out is None else out
        return rds_get_state_rows(self.h, row0, nrows, out, W)

    def set_state_rows(self, row0, buf):
        rds_set_state_rows(self.h, row0, buf, self.shape[1])

    def set_energy_rows(self, row0, row1=-1):
        rds_set_energy_rows(self.h, row0, row1)

    def continue_check(self, iters, row0, row1):
        """`iters` more iterations; returns the stopping-rule sums (du^2, dv^2) of the last one
        over rows [row0, row1) (row strips: all-reduce them, strips.StripSolver.solve_tol)."""
        return rds_continue_check(self.h, iters, row0, row1)

    def abs_histogram(self, row0, row1, prefix, mask, shift):
        """One radix pass of the q -> q^ search over rows [row0, row1) (256 counts)."""
        return rds_abs_histogram(self.h, row0, row1, prefix, mask, shift)

    def solve_tol(self, lam, theta, tau, delta, max_iters, tol, check_every=0):
        """Stop at the first check (every check_every iterations, and at max_iters) where
        max(||u^l - u^(l-1)||, ||v^l - v^(l-1)||) <= tol.  The norm is
        the library default RDS_OPT_STOP_NORM = 0, the Euclidean norm over pixels of unit
        area (reading R-F2); set_option(RDS_OPT_STOP_NORM, 1) selects the RMS instead.
        Returns the stats dict (iters, converged, residual)."""
        rds_solve_tol(self.h, lam, theta, tau, math.inf if delta is None else delta,
                      max_iters, tol, check_every)
        return self.stats()

    def solve_gt(self, lam, theta, tau, delta, max_iters, tol, check_every=10):
        """float64 solve to tolerance (PAPER.md:234-238 ground truth; delta=inf = original
        method).  Returns {iters, converged, residual}."""
        return rds_solve_gt(self.h, lam, theta, tau, math.inf if delta is None else delta,
                            max_iters, tol, check_every)

    def u_gt(self, out=None):
        out = np.empty(self.shape, np.float64) if out is None else out
        return _get(_lib.rds_get_u_gt, self.h, out, np.float64, self.shape)

    def compare_gt(self, eps=0.5):
        """(E1, E2) of the current float u against u^GT."""
        return rds_compare_gt(self.h, eps)

    def _out(self, dtype, out):
        return np.empty(self.shape, dtype=dtype) if out is None else out

    def u(self, out=None):
        return rds_get_u(self.h, self._out(np.float32, out), self.shape)

    def mask(self, out=None):
        return rds_get_mask(self.h, self._out(np.uint8, out), self.shape)

    def v(self, out=None):
        return rds_get_v(self.h, self._out(np.float32, out), self.shape)

    def p(self):
        return rds_get_p(self.h, np.empty(self.shape, np.float32),
                         np.empty(self.shape, np.float32), self.shape)

    def fitting(self, out=None):
        return rds_get_fitting(self.h, self._out(np.float32, out), self.shape)

    def labels(self, out=None):
        return rds_get_labels(self.h, self._out(np.uint8, out), self.shape)

    def active_tiles(self):
        return rds_get_active_tiles(self.h)

    def energy(self):
        return rds_energy(self.h)

    def stats(self):
        return rds_get_stats(self.h)

    def check_frame(self):
        """Frame elements outside the image that kernels overwrote (must be 0)."""
        n = ctypes.c_int64()
        _check(_lib.rds_check_frame(self.h, ctypes.byref(n)), self.h)
        return n.value


# ------------------------------------------------------------------------------------------
# f4: 3-D volumes (rds3_*)
# ------------------------------------------------------------------------------------------

def _check3(rc, h):
    if rc != RDS_OK:
        raise RdsError(rc, _lib.rds3_last_error(h).decode() if h else "")


class Solver3:
    """One rds3 handle for a D x H x W volume (host numpy or device torch buffers)."""

    def __init__(self, D, H, W, stream=None):
        self.shape = (int(D), int(H), int(W))
        h = ctypes.c_void_p()
        _check3(_lib.rds3_create(int(D), int(H), int(W), ctypes.byref(h)), None)
        self.h = h
        if stream is not None:
            _check3(_lib.rds3_set_stream(self.h, _stream_arg(stream)), self.h)

    def close(self):
        if self.h is not None:
            _lib.rds3_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_kz(self, kz):
        _check3(_lib.rds3_set_kz(self.h, int(kz)), self.h)

    def set_kfuse(self, kf):
        """Iterations per pass over the volume (1 .. 3; 0 = automatic, 1)."""
        _check3(_lib.rds3_set_kfuse(self.h, int(kf)), self.h)

    def set_image(self, z):
        p, dev, _k = _buf(z, np.float32, self.shape)
        _check3(_lib.rds3_set_image(self.h, p, dev), self.h)

    def set_fitting(self, c1, c2, gamma=0.0, P=None):
        if P is None:
            p, dev, _k = None, 0, None
        else:
            p, dev, _k = _buf(P, np.float32, self.shape)
        _check3(_lib.rds3_set_fitting(self.h, float(c1), float(c2), float(gamma), p, dev), self.h)

    def absmax(self):
        out = ctypes.c_float()
        _check3(_lib.rds3_fitting_absmax(self.h, ctypes.byref(out)), self.h)
        return np.float32(out.value)

    def solve(self, lam, theta, tau, delta, iters):
        _check3(_lib.rds3_solve(self.h, float(lam), float(theta), float(tau),
                                float(math.inf if delta is None else delta), int(iters)), self.h)

    def _get(self, fn, dtype, out):
        out = np.empty(self.shape, dtype) if out is None else out
        p, dev, _k = _buf(out, dtype, self.shape, writable=True)
        _check3(fn(self.h, p, dev), self.h)
        return out

    def u(self, out=None):
        return self._get(_lib.rds3_get_u, np.float32, out)

    def v(self, out=None):
        return self._get(_lib.rds3_get_v, np.float32, out)

    def mask(self, out=None):
        return self._get(_lib.rds3_get_mask, np.uint8, out)

    def labels(self, out=None):
        return self._get(_lib.rds3_get_labels, np.uint8, out)

    def p(self):
        outs = [np.empty(self.shape, np.float32) for _ in range(3)]
        ps = [_buf(o, np.float32, self.shape, writable=True) for o in outs]
        _check3(_lib.rds3_get_p(self.h, ps[0][0], ps[1][0], ps[2][0], 0), self.h)
        return tuple(outs)

    def stats(self):
        n_rd, it, kz, ms = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_float()
        _check3(_lib.rds3_get_stats(self.h, ctypes.byref(n_rd), ctypes.byref(it),
                                    ctypes.byref(kz), ctypes.byref(ms)), self.h)
        return {"n_rd": n_rd.value, "iters": it.value, "kz": kz.value, "ms": ms.value}


class BatchSolver(Solver):
    """B independent H x W images solved together (rds_create_batch).  Inputs and outputs are
    (B, H, W) arrays (the same memory as the stacked (B*H, W) problem)."""

    def __init__(self, B, H, W, **kw):
        super().__init__(H, W, batch=B, **kw)
        self.bshape = (int(B), int(H), int(W))

    def _flat(self, a):
        return None if a is None else a.reshape(self.shape)

    def set_image(self, z):
        super().set_image(self._flat(z))

    def set_fitting(self, c1, c2, gamma=0.0, P=None):
        super().set_fitting(c1, c2, gamma, self._flat(P))

    def u(self, out=None):
        return super().u(self._flat(out)).reshape(self.bshape)

    def v(self, out=None):
        return super().v(self._flat(out)).reshape(self.bshape)

    def mask(self, out=None):
        return super().mask(self._flat(out)).reshape(self.bshape)

    def labels(self, out=None):
        return super().labels(self._flat(out)).reshape(self.bshape)

    def fitting(self, out=None):
        return super().fitting(self._flat(out)).reshape(self.bshape)

    def p(self):
        p1, p2 = super().p()
        return p1.reshape(self.bshape), p2.reshape(self.bshape)
