"""CPU oracle for the restricted-domain dual iteration (arXiv 1807.11534) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1807_11534_b200``) never imports it; the two share no code (only the seeded input
generators in ``paper_1807_11534_b200/workloads.py``, which hold none of the method's
arithmetic).

The arithmetic lives in ``oracle.c`` (plain C, float64 iteration, float32 fitting/band test);
this module is argument marshalling via ctypes plus a small set of pure-numpy reference
helpers that restate the paper's definitions for tiny cases.  See ``oracle.c`` for the
PAPER.md citations of every function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

LAB_BG, LAB_FG, LAB_RD = 0, 1, 2
NTRACE = 5  # must match ORC_NTRACE in oracle.c (checked at load)

GCC_FLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-Wall"]


def _src_hash() -> str:
    import hashlib

    with open(_SRC, "rb") as fh:
        return hashlib.sha256(fh.read() + " ".join(GCC_FLAGS).encode()).hexdigest()


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no contraction, no fast-math); rebuilt whenever the
    content hash of oracle.c and the flags differs from the one recorded beside it."""
    stamp = _LIB_PATH + ".srchash"
    h = _src_hash()
    stale = not os.path.exists(_LIB_PATH) or not os.path.exists(stamp) or \
        open(stamp).read().strip() != h
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
        with open(stamp, "w") as fh:
            fh.write(h)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        d = ctypes.c_double
        f = ctypes.c_float
        i = ctypes.c_int
        lib.orc_set_threads.argtypes = [i]
        lib.orc_get_threads.restype = i
        lib.orc_fitting.argtypes = [P, P, i64, f, f, f, P]
        lib.orc_absmax.argtypes = [P, i64]
        lib.orc_absmax.restype = f
        lib.orc_labels.argtypes = [P, i64, f, P]
        lib.orc_tiles.argtypes = [P, i64, i64, i, i, P]
        lib.orc_tiles.restype = i64
        lib.orc_grad.argtypes = [P, i64, i64, P, P]
        lib.orc_div.argtypes = [P, P, i64, i64, P]
        lib.orc_tv.argtypes = [P, i64, i64]
        lib.orc_tv.restype = d
        lib.orc_energy.argtypes = [P, i64, i64, d, P, P, P, P, P]
        lib.orc_solve.argtypes = [P, i64, i64, f, d, d, d, i, i, P, P, P, P, P, P, P, P, P]
        lib.orc_solve.restype = i
        lib.orc_solve_tol.argtypes = [P, i64, i64, f, d, d, d, i, i, d, i, P, P, P, P, P,
                                      ctypes.POINTER(i), ctypes.POINTER(d)]
        lib.orc_solve_tol.restype = i
        lib.orc_solve_plain.argtypes = [P, i64, i64, d, d, d, i, P, P, P, P]
        lib.orc_solve_plain.restype = i
        lib.orc_grad3.argtypes = [P, i64, i64, i64, P, P, P]
        lib.orc_div3.argtypes = [P, P, P, i64, i64, i64, P]
        lib.orc_solve3.argtypes = [P, i64, i64, i64, f, d, d, d, i, P, P, P, P, P, P]
        lib.orc_solve3.restype = i
        lib.orc_solve3_plain.argtypes = [P, i64, i64, i64, d, d, d, i, P, P, P, P, P]
        lib.orc_solve3_plain.restype = i
        lib.orc_inner.argtypes = [P, i64, i64, f, d, d, i, P, P, P, P]
        lib.orc_inner.restype = i
        lib.orc_band_for_fraction.argtypes = [P, i64, d]
        lib.orc_band_for_fraction.restype = f
        lib.orc_ntrace.restype = i
        lib.orc_last_loop_seconds.restype = d
        assert lib.orc_ntrace() == NTRACE
        _lib = lib
        return lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    _load().orc_set_threads(int(n))


def get_threads() -> int:
    return int(_load().orc_get_threads())


def last_loop_seconds() -> float:
    """Wall time of the last solve's K-loop alone (no labels, initialisation or copies)."""
    return float(_load().orc_last_loop_seconds())


# ---------------------------------------------------------------------------------------------
# A1 / A2
# ---------------------------------------------------------------------------------------------

def fitting(z, c1, c2, gamma=0.0, P=None):
    """f = (z-c1)^2 - (z-c2)^2 (+ gamma P), float32 with fixed op order."""
    z = _f32(z)
    if gamma != 0.0 and P is None:
        raise ValueError("P required when gamma != 0")
    Pa = _f32(P) if P is not None else None
    out = np.empty_like(z)
    _load().orc_fitting(_ptr(z), _ptr(Pa), z.size, np.float32(c1), np.float32(c2),
                        np.float32(gamma), _ptr(out))
    return out


def absmax(f) -> np.float32:
    f = _f32(f)
    return np.float32(_load().orc_absmax(_ptr(f), f.size))


def labels(f, delta):
    """0=BG, 1=FG, 2=RD (RD <=> |f| < delta)."""
    f = _f32(f)
    out = np.empty(f.shape, dtype=np.uint8)
    _load().orc_labels(_ptr(f), f.size, np.float32(delta), _ptr(out))
    return out


def band_for_fraction(f, q) -> np.float32:
    """q -> q^: smallest float32 q^ with #{|f| < q^} >= ceil(q N)."""
    f = _f32(f)
    return np.float32(_load().orc_band_for_fraction(_ptr(f), f.size, float(q)))


def tiles(lab, th=32, tw=32):
    """Ascending list of active tile indices t = ti*ceil(W/tw)+tj."""
    lab = np.ascontiguousarray(lab, dtype=np.uint8)
    H, W = lab.shape
    nt = ((H + th - 1) // th) * ((W + tw - 1) // tw)
    out = np.empty(max(nt, 1), dtype=np.int32)
    cnt = _load().orc_tiles(_ptr(lab), H, W, th, tw, _ptr(out))
    return out[:cnt].copy()


# ---------------------------------------------------------------------------------------------
# operators / energies
# ---------------------------------------------------------------------------------------------

def grad(u):
    u = _f64(u)
    H, W = u.shape
    g1 = np.empty_like(u)
    g2 = np.empty_like(u)
    _load().orc_grad(_ptr(u), H, W, _ptr(g1), _ptr(g2))
    return g1, g2


def div(p1, p2):
    p1 = _f64(p1)
    p2 = _f64(p2)
    H, W = p1.shape
    d = np.empty_like(p1)
    _load().orc_div(_ptr(p1), _ptr(p2), H, W, _ptr(d))
    return d


def tv(u) -> float:
    u = _f64(u)
    H, W = u.shape
    return float(_load().orc_tv(_ptr(u), H, W))


ENERGY_KEYS = ("E_v", "E_u", "D_p", "gap", "TV_v", "fit_v")


def energy(f, lam, u, v, p1, p2) -> dict:
    f = _f32(f)
    H, W = f.shape
    u, v, p1, p2 = (_f64(a) for a in (u, v, p1, p2))
    out = np.empty(6, dtype=np.float64)
    _load().orc_energy(_ptr(f), H, W, float(lam), _ptr(u), _ptr(v), _ptr(p1), _ptr(p2),
                       _ptr(out))
    return dict(zip(ENERGY_KEYS, out.tolist()))


# ---------------------------------------------------------------------------------------------
# the iteration
# ---------------------------------------------------------------------------------------------

def solve(f, delta, lam, theta, tau, iters, inner_steps=1, init=None, trace=False):
    """Restricted-domain dual iteration (oracle.c orc_solve).  ``init`` = (v, p1, p2) warm
    start or None.  Returns dict u, v, p1, p2, labels (+ trace [iters x NTRACE])."""
    f = _f32(f)
    H, W = f.shape
    u = np.empty((H, W), dtype=np.float64)
    v = np.empty_like(u)
    p1 = np.empty_like(u)
    p2 = np.empty_like(u)
    lab = np.empty((H, W), dtype=np.uint8)
    vi = p1i = p2i = None
    if init is not None:
        vi, p1i, p2i = (_f64(a) for a in init)
    tr = np.empty((max(iters, 1), NTRACE), dtype=np.float64) if trace else None
    rc = _load().orc_solve(_ptr(f), H, W, np.float32(delta), float(lam), float(theta),
                           float(tau), int(iters), int(inner_steps), _ptr(vi), _ptr(p1i),
                           _ptr(p2i), _ptr(u), _ptr(v), _ptr(p1), _ptr(p2), _ptr(lab),
                           _ptr(tr))
    if rc != 0:
        raise ValueError(f"orc_solve rc={rc}")
    out = dict(u=u, v=v, p1=p1, p2=p2, labels=lab)
    if trace:
        out["trace"] = tr[:iters]
    return out


def solve_tol(f, delta, lam, theta, tau, max_iters, tol, check_every, norm="l2"):
    """The iteration with the paper's stopping rule (oracle.c orc_solve_tol):
    checks after every check_every iterations and at max_iters; norm "l2" (Euclidean over
    pixels of unit area, reading R-F2) or "rms".  Returns dict u, v, p1, p2, labels, iters,
    residual."""
    f = _f32(f)
    H, W = f.shape
    u = np.empty((H, W), dtype=np.float64)
    v = np.empty_like(u)
    p1 = np.empty_like(u)
    p2 = np.empty_like(u)
    lab = np.empty((H, W), dtype=np.uint8)
    it = ctypes.c_int()
    res = ctypes.c_double()
    rc = _load().orc_solve_tol(_ptr(f), H, W, np.float32(delta), float(lam), float(theta),
                               float(tau), int(max_iters), int(check_every), float(tol),
                               {"l2": 0, "rms": 1}[norm], _ptr(u),
                               _ptr(v), _ptr(p1), _ptr(p2), _ptr(lab), ctypes.byref(it),
                               ctypes.byref(res))
    if rc != 0:
        raise ValueError(f"orc_solve_tol rc={rc}")
    return dict(u=u, v=v, p1=p1, p2=p2, labels=lab, iters=it.value, residual=res.value)


# ------------------------------------------------------------------------------------------
# f4: 3-D volumes (oracle.c orc_*3, reading R-F4).  Arrays are (D, H, W).
# ------------------------------------------------------------------------------------------

def grad3(u):
    u = _f64(u)
    D, H, W = u.shape
    g = [np.empty_like(u) for _ in range(3)]
    _load().orc_grad3(_ptr(u), D, H, W, _ptr(g[0]), _ptr(g[1]), _ptr(g[2]))
    return tuple(g)


def div3(p1, p2, p3):
    p1, p2, p3 = _f64(p1), _f64(p2), _f64(p3)
    D, H, W = p1.shape
    d = np.empty_like(p1)
    _load().orc_div3(_ptr(p1), _ptr(p2), _ptr(p3), D, H, W, _ptr(d))
    return d


def solve3(f, delta, lam, theta, tau, iters):
    """Restricted-domain iteration on a volume f (D, H, W) float32: dict u, v, p1, p2, p3,
    labels."""
    f = _f32(f)
    D, H, W = f.shape
    out = {k: np.empty((D, H, W), np.float64) for k in ("u", "v", "p1", "p2", "p3")}
    lab = np.empty((D, H, W), np.uint8)
    rc = _load().orc_solve3(_ptr(f), D, H, W, np.float32(delta), float(lam), float(theta),
                            float(tau), int(iters), _ptr(out["u"]), _ptr(out["v"]),
                            _ptr(out["p1"]), _ptr(out["p2"]), _ptr(out["p3"]), _ptr(lab))
    if rc != 0:
        raise ValueError(f"orc_solve3 rc={rc}")
    out["labels"] = lab
    return out


def solve3_plain(f, lam, theta, tau, iters):
    f = _f32(f)
    D, H, W = f.shape
    out = {k: np.empty((D, H, W), np.float64) for k in ("u", "v", "p1", "p2", "p3")}
    rc = _load().orc_solve3_plain(_ptr(f), D, H, W, float(lam), float(theta), float(tau),
                                  int(iters), _ptr(out["u"]), _ptr(out["v"]), _ptr(out["p1"]),
                                  _ptr(out["p2"]), _ptr(out["p3"]))
    if rc != 0:
        raise ValueError(f"orc_solve3_plain rc={rc}")
    return out


def tanimoto(a, b):
    """E1 of PAPER.md:247 (Tanimoto coefficient of two thresholded results): N(a n b) /
    N(a u b) over pixels ("number of nodes"); 1 when both sets are empty (reading R-C15)."""
    a = np.asarray(a, bool)
    b = np.asarray(b, bool)
    union = int(np.count_nonzero(a | b))
    return 1.0 if union == 0 else int(np.count_nonzero(a & b)) / union


def l2_error(u, ugt):
    """E2 of PAPER.md:247, the integral of (u* - u^GT)^2 over Omega with unit pixel area
    (reading R-C15)."""
    d = np.asarray(u, np.float64) - np.asarray(ugt, np.float64)
    return float(np.sum(d * d))


def solve_plain(f, lam, theta, tau, iters):
    """Unrestricted Bresson/Chambolle iteration, independent loops."""
    f = _f32(f)
    H, W = f.shape
    u = np.empty((H, W), dtype=np.float64)
    v = np.empty_like(u)
    p1 = np.empty_like(u)
    p2 = np.empty_like(u)
    rc = _load().orc_solve_plain(_ptr(f), H, W, float(lam), float(theta), float(tau),
                                 int(iters), _ptr(u), _ptr(v), _ptr(p1), _ptr(p2))
    if rc != 0:
        raise ValueError(f"orc_solve_plain rc={rc}")
    return dict(u=u, v=v, p1=p1, p2=p2)


def inner(f, delta, theta, tau, steps, v, p1=None, p2=None):
    """Chambolle inner iteration with v fixed; returns (p1, p2, obj[steps])."""
    f = _f32(f)
    H, W = f.shape
    v = _f64(v)
    p1 = np.zeros((H, W)) if p1 is None else _f64(p1).copy()
    p2 = np.zeros((H, W)) if p2 is None else _f64(p2).copy()
    obj = np.empty(steps, dtype=np.float64)
    _load().orc_inner(_ptr(f), H, W, np.float32(delta), float(theta), float(tau), int(steps),
                      _ptr(v), _ptr(p1), _ptr(p2), _ptr(obj))
    return p1, p2, obj


def mask(u, eps=0.5):
    """Threshold GT(x) = [u(x) > eps] (strict, eps = 0.5)."""
    return (np.asarray(u) > eps).astype(np.uint8)
