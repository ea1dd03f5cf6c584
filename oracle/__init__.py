"""CPU oracle for the dense Jacobi sweep — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path (``paper_1403_5805_b200``) never
imports it and shares no code with it.  The arithmetic lives in ``oracle.c`` (plain C, fp64,
ascending-j sums, no FMA contraction), which cites the paper passage each step follows
(PAPER.md:55 component equation, PAPER.md:59-66 pseudocode, PAPER.md:53 a_ii != 0).

Parity unpinned: none of the functions below (every one is pinned in tests/test_oracle_pins.py).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

CONVERGED, MAX_ITER = 0, 1
EINVAL, EZERODIAG, ENONFINITE, ENOMEM = -1, -2, -3, -4

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make oracle` (or __graft_entry__.build())")
        lib = ctypes.CDLL(_LIB_PATH)
        i64, dp, vp = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
        lib.oracle_jacobi.argtypes = [i64, ctypes.c_int, vp, i64, dp, dp, i64, ctypes.c_double, dp,
                                      ctypes.POINTER(i64), dp, ctypes.c_int]
        lib.oracle_jacobi.restype = ctypes.c_int
        lib.oracle_sweep_rows.argtypes = [i64, ctypes.c_int, vp, i64, i64, i64, dp, dp, dp]
        lib.oracle_sweep_rows.restype = None
        lib.oracle_jacobi_norm.argtypes = lib.oracle_jacobi.argtypes + [ctypes.c_int]
        lib.oracle_jacobi_norm.restype = ctypes.c_int
        lib.oracle_l2_dist.argtypes = [i64, dp, dp]
        lib.oracle_l2_dist.restype = ctypes.c_double
        lib.oracle_maxnorm_dist.argtypes = [i64, dp, dp]
        lib.oracle_maxnorm_dist.restype = ctypes.c_double
        lib.oracle_ge_solve.argtypes = [i64, dp, dp, dp]
        lib.oracle_ge_solve.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64vec(v, n, name):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (n,):
        raise ValueError(f"{name} must have shape ({n},), got {v.shape}")
    return v


def jacobi(A, b, x0=None, max_iter=100, tol=0.0, nthreads=1, history=False, norm="max"):
    """PAPER.md:59-66 with the max-norm distance (norm="max", north_star) or the paper's Euclidean
    distance of PAPER.md:94 (norm="l2").  A: (n, n) float64 or float32 (fp32 values are widened
    exactly).  Returns (status, x, iters[, hist]); x is None when status < 0."""
    A = np.asarray(A)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("A must be square")
    n = A.shape[0]
    a_f32 = 1 if A.dtype == np.float32 else 0
    A = np.ascontiguousarray(A, dtype=np.float32 if a_f32 else np.float64)
    b = _f64vec(b, n, "b")
    x0 = np.zeros(n) if x0 is None else _f64vec(x0, n, "x0")
    x = np.empty(n)
    it = ctypes.c_int64(-1)
    hist = np.full(max(int(max_iter), 1), np.nan) if history else None
    st = _load().oracle_jacobi_norm(n, a_f32, A.ctypes.data, n, _dp(b), _dp(x0), int(max_iter), float(tol),
                                    _dp(x), ctypes.byref(it), _dp(hist) if history else None, int(nthreads),
                                    {"max": 0, "l2": 1}[norm])
    out = (st, x if st >= 0 else None, it.value if st >= 0 else None)
    if history:
        out = out + ((hist[: it.value] if st >= 0 else None),)
    return out


def sweep_rows(A_rows, r0, b_rows, x_old):
    """One application of PAPER.md:55 to rows r0 .. r0+len(A_rows)-1 (A_rows: their full rows)."""
    A_rows = np.asarray(A_rows)
    a_f32 = 1 if A_rows.dtype == np.float32 else 0
    A_rows = np.ascontiguousarray(A_rows, dtype=np.float32 if a_f32 else np.float64)
    rows, n = A_rows.shape
    b_rows = _f64vec(b_rows, rows, "b_rows")
    x_old = _f64vec(x_old, n, "x_old")
    out = np.empty(rows)
    _load().oracle_sweep_rows(n, a_f32, A_rows.ctypes.data, n, int(r0), int(r0) + rows, _dp(b_rows),
                              _dp(x_old), _dp(out))
    return out


def maxnorm_dist(u, v):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    return _load().oracle_maxnorm_dist(u.shape[0], _dp(u), _dp(v))


def l2_dist(u, v):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    return _load().oracle_l2_dist(u.shape[0], _dp(u), _dp(v))


def ge_solve(A, b):
    """Gaussian elimination with partial pivoting (fp64).  Returns x or raises on singular A."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    b = _f64vec(b, n, "b")
    x = np.empty(n)
    st = _load().oracle_ge_solve(n, _dp(A), _dp(b), _dp(x))
    if st != 0:
        raise np.linalg.LinAlgError(f"oracle_ge_solve status {st}")
    return x
