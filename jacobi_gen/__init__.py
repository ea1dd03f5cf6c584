"""Seeded synthetic linear systems (input generator shared by the oracle and the CUDA path).

Holds none of the Jacobi method's arithmetic: it only builds A, b = A x* and x* as described in
``jacobi_gen.h`` and DESIGN.md §4 (input recipe).  Host functions work without a GPU; the device
twin writes bitwise-identical values straight into HBM (needed for configs whose A is 34-69 GB).

Configs (BASELINE.json ``configs``, all seed 0, x0 = 0):
  c1  n=256    fp64  diag = rowabs + U[1,2]
  c2  n=4096   fp64  diag = rowabs + U[1,2]
  c3  n=16384  fp64  diag = 1.05 * rowabs
  c4  n=65536  fp64  diag = rowabs + U[1,2]     (headline)
  c5  n=131072 fp32  diag = 1.2 * rowabs
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libjacobigen.so")

F64, F32 = 0, 1
DIAG_ADD, DIAG_SCALE = 0, 1


class _Cfg(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("seed", ctypes.c_uint64), ("a_dtype", ctypes.c_int),
                ("diag_mode", ctypes.c_int), ("diag_scale", ctypes.c_double)]


@dataclass(frozen=True)
class GenConfig:
    n: int
    seed: int = 0
    a_dtype: int = F64
    diag_mode: int = DIAG_ADD
    diag_scale: float = 0.0

    def c(self):
        return _Cfg(self.n, self.seed, self.a_dtype, self.diag_mode, self.diag_scale)

    @property
    def np_dtype(self):
        return np.float32 if self.a_dtype == F32 else np.float64


CONFIGS = {
    "c1": GenConfig(256),
    "c2": GenConfig(4096),
    "c3": GenConfig(16384, diag_mode=DIAG_SCALE, diag_scale=1.05),
    "c4": GenConfig(65536),
    "c5": GenConfig(131072, a_dtype=F32, diag_mode=DIAG_SCALE, diag_scale=1.2),
}

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make gen` (or __graft_entry__.build())")
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        i64, dp, vp = ctypes.c_int64, P(ctypes.c_double), ctypes.c_void_p
        lib.jgen_host_rows.argtypes = [P(_Cfg), i64, i64, vp, i64, dp, ctypes.c_int]
        lib.jgen_host_xstar.argtypes = [P(_Cfg), dp]
        lib.jgen_host_diag_b.argtypes = [P(_Cfg), i64, i64, dp, dp, ctypes.c_int]
        lib.jgen_device_rows.argtypes = [P(_Cfg), i64, i64, vp, i64, vp, vp]
        lib.jgen_device_xstar.argtypes = [P(_Cfg), vp, vp]
        for f in ("jgen_host_rows", "jgen_host_xstar", "jgen_host_diag_b", "jgen_device_rows",
                  "jgen_device_xstar"):
            getattr(lib, f).restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _threads():
    return max(1, len(os.sched_getaffinity(0)))


def host_rows(cfg: GenConfig, r0: int, r1: int, lda: int | None = None, nthreads: int | None = None,
              out: np.ndarray | None = None):
    """Rows [r0, r1) of A (shape (r1-r0, lda)) and the matching slice of b."""
    lda = cfg.n if lda is None else lda
    A = out if out is not None else np.empty((r1 - r0, lda), dtype=cfg.np_dtype)
    assert A.flags.c_contiguous and A.dtype == cfg.np_dtype and A.shape == (r1 - r0, lda)
    b = np.empty(r1 - r0)
    c = cfg.c()
    st = _load().jgen_host_rows(ctypes.byref(c), r0, r1, A.ctypes.data, lda, _dp(b), nthreads or _threads())
    if st != 0:
        raise ValueError(f"jgen_host_rows failed ({st})")
    return A, b


def host_xstar(cfg: GenConfig):
    xs = np.empty(cfg.n)
    c = cfg.c()
    if _load().jgen_host_xstar(ctypes.byref(c), _dp(xs)) != 0:
        raise ValueError("jgen_host_xstar failed")
    return xs


def host_diag_b(cfg: GenConfig, r0: int, r1: int, nthreads: int | None = None):
    d = np.empty(r1 - r0)
    b = np.empty(r1 - r0)
    c = cfg.c()
    if _load().jgen_host_diag_b(ctypes.byref(c), r0, r1, _dp(d), _dp(b), nthreads or _threads()) != 0:
        raise ValueError("jgen_host_diag_b failed")
    return d, b


def host_system(cfg: GenConfig, nthreads: int | None = None):
    """(A, b, x*) for the whole system (only for sizes that fit host RAM)."""
    A, b = host_rows(cfg, 0, cfg.n, nthreads=nthreads)
    return A, b, host_xstar(cfg)


def device_rows(cfg: GenConfig, r0: int, r1: int, A_ptr: int, lda: int, b_ptr: int | None, stream: int = 0):
    """Enqueue the device twin: rows [r0, r1) into device memory at A_ptr (lda elements per row)."""
    c = cfg.c()
    st = _load().jgen_device_rows(ctypes.byref(c), r0, r1, ctypes.c_void_p(A_ptr), lda,
                                  ctypes.c_void_p(b_ptr) if b_ptr else None, ctypes.c_void_p(stream))
    if st != 0:
        raise RuntimeError(f"jgen_device_rows failed ({st})")


def device_xstar(cfg: GenConfig, ptr: int, stream: int = 0):
    c = cfg.c()
    if _load().jgen_device_xstar(ctypes.byref(c), ctypes.c_void_p(ptr), ctypes.c_void_p(stream)) != 0:
        raise RuntimeError("jgen_device_xstar failed")


def slow_companion(n: int, seed: int, f32: bool = False):
    """(A, b, x*) of c3's truly slow companion (R21; a parity case, not a
    BASELINE.json config): off-diagonals U[0,1) — the paper's own distribution, PAPER.md:154 — and
    a_ii = 1.05 x the row sum, so T = -D^-1(L+U) has rho(T) = 1/1.05 (~360-380 sweeps to 1e-10).
    numpy's seeded generator on the host (sizes that fit host RAM); b = A x* over the stored values."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(0, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, 1.05 * A.sum(1))
    if f32:
        A = A.astype(np.float32)
    xs = rng.uniform(-1, 1, n)
    return A, A.astype(np.float64) @ xs, xs
