"""Python binding of libjacobi.so (include/jacobi.h): argument marshalling only.

Every step of the Jacobi sweep runs in the library's sm_100a kernels.  There is no Python or CPU
fallback: if ``libjacobi.so`` is missing the import fails loudly, and without a CUDA device every
call returns JACOBI_ECUDA (raised as JacobiError).

Host inputs are numpy arrays; device inputs are torch CUDA tensors (PyTorch supplies device memory,
streams and process groups only).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# JACOBI_LIB=check loads the bounds-checked build (make lib-check) — same API, checks in the kernels;
# JACOBI_LIB=<path>.so loads a probe build of the same sources (e.g. -DJACOBI_SM_TIMING).
_LIBSEL = os.environ.get("JACOBI_LIB", "")
LIB_PATH = (os.path.join(_HERE, "libjacobi_check.so") if _LIBSEL == "check" else
            os.path.abspath(_LIBSEL) if _LIBSEL.endswith(".so") else os.path.join(_HERE, "libjacobi.so"))

CONVERGED, MAX_ITER = 0, 1
EINVAL, EZERODIAG, ENONFINITE, ENOMEM, ECUDA, ENCCL, EINDIVISIBLE = -1, -2, -3, -4, -5, -6, -7
F64, F32 = 0, 1
NORM_MAX, NORM_L2 = 0, 1
STATUS_NAMES = {0: "CONVERGED", 1: "MAX_ITER", -1: "EINVAL", -2: "EZERODIAG", -3: "ENONFINITE",
                -4: "ENOMEM", -5: "ECUDA", -6: "ENCCL", -7: "EINDIVISIBLE"}

# Every symbol include/jacobi.h declares (checked by tests/test_capi.py).
EXPORTS = ("jacobi_solve", "jacobi_solve_f32a", "jacobi_plan_create", "jacobi_plan_solve",
           "jacobi_plan_solve_device", "jacobi_plan_destroy", "jacobi_plan_set_row_blocks",
           "jacobi_plan_set_batch", "jacobi_plan_set_norm", "jacobi_plan_info", "jacobi_plan_time_sweeps",
           "jacobi_plan_time_shard", "jacobi_partition",
           "jacobi_nccl_unique_id", "jacobi_dist_plan_create", "jacobi_dist_plan_create_colwise",
           "jacobi_plan_set_col_blocks", "jacobi_plan_ipc_export", "jacobi_plan_ipc_attach",
           "jacobi_plan_set_p2p_emulation", "jacobi_bwprobe", "jacobi_last_error",
           "jacobi_version", "jacobi_variant_name", "jacobi_debug_bounds_check")


def bounds_violations(reset: bool = True):
    """(checked_build, mask) from jacobi_debug_bounds_check (libjacobi_check.so records violations)."""
    v = ctypes.c_ulonglong()
    checked = _lib.jacobi_debug_bounds_check(ctypes.byref(v), 1 if reset else 0)
    return bool(checked), int(v.value)


def variant_name(v: int) -> str:
    """Name of sweep-kernel variant v (csrc/sweep.cu kVariants; all bitwise identical)."""
    nm = _lib.jacobi_variant_name(int(v))
    return nm.decode() if nm else f"variant {v}"


class JacobiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class PlanInfo(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("lda", ctypes.c_int64), ("rows", ctypes.c_int64),
                ("row0", ctypes.c_int64), ("dtype", ctypes.c_int), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("chunk_cols", ctypes.c_int), ("rows_per_warp", ctypes.c_int),
                ("grid_ctas", ctypes.c_int), ("threads_per_cta", ctypes.c_int), ("a_borrowed", ctypes.c_int),
                ("sweeps_launched", ctypes.c_int64), ("bytes_per_sweep", ctypes.c_double),
                ("variant", ctypes.c_int), ("num_variants", ctypes.c_int), ("cluster_ctas", ctypes.c_int),
                ("persistent_ctas", ctypes.c_int), ("l2_keep_permille", ctypes.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
                          "there is no fallback implementation")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    P = ctypes.POINTER
    sig = {
        "jacobi_solve": ([i64, vp, vp, vp, i64, dbl, vp, P(i64)], i32),
        "jacobi_solve_f32a": ([i64, vp, vp, vp, i64, dbl, vp, P(i64)], i32),
        "jacobi_plan_create": ([P(vp), i64, i32, vp, i64, i32, vp], i32),
        "jacobi_plan_solve": ([vp, vp, vp, i64, dbl, vp, P(i64), vp], i32),
        "jacobi_plan_solve_device": ([vp, vp, vp, i64, dbl, vp, P(i64), vp], i32),
        "jacobi_plan_destroy": ([vp], None),
        "jacobi_plan_set_row_blocks": ([vp, i32], i32),
        "jacobi_plan_set_batch": ([vp, i32], i32),
        "jacobi_plan_set_norm": ([vp, i32], i32),
        "jacobi_plan_info": ([vp, P(PlanInfo)], i32),
        "jacobi_plan_time_sweeps": ([vp, vp, vp, i32, P(ctypes.c_float)], i32),
        "jacobi_plan_time_shard": ([vp, i32, i32, vp, vp, i32, i32, P(ctypes.c_float), P(i32)], i32),
        "jacobi_partition": ([i64, i32, i32, P(i64), P(i64)], i32),
        "jacobi_nccl_unique_id": ([vp], i32),
        "jacobi_dist_plan_create": ([P(vp), vp, i32, i32, i64, i32, vp, i64, i32, vp], i32),
        "jacobi_dist_plan_create_colwise": ([P(vp), vp, i32, i32, i64, i32, vp, i64, i32, vp], i32),
        "jacobi_plan_set_col_blocks": ([vp, i32], i32),
        "jacobi_plan_ipc_export": ([vp, vp], i32),
        "jacobi_plan_ipc_attach": ([vp, vp], i32),
        "jacobi_plan_set_p2p_emulation": ([vp, i32], i32),
        "jacobi_bwprobe": ([i64, i32, P(dbl)], i32),
        "jacobi_last_error": ([], ctypes.c_char_p),
        "jacobi_version": ([], i32),
        "jacobi_variant_name": ([i32], ctypes.c_char_p),
        "jacobi_debug_bounds_check": ([P(ctypes.c_ulonglong), i32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    return lib


_lib = _load()


def last_error() -> str:
    return _lib.jacobi_last_error().decode()


def _check(st):
    if st < 0:
        raise JacobiError(st, last_error())
    return st


def _host_f64(v, n, name):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (n,):
        raise ValueError(f"{name} must have shape ({n},), got {v.shape}")
    return v


def _is_torch_cuda(t):
    return type(t).__module__.startswith("torch") and getattr(t, "is_cuda", False)


def _dev_ptr(t, n, name, dtype_name="float64"):
    if not _is_torch_cuda(t):
        raise TypeError(f"{name} must be a torch CUDA tensor")
    if str(t.dtype) != f"torch.{dtype_name}" or not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name} must be a contiguous {dtype_name} CUDA tensor with {n} elements")
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class SolveResult:
    status: int
    x: object
    iters: int
    hist: object = None

    @property
    def converged(self):
        return self.status == CONVERGED


def solve(A, b, x0=None, max_iter=100, tol=0.0):
    """One-shot ``jacobi_solve`` / ``jacobi_solve_f32a`` on host (numpy) arrays."""
    A = np.asarray(A)
    n = A.shape[0]
    if A.ndim != 2 or A.shape[1] != n:
        raise ValueError("A must be square")
    f32 = A.dtype == np.float32
    A = np.ascontiguousarray(A, dtype=np.float32 if f32 else np.float64)
    b = _host_f64(b, n, "b")
    x0 = np.zeros(n) if x0 is None else _host_f64(x0, n, "x0")
    x = np.empty(n)
    it = ctypes.c_int64(-1)
    fn = _lib.jacobi_solve_f32a if f32 else _lib.jacobi_solve
    st = _check(fn(n, A.ctypes.data, b.ctypes.data, x0.ctypes.data, int(max_iter), float(tol), x.ctypes.data,
                   ctypes.byref(it)))
    return SolveResult(st, x, it.value)


class Plan:
    """A resident system (``jacobi_plan_create`` / ``jacobi_dist_plan_create``).

    A: numpy array (host; copied) or torch CUDA tensor (device; borrowed, must outlive the plan).
    For a distributed plan pass ``dist=(uid_bytes, rank, nranks)`` and A = this rank's row block
    (``layout="rows"``, §3.1) or its n x m column slab (``layout="cols"``, §3.2)."""

    def __init__(self, A, n=None, lda=None, stream=None, dist=None, layout="rows"):
        on_dev = _is_torch_cuda(A)
        if on_dev:
            dt = str(A.dtype)
            if dt not in ("torch.float64", "torch.float32") or A.dim() != 2 or A.stride(1) != 1:
                raise ValueError("device A must be a 2-D row-major float64/float32 CUDA tensor")
            self.dtype = F32 if dt == "torch.float32" else F64
            rows, cols = A.shape
            lda = A.stride(0) if lda is None else lda
            ptr = A.data_ptr()
        else:
            A = np.asarray(A)
            self.dtype = F32 if A.dtype == np.float32 else F64
            A = np.ascontiguousarray(A, dtype=np.float32 if self.dtype == F32 else np.float64)
            rows, cols = A.shape
            lda = cols if lda is None else lda
            ptr = A.ctypes.data
        self.n = int(n if n is not None else cols)
        self._A_ref = A  # keep the host/device buffer alive for the plan's lifetime
        h = ctypes.c_void_p()
        s = ctypes.c_void_p(stream if stream is not None else 0)
        if dist is None:
            _check(_lib.jacobi_plan_create(ctypes.byref(h), self.n, self.dtype, ctypes.c_void_p(ptr), lda,
                                           int(on_dev), s))
        else:
            uid, rank, nranks = dist
            ub = ctypes.create_string_buffer(bytes(uid), 128)
            create = {"rows": _lib.jacobi_dist_plan_create, "cols": _lib.jacobi_dist_plan_create_colwise}[layout]
            _check(create(ctypes.byref(h), ub, int(rank), int(nranks), self.n, self.dtype, ctypes.c_void_p(ptr), lda,
                          int(on_dev), s))
        self._h = h
        self._rows = self.info.rows  # rows this plan owns (b's length); fixed for the plan's life

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.jacobi_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def info(self) -> PlanInfo:
        inf = PlanInfo()
        _check(_lib.jacobi_plan_info(self._h, ctypes.byref(inf)))
        return inf

    def set_row_blocks(self, nblocks):
        _check(_lib.jacobi_plan_set_row_blocks(self._h, int(nblocks)))

    def set_p2p_emulation(self, nranks):
        _check(_lib.jacobi_plan_set_p2p_emulation(self._h, int(nranks)))

    def ipc_export(self) -> bytes:
        buf = ctypes.create_string_buffer(256)
        _check(_lib.jacobi_plan_ipc_export(self._h, buf))
        return buf.raw

    def ipc_attach(self, all_handles: bytes):
        buf = ctypes.create_string_buffer(bytes(all_handles), len(all_handles))
        _check(_lib.jacobi_plan_ipc_attach(self._h, buf))

    def set_col_blocks(self, nblocks):
        _check(_lib.jacobi_plan_set_col_blocks(self._h, int(nblocks)))

    def set_norm(self, norm):
        """'max' (north_star, default) or 'l2' (the paper's Euclidean distance)."""
        _check(_lib.jacobi_plan_set_norm(self._h, {"max": NORM_MAX, "l2": NORM_L2}.get(norm, -1)))

    def set_batch(self, k):
        _check(_lib.jacobi_plan_set_batch(self._h, int(k)))

    def solve(self, b, x0=None, max_iter=100, tol=0.0, history=False):
        """Host-pointer solve.  b: this plan's rows; x0/x: length n (numpy)."""
        b = _host_f64(b, self._rows, "b")
        x0 = np.zeros(self.n) if x0 is None else _host_f64(x0, self.n, "x0")
        x = np.empty(self.n)
        it = ctypes.c_int64(-1)
        hist = np.empty(max(int(max_iter), 1)) if history else None
        st = _check(_lib.jacobi_plan_solve(self._h, b.ctypes.data, x0.ctypes.data, int(max_iter), float(tol),
                                           x.ctypes.data, ctypes.byref(it), hist.ctypes.data if history else None))
        return SolveResult(st, x, it.value, hist[: it.value] if history else None)

    def solve_device(self, b, x0, x_out, max_iter=100, tol=0.0, hist=None):
        """Device-pointer solve on torch CUDA tensors (results written into x_out / hist).  hist
        (optional) needs max(max_iter, 1) float64 elements: the kernels write d_k into it while the
        solve runs (jacobi.h), so a short tensor would be written past its end."""
        if hist is not None and (not _is_torch_cuda(hist) or hist.numel() < max(int(max_iter), 1)):
            raise ValueError(f"hist must be a CUDA tensor with at least max(max_iter, 1) = {max(int(max_iter), 1)} "
                             "elements")
        it = ctypes.c_int64(-1)
        st = _check(_lib.jacobi_plan_solve_device(
            self._h, _dev_ptr(b, self._rows, "b"), _dev_ptr(x0, self.n, "x0"), int(max_iter), float(tol),
            _dev_ptr(x_out, self.n, "x_out"), ctypes.byref(it),
            _dev_ptr(hist, hist.numel(), "hist") if hist is not None else None))
        return SolveResult(st, x_out, it.value, hist)

    def time_sweeps(self, b, x0, sweeps):
        inf = self.info
        ms = (ctypes.c_float * sweeps)()
        _check(_lib.jacobi_plan_time_sweeps(self._h, _dev_ptr(b, inf.rows, "b"), _dev_ptr(x0, self.n, "x0"),
                                            int(sweeps), ms))
        return np.array(ms[:], dtype=np.float64)


    def time_shard(self, b, x0, nranks, rank=0, sweeps=20, mode="graph"):
        """jacobi_plan_time_shard: ms per sweep of rank `rank`'s row block of an nranks-rank plan, on this
        GPU, exchange excluded.  mode: "graph", "persistent", "persistent-push" or "colslab" (rank `rank`'s
        column slab of a column-wise plan, NEXT-4).  Returns (ms, variant)."""
        ms = ctypes.c_float()
        v = ctypes.c_int()
        m = {"graph": 0, "persistent": 1, "persistent-push": 2, "colslab": 3}[mode]
        _check(_lib.jacobi_plan_time_shard(self._h, int(nranks), int(rank), _dev_ptr(b, self.n, "b"),
                                           _dev_ptr(x0, self.n, "x0"), int(sweeps), m, ctypes.byref(ms),
                                           ctypes.byref(v)))
        return float(ms.value), int(v.value)


def partition(n, nranks, rank):
    r0, m = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.jacobi_partition(int(n), int(nranks), int(rank), ctypes.byref(r0), ctypes.byref(m)))
    return r0.value, m.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.jacobi_nccl_unique_id(buf))
    return buf.raw


def bwprobe(nbytes=32 << 30, reps=5):
    g = ctypes.c_double()
    _check(_lib.jacobi_bwprobe(int(nbytes), int(reps), ctypes.byref(g)))
    return g.value


def version():
    return _lib.jacobi_version()
