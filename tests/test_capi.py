"""C-ABI library checks that need no GPU: it loads, exports every symbol include/jacobi.h declares,
validates arguments before touching CUDA, partitions rows, and has no CPU fallback."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "jacobi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(jacobi_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def jb():
    import subprocess
    so = os.path.join(ROOT, "paper_1403_5805_b200", "libjacobi.so")
    if not os.path.exists(so):
        r = subprocess.run(["make", "-C", ROOT, "lib"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
    import paper_1403_5805_b200 as jb
    return jb


def test_exports_every_header_symbol(jb):
    names = _header_functions()
    assert len(names) >= 16
    lib = ctypes.CDLL(jb.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), f"libjacobi.so does not export {name}"
    assert set(names) == set(jb.EXPORTS)
    assert jb.version() == 100


def test_einval_before_any_cuda_call(jb):
    lib = jb._lib
    x = np.zeros(4)
    it = ctypes.c_int64(-7)
    A = np.eye(4)
    # n < 1, NULL pointers, max_iter < 0, tol < 0 / NaN
    assert lib.jacobi_solve(0, A.ctypes.data, x.ctypes.data, x.ctypes.data, 5, 0.0, x.ctypes.data, ctypes.byref(it)) == jb.EINVAL
    assert lib.jacobi_solve(4, None, x.ctypes.data, x.ctypes.data, 5, 0.0, x.ctypes.data, ctypes.byref(it)) == jb.EINVAL
    assert lib.jacobi_solve(4, A.ctypes.data, x.ctypes.data, x.ctypes.data, -1, 0.0, x.ctypes.data, ctypes.byref(it)) == jb.EINVAL
    assert lib.jacobi_solve(4, A.ctypes.data, x.ctypes.data, x.ctypes.data, 5, -1.0, x.ctypes.data, ctypes.byref(it)) == jb.EINVAL
    assert lib.jacobi_solve(4, A.ctypes.data, x.ctypes.data, x.ctypes.data, 5, float("nan"), x.ctypes.data, ctypes.byref(it)) == jb.EINVAL
    assert it.value == -7  # outputs untouched on error
    assert "bad argument" in jb.last_error()
    h = ctypes.c_void_p()
    assert lib.jacobi_plan_create(ctypes.byref(h), 4, 7, A.ctypes.data, 4, 0, None) == jb.EINVAL
    assert lib.jacobi_plan_create(ctypes.byref(h), 4, 0, A.ctypes.data, 3, 0, None) == jb.EINVAL
    assert lib.jacobi_plan_solve(None, x.ctypes.data, x.ctypes.data, 5, 0.0, x.ctypes.data, ctypes.byref(it), None) == jb.EINVAL
    with pytest.raises(jb.JacobiError) as e:
        jb.solve(np.eye(3), np.ones(3), max_iter=-2)
    assert e.value.status == jb.EINVAL


def test_partition(jb):
    assert jb.partition(8, 2, 0) == (0, 4) and jb.partition(8, 2, 1) == (4, 4)
    assert jb.partition(8, 8, 5) == (5, 1)
    with pytest.raises(jb.JacobiError) as e:
        jb.partition(8, 3, 0)
    assert e.value.status == jb.EINDIVISIBLE
    for n in (1, 12, 96, 1024):
        for p in [d for d in range(1, 17) if n % d == 0]:
            cover = []
            for r in range(p):
                r0, m = jb.partition(n, p, r)
                cover.extend(range(r0, r0 + m))
            assert cover == list(range(n))


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU path")
def test_no_cpu_fallback_without_gpu(jb):
    with pytest.raises(jb.JacobiError) as e:
        jb.solve(np.array([[2.0, 1.0], [1.0, 3.0]]), np.array([3.0, 4.0]), max_iter=5)
    assert e.value.status == jb.ECUDA


def test_variant_names_without_gpu(jb):
    """jacobi_variant_name is pure host code: names for the compiled variants, NULL past the end."""
    names = [jb.variant_name(v) for v in range(64)]
    assert names[0].startswith("k_sweep") and names[3] == "k_sweep_cta R4 U1"
    known = [n for n in names if not n.startswith("variant ")]
    assert len(known) == 14 and len(set(known)) == len(known)
    assert jb._lib.jacobi_variant_name(-1) is None and jb._lib.jacobi_variant_name(10**6) is None


def test_bounds_checked_build_exports_the_same_abi(jb):
    """libjacobi_check.so (make lib-check) is the same C-ABI with device-side bounds checks: it exports
    every header symbol and reports itself as checked; the release library reports 0 (checks compiled out)."""
    import subprocess
    so = os.path.join(ROOT, "paper_1403_5805_b200", "libjacobi_check.so")
    if not os.path.exists(so):
        r = subprocess.run(["make", "-C", ROOT, "lib-check"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
    chk = ctypes.CDLL(so)
    for name in _header_functions():
        assert hasattr(chk, name), name
    v = ctypes.c_ulonglong(7)
    assert jb._lib.jacobi_debug_bounds_check(ctypes.byref(v), 0) == 0 and v.value == 0
    chk.jacobi_debug_bounds_check.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    assert chk.jacobi_debug_bounds_check(ctypes.byref(v), 0) == 1


def test_default_variant_indices_keep_their_names(jb):
    """csrc/sweep.cu selects defaults by table index (default_variant, push_variant); DESIGN.md names
    variants by these indices (round-2 table; profiles/*_r01_* files use the round-1 numbering, which
    DESIGN.md §6 maps).  Appending variants must not shift them."""
    expect = {0: "k_sweep R4 U2", 1: "k_sweep R8 U1", 2: "k_sweep_cta R8 U1", 3: "k_sweep_cta R4 U1",
              4: "k_sweep_cta R8 U1 fused-exchange", 5: "k_sweep_panel R4 U1", 6: "k_sweep_panel R4 U1 x-smem",
              7: "k_sweep_cta R8 U1 L2-policy", 8: "k_sweep_cta R8 U1 L2-policy rows/2",
              9: "k_sweep_cta R8 U1 L2-policy dynamic", 10: "k_sweep_cta R4 U2 L2-policy dynamic",
              11: "k_sweep_cta R4 U2 dynamic fused-exchange", 12: "k_sweep_group R8 G4 x-smem",
              13: "k_sweep R4 U2 L2-policy"}
    for v, name in expect.items():
        assert jb.variant_name(v) == name, (v, jb.variant_name(v))
