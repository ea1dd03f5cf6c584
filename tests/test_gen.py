"""Input generator (jacobi_gen/) checks: the recipe of DESIGN.md §4 and jacobi_gen.h."""
import numpy as np
import pytest

import jacobi_gen as g


def test_c1_recipe_properties():
    cfg = g.CONFIGS["c1"]
    A, b, xs = g.host_system(cfg)
    n = cfg.n
    off = A.copy()
    np.fill_diagonal(off, 0.0)
    # off-diagonals on the 2^-31 grid in [-1, 1)
    assert off.min() >= -1.0 and off.max() < 1.0
    assert np.array_equal(off * 2.0 ** 31, np.round(off * 2.0 ** 31))
    rowabs = np.abs(off).sum(1)
    extra = np.diag(A) - rowabs
    assert (extra >= 1.0 - 1e-12).all() and (extra < 2.0 + 1e-12).all()  # rowabs + U[1,2)
    assert np.abs(xs).max() <= 1.0
    # b = A x* up to the two documented roundings
    np.testing.assert_allclose(A @ xs, b, rtol=0, atol=1e-12 * np.abs(b).max())
    # mean/std of U[-1,1) draws
    v = off[~np.eye(n, dtype=bool)]
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1 / np.sqrt(3)) < 0.01


def test_scale_mode_and_fp32_storage():
    cfg = g.GenConfig(512, a_dtype=g.F32, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
    A, b, xs = g.host_system(cfg)
    assert A.dtype == np.float32
    off = A.astype(np.float64)
    d = np.diag(off).copy()
    np.fill_diagonal(off, 0.0)
    assert np.array_equal(off * 2.0 ** 23, np.round(off * 2.0 ** 23))  # exact in fp32
    rowabs = np.abs(off).sum(1)
    np.testing.assert_allclose(d, 1.2 * rowabs, rtol=1e-7)
    np.testing.assert_allclose(A.astype(np.float64) @ xs, b, rtol=0, atol=1e-12 * np.abs(b).max())
    cfg3 = g.GenConfig(300, diag_mode=g.DIAG_SCALE, diag_scale=1.05)
    A3, _, _ = g.host_system(cfg3)
    off3 = np.abs(A3).sum(1) - np.abs(np.diag(A3))
    np.testing.assert_allclose(np.diag(A3), 1.05 * off3, rtol=1e-15)


def test_row_addressable_thread_invariant_and_seeded():
    cfg = g.GenConfig(333, seed=5)
    A, b, _ = g.host_system(cfg, nthreads=7)
    A1, b1 = g.host_rows(cfg, 100, 140, nthreads=1)
    assert np.array_equal(A[100:140], A1) and np.array_equal(b[100:140], b1)
    Ap, bp = g.host_rows(cfg, 0, 333, lda=340)
    assert np.array_equal(Ap[:, :333], A) and (Ap[:, 333:] == 0).all() and np.array_equal(bp, b)
    d, bd = g.host_diag_b(cfg, 0, 333)
    assert np.array_equal(d, np.diag(A)) and np.array_equal(bd, b)
    A2, b2, _ = g.host_system(g.GenConfig(333, seed=6))
    assert not np.array_equal(A, A2)
    A3, b3, _ = g.host_system(cfg)
    assert np.array_equal(A, A3) and np.array_equal(b, b3)


def test_n1():
    A, b, xs = g.host_system(g.GenConfig(1))
    assert A.shape == (1, 1) and 1.0 <= A[0, 0] < 2.0 and b[0] == A[0, 0] * xs[0]
