"""Pins for the CPU oracle (oracle/), independent of the oracle itself.

Each test checks the oracle against something the paper or mathematics fixes: closed forms, exact
rational arithmetic (Python fractions), a LAPACK solve, invariants, or special cases.  None of
these values come from the CUDA path.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U = 2.0 ** -53


def dominant_system(n, rng, margin=(1.0, 2.0)):
    """Random strictly row-diagonally-dominant system (PAPER.md:51 condition, j != i reading R7)."""
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    d = np.abs(A).sum(1) + rng.uniform(*margin, n)
    d *= rng.choice([-1.0, 1.0], n)
    np.fill_diagonal(A, d)
    xs = rng.uniform(-1, 1, n)
    return A, A @ xs, xs


def exact_jacobi(A, b, x0, kmax):
    """PAPER.md:55 iterated in exact rational arithmetic on the given fp64 inputs."""
    n = len(b)
    Af = [[Fraction(float(v)) for v in row] for row in A]
    bf = [Fraction(float(v)) for v in b]
    x = [Fraction(float(v)) for v in x0]
    out = []
    for _ in range(kmax):
        xn = [(bf[i] - sum(Af[i][j] * x[j] for j in range(n) if j != i)) / Af[i][i] for i in range(n)]
        d = max(abs(xn[i] - x[i]) for i in range(n))
        out.append((xn, d))
        x = xn
    return out


# ---------------------------------------------------------------- P1: 2x2 closed form
def test_p1_two_by_two_closed_form_and_iteration_count():
    """A=[[2,1],[1,3]], b=[3,4], x0=0.  Closed form:
    x^(2m) = (1 - 6^-m)[1,1], x^(2m+1) = [1 + 6^-m/2, 1 + 6^-m/3]; d_2m = 4*6^-m, d_2m+1 = 1.5*6^-m."""
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = np.array([3.0, 4.0])
    for k in range(1, 31):
        st, x, it = oracle.jacobi(A, b, None, k, 0.0)
        assert st == oracle.MAX_ITER and it == k
        m = k // 2
        if k % 2 == 0:
            ref = np.array([1 - 6.0 ** -m, 1 - 6.0 ** -m])
        else:
            ref = np.array([1 + 6.0 ** -m / 2, 1 + 6.0 ** -m / 3])
        assert np.allclose(x, ref, rtol=8 * U, atol=0)
    st, x, it, h = oracle.jacobi(A, b, None, 1000, 1e-12, history=True)
    assert (st, it) == (oracle.CONVERGED, 33)
    for k in range(1, 34):
        m = k // 2
        ref = 4 * 6.0 ** -m if k % 2 == 0 else 1.5 * 6.0 ** -m
        assert h[k - 1] == pytest.approx(ref, rel=1e-9)
    assert h[31] >= 1e-12 > h[32]  # d_32 = 1.41787e-12 not < tol; d_33 = 5.31686e-13 is
    assert np.allclose(x, [1.0, 1.0], atol=1e-12)
    # SPEC.md:145-146 single steps
    assert np.array_equal(oracle.sweep_rows(A, 0, b, np.zeros(2)), [1.5, 4.0 / 3.0])
    np.testing.assert_allclose(oracle.sweep_rows(A, 0, b, np.array([1.5, 4 / 3])), [5 / 6, 5 / 6], rtol=2 * U)


# ---------------------------------------------------------------- P2: 3x3 golden exact iterates
def _read_golden_p2():
    rows = []
    with open(os.path.join(GOLDEN, "p2_3x3_iterates.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("A "):
                A = [[int(v) for v in r.split()] for r in line[2:].split(";")]
            elif line.startswith("b "):
                b = [int(v) for v in line[2:].split()]
            else:
                k, xs, d = [p.strip() for p in line.split("|")]
                rows.append((int(k), [Fraction(v) for v in xs.split()], Fraction(d)))
    return np.array(A, float), np.array(b, float), rows


def test_p2_three_by_three_exact_iterates():
    A, b, rows = _read_golden_p2()
    exact = exact_jacobi(A, b, np.zeros(3), 4)
    for (k, xs, d), (xe, de) in zip(rows, exact):
        assert xe == xs and de == d  # the golden file agrees with exact rational arithmetic
        st, x, it, h = oracle.jacobi(A, b, None, k, 0.0, history=True)
        assert it == k
        np.testing.assert_allclose(x, [float(v) for v in xs], rtol=16 * U, atol=16 * U)
        assert h[-1] == pytest.approx(float(d), rel=1e-14)
    # ||T||inf = 0.8
    T = np.abs(A) / np.abs(np.diag(A))[:, None]
    np.fill_diagonal(T, 0)
    assert T.sum(1).max() == pytest.approx(0.8)


# ---------------------------------------------------------------- P3: first sweep from zero
def test_p3_first_sweep_is_b_over_diag_bitwise():
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 64, 129):
        A, b, _ = dominant_system(n, rng)
        st, x, it, h = oracle.jacobi(A, b, np.zeros(n), 1, 0.0, history=True)
        ref = b / np.diag(A)
        assert np.array_equal(x, ref)
        assert h[0] == np.max(np.abs(ref))


# ---------------------------------------------------------------- P4: diagonal systems
def test_p4_diagonal_system_stop_counting():
    rng = np.random.default_rng(4)
    d = rng.uniform(1, 2, 10)
    A = np.diag(d)
    b = rng.uniform(-1, 1, 10)
    st, x, it = oracle.jacobi(A, b, None, 50, 1e-300)
    assert (st, it) == (oracle.CONVERGED, 2) and np.array_equal(x, b / d)
    st, x, it = oracle.jacobi(A, b, b / d, 50, 1e-300)
    assert (st, it) == (oracle.CONVERGED, 1)
    st, x, it = oracle.jacobi(np.array([[4.0]]), np.array([2.0]), None, 5, 0.0)  # n = 1
    assert (st, it) == (oracle.MAX_ITER, 5) and x[0] == 0.5


# ---------------------------------------------------------------- P5: integer fixed point
def test_p5_integer_planted_fixed_point():
    A, b, _ = _read_golden_p2()
    xs = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(A @ xs, b)
    st, x, it, h = oracle.jacobi(A, b, xs, 10, 1e-300, history=True)
    assert (st, it) == (oracle.CONVERGED, 1) and np.array_equal(x, xs) and h[0] == 0.0


# ---------------------------------------------------------------- P6: power-of-two row scaling
def test_p6_power_of_two_row_scaling_is_bitwise_invariant():
    rng = np.random.default_rng(6)
    A, b, _ = dominant_system(40, rng)
    e = rng.integers(-20, 21, 40)
    s = np.ldexp(1.0, e)
    x0 = rng.uniform(-1, 1, 40)
    r1 = oracle.jacobi(A, b, x0, 25, 0.0, history=True)
    r2 = oracle.jacobi(A * s[:, None], b * s, x0, 25, 0.0, history=True)
    assert np.array_equal(r1[1], r2[1]) and np.array_equal(r1[3], r2[3])


# ---------------------------------------------------------------- P7: direct solves
def test_p7_converged_value_matches_gaussian_elimination_and_lapack():
    rng = np.random.default_rng(7)
    for t in range(20):
        n = int(rng.integers(1, 65))
        A, b, _ = dominant_system(n, rng)
        x_ge = oracle.ge_solve(A, b)
        x_np = np.linalg.solve(A, b)  # LAPACK gesv
        assert np.max(np.abs(x_ge - x_np)) <= 1e-12 * max(1.0, np.max(np.abs(x_np)))
        st, x, it = oracle.jacobi(A, b, None, 10000, 1e-14)
        assert st == oracle.CONVERGED
        assert np.max(np.abs(x - x_ge)) <= 1e-10 * max(1.0, np.max(np.abs(x_ge)))
    # SPEC.md:471-473 style: GE on a system needing pivoting
    A = np.array([[0.0, 1.0], [2.0, 1.0]])
    np.testing.assert_allclose(oracle.ge_solve(A, np.array([1.0, 3.0])), [1.0, 1.0])


# ---------------------------------------------------------------- P8: planted solution (generator c1)
def test_p8_planted_solution_c1():
    import jacobi_gen as g
    A, b, xs = g.host_system(g.CONFIGS["c1"])
    st, x, it = oracle.jacobi(A, b, None, 200, 0.0, nthreads=4)
    assert (st, it) == (oracle.MAX_ITER, 200)
    assert np.max(np.abs(x - xs)) <= 1e-12
    st, x, it, h = oracle.jacobi(A, b, None, 200, 1e-12, history=True)
    assert st == oracle.CONVERGED and h[-1] < 1e-12 <= h[-2]


# ---------------------------------------------------------------- P9: contraction
def test_p9_contraction_bounds():
    rng = np.random.default_rng(9)
    for n in (5, 17, 60):
        A, b, _ = dominant_system(n, rng, margin=(0.05, 0.5))
        xs = oracle.ge_solve(A, b)
        T = np.abs(A) / np.abs(np.diag(A))[:, None]
        np.fill_diagonal(T, 0.0)
        tn = T.sum(1).max()
        assert tn < 1.0  # dominance => ||T||inf < 1
        x0 = rng.uniform(-1, 1, n)
        e0 = np.max(np.abs(x0 - xs))
        st, x, it, h = oracle.jacobi(A, b, x0, 60, 0.0, history=True)
        xk = x0
        for k in range(1, 61):
            xk = oracle.sweep_rows(A, 0, b, xk)
            assert np.max(np.abs(xk - xs)) <= tn ** k * e0 + 1e-13
        for k in range(1, 60):  # scaled residual D^-1(b - A x^(k)) = x^(k+1) - x^(k) contracts
            assert h[k] <= tn * h[k - 1] + 1e-14


def test_p9b_slow_companion_rate_is_exactly_one_over_1_05():
    """SURVEY.md Q21's slow companion (off-diagonals U[0,1); a_ii = 1.05 x row sum):
    T = -D^-1(L+U) is entrywise non-positive with every row of |T| summing to 1/1.05, so T 1 = -(1/1.05) 1
    and rho(T) = ||T||inf = 1/1.05 (Perron).  Once that mode dominates, d_{k+1} / d_k equals 1/1.05 to
    rounding; a dropped or doubled term, a wrong diagonal or an off-by-one row index changes the rate."""
    rng = np.random.default_rng(5)
    for n in (50, 200):
        A = rng.uniform(0, 1, (n, n))
        np.fill_diagonal(A, 0.0)
        np.fill_diagonal(A, 1.05 * A.sum(1))
        b = A @ rng.uniform(-1, 1, n)
        st, x, it, h = oracle.jacobi(A, b, None, 300, 0.0, history=True)
        assert (st, it) == (oracle.MAX_ITER, 300)
        h = np.asarray(h)
        assert np.all(h[1:] <= h[:-1] / 1.05 + 1e-14)  # ||T||inf bound (P9) from the first sweep on
        ratio = h[1:] / h[:-1]
        assert np.max(np.abs(ratio[100:250] - 1 / 1.05)) <= 1e-8


# ---------------------------------------------------------------- P10: exact rational brute force
def test_p10_exact_rational_brute_force():
    rng = np.random.default_rng(10)
    for n in (1, 2, 3, 4, 6):
        A, b, _ = dominant_system(n, rng)
        x0 = rng.uniform(-1, 1, n)
        exact = exact_jacobi(A, b, x0, 12)
        M = max(float(max(abs(v) for v in xe)) for xe, _ in exact) + np.max(np.abs(b))
        for k, (xe, de) in enumerate(exact, start=1):
            st, x, it, h = oracle.jacobi(A, b, x0, k, 0.0, history=True)
            err = max(abs(Fraction(float(x[i])) - xe[i]) for i in range(n))
            assert float(err) <= 4 * k * (n + 2) * U * M
            assert abs(h[-1] - float(de)) <= 8 * k * (n + 2) * U * M


# ---------------------------------------------------------------- P11: split runs
def test_p11_split_run_is_bitwise_equal():
    rng = np.random.default_rng(11)
    A, b, _ = dominant_system(50, rng, margin=(0.01, 0.1))
    x0 = rng.uniform(-1, 1, 50)
    _, xa, _, ha = oracle.jacobi(A, b, x0, 17, 0.0, history=True)
    _, x1, _, h1 = oracle.jacobi(A, b, x0, 9, 0.0, history=True)
    _, x2, _, h2 = oracle.jacobi(A, b, x1, 8, 0.0, history=True)
    assert np.array_equal(xa, x2) and np.array_equal(ha, np.concatenate([h1, h2]))


# ---------------------------------------------------------------- P13: determinism / threads
def test_p13_thread_count_and_repeat_invariance():
    rng = np.random.default_rng(13)
    A, b, _ = dominant_system(97, rng)
    ref = oracle.jacobi(A, b, None, 30, 0.0, nthreads=1, history=True)
    for t in (2, 3, 8, 97):
        r = oracle.jacobi(A, b, None, 30, 0.0, nthreads=t, history=True)
        assert np.array_equal(r[1], ref[1]) and np.array_equal(r[3], ref[3])


# ---------------------------------------------------------------- P14: divergent paper regime
@pytest.mark.parametrize("n", [8, 64])
def test_p14_paper_raw_regime_diverges_to_max_iter(n):
    """A, B, X random in [0,1] (not dominant), tol 1e-8 'to guarantee that L will be
    reached'.  The iterates overflow; NaN is sticky, so the run never converges."""
    rng = np.random.default_rng(14)
    A = rng.uniform(0, 1, (n, n))
    b = rng.uniform(0, 1, n)
    x0 = rng.uniform(0, 1, n)
    st, x, it, h = oracle.jacobi(A, b, x0, 1000, 1e-8, history=True)
    assert (st, it) == (oracle.MAX_ITER, 1000)
    bad = ~np.isfinite(h)
    assert bad.any()
    first_bad = np.argmax(bad)  # inf (alternating-sign overflow) or NaN (inf - inf); either is sticky
    assert bad[first_bad:].all() and first_bad > 0
    assert not np.isfinite(x).all()


# ---------------------------------------------------------------- error semantics (§8(b))
def test_errors_and_edge_cases():
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = np.array([3.0, 4.0])
    assert oracle.jacobi(A, b, None, -1, 1e-3)[0] == oracle.EINVAL
    assert oracle.jacobi(A, b, None, 5, -1.0)[0] == oracle.EINVAL
    assert oracle.jacobi(A, b, None, 5, float("nan"))[0] == oracle.EINVAL
    Z = np.array([[1.0, 0, 0], [0, 0.0, 0], [0, 0, 0.0]])
    assert oracle.jacobi(Z, np.ones(3), None, 5, 0.0)[0] == oracle.EZERODIAG
    Zn = Z.copy(); Zn[0, 1] = np.nan  # zero diagonal takes precedence over non-finite
    assert oracle.jacobi(Zn, np.ones(3), None, 5, 0.0)[0] == oracle.EZERODIAG
    An = A.copy(); An[1, 0] = np.inf
    assert oracle.jacobi(An, b, None, 5, 0.0)[0] == oracle.ENONFINITE
    assert oracle.jacobi(A, np.array([1.0, np.nan]), None, 5, 0.0)[0] == oracle.ENONFINITE
    assert oracle.jacobi(A, b, np.array([np.inf, 0.0]), 5, 0.0)[0] == oracle.ENONFINITE
    x0 = np.array([0.25, -0.5])
    st, x, it = oracle.jacobi(A, b, x0, 0, 1e-3)  # max_iter = 0 -> X^0, MAX_ITER (R14)
    assert (st, it) == (oracle.MAX_ITER, 0) and np.array_equal(x, x0)
    st, x, it = oracle.jacobi(A, b, None, 5, math.inf)  # tol = inf converges at k = 1 (R13)
    assert (st, it) == (oracle.CONVERGED, 1)
    st, x, it = oracle.jacobi(A, b, None, 300, 0.0)  # tol = 0 never converges
    assert (st, it) == (oracle.MAX_ITER, 300)


def test_sweep_rows_matches_full_sweep_on_row_subsets():
    rng = np.random.default_rng(15)
    A, b, _ = dominant_system(33, rng)
    x0 = rng.uniform(-1, 1, 33)
    _, x1, _ = oracle.jacobi(A, b, x0, 1, 0.0)
    for r0, r1 in ((0, 33), (5, 6), (10, 30)):
        assert np.array_equal(oracle.sweep_rows(A[r0:r1], r0, b[r0:r1], x0), x1[r0:r1])


def test_fp32_storage_widens_exactly():
    rng = np.random.default_rng(16)
    A, b, _ = dominant_system(20, rng)
    A32 = A.astype(np.float32)
    r32 = oracle.jacobi(A32, b, None, 12, 0.0, history=True)
    r64 = oracle.jacobi(A32.astype(np.float64), b, None, 12, 0.0, history=True)
    assert np.array_equal(r32[1], r64[1]) and np.array_equal(r32[3], r64[3])


# ---------------------------------------------------------------- NEXT-2: the paper's Euclidean stop rule
def test_l2_distance_pins():
    """||X^(k+1) - X^(k)|| = sqrt(sum_i (X_i^(k+1) - X_i^(k))^2)."""
    assert oracle.l2_dist([3.0, 0.0], [0.0, 4.0]) == 5.0  # SPEC.md:79 (3-4-5)
    assert oracle.l2_dist([1.0, 1, 1, 1], [0.0, 0, 0, 0]) == 2.0
    assert oracle.l2_dist([1.0, 2, 3], [1.0, 2, 3]) == 0.0
    # 2x2 closed form (P1): d_2m = 5 * 6^-m (a 3-4-5 triangle scaled by 6^-m), d_2m+1 = sqrt(145)/6 * 6^-m
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = np.array([3.0, 4.0])
    st, x, it, h = oracle.jacobi(A, b, None, 1000, 1e-12, history=True, norm="l2")
    for k in range(1, it + 1):
        m = k // 2
        ref = 5 * 6.0 ** -m if k % 2 == 0 else math.sqrt(145) / 6 * 6.0 ** -m
        assert h[k - 1] == pytest.approx(ref, rel=1e-9)
    assert (st, it) == (oracle.CONVERGED, 33) and h[31] >= 1e-12 > h[32]  # d_32 = 5*6^-16 = 1.77e-12
    # exact-rational iterates (P2 golden) with the Euclidean distance
    A3, b3, rows = _read_golden_p2()
    for k, xs, d in rows:
        st, x, it, h = oracle.jacobi(A3, b3, None, k, 0.0, history=True, norm="l2")
        prev = [Fraction(0)] * 3 if k == 1 else rows[k - 2][1]
        ref = math.sqrt(float(sum((xs[i] - prev[i]) ** 2 for i in range(3))))
        assert h[-1] == pytest.approx(ref, rel=1e-14)
    # L2 >= max norm, so with the same tol the L2 rule never stops earlier
    rng = np.random.default_rng(21)
    A, b, _ = dominant_system(40, rng, margin=(0.05, 0.3))
    r_max = oracle.jacobi(A, b, None, 5000, 1e-10)
    r_l2 = oracle.jacobi(A, b, None, 5000, 1e-10, norm="l2")
    assert r_l2[2] >= r_max[2]
