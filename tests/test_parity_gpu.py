"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): relative L-inf error <= 1e-10 for fp64 and <= 1e-4 for fp32
A storage (self-checked at 1e-10: both sides accumulate in fp64 on identical fp32 values), and the
same iteration count.  Bitwise checks where the arithmetic fixes the bits: sweep 1 from x0 = 0
(P3), row-block invariance (P12a), determinism (P13), split runs (P11), batch-size invariance.
"""
import math

import numpy as np
import pytest

import jacobi_gen as g
import oracle

pytestmark = pytest.mark.gpu

TOL64 = 1e-10
TOL32 = 1e-4


@pytest.fixture(scope="module")
def jb():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1403_5805_b200 as jb
    return jb


def rel_linf(x, ref):
    den = np.max(np.abs(ref))
    err = np.max(np.abs(np.asarray(x) - ref))
    return err / den if den > 0 else err


def match_oracle(r, orc, tol=TOL64):
    """Status, iteration count, x (relative L-inf <= tol) and, when both sides kept it, the d_k history
    of a GPU result against an oracle.jacobi(..., history=True) tuple."""
    st_o, x_o, it_o, h_o = orc
    assert (r.status, r.iters) == (st_o, it_o), (r.status, r.iters, st_o, it_o)
    assert rel_linf(r.x, x_o) <= tol
    if r.hist is not None:
        np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


def dominant(n, seed, scale=None, f32=False):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    rs = np.abs(A).sum(1)
    d = rs * scale if scale else rs + rng.uniform(1, 2, n)
    d[d == 0] = 1.0  # n = 1: no off-diagonals
    np.fill_diagonal(A, d * rng.choice([-1.0, 1.0], n))
    if f32:
        A = A.astype(np.float32)
    xs = rng.uniform(-1, 1, n)
    b = A.astype(np.float64) @ xs
    return A, b, xs


# ------------------------------------------------------------------ configs c1 / c2
def test_c1_fixed_200_and_tol_stop(jb):
    A, b, xs = g.host_system(g.CONFIGS["c1"])
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 200, 0.0, nthreads=8, history=True)
    with jb.Plan(A) as p:
        r = p.solve(b, None, 200, 0.0, history=True)
        assert (r.status, r.iters) == (jb.MAX_ITER, it_o) == (jb.MAX_ITER, 200)
        assert rel_linf(r.x, x_o) <= TOL64
        assert np.max(np.abs(r.x - xs)) <= 1e-12  # P8 planted
        # tol = 1e-12 stop run (BASELINE.json configs[0]); same iteration count as the oracle
        st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 200, 1e-12, history=True)
        r = p.solve(b, None, 200, 1e-12, history=True)
        assert (r.status, r.iters) == (st_o, it_o) == (jb.CONVERGED, 12)
        assert rel_linf(r.x, x_o) <= TOL64
        np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


def test_c2_parity_and_planted(jb):
    A, b, xs = g.host_system(g.CONFIGS["c2"])
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 40, 0.0, nthreads=16, history=True)
    with jb.Plan(A) as p:
        r = p.solve(b, None, 40, 0.0, history=True)
        assert r.iters == 40 and rel_linf(r.x, x_o) <= TOL64
        # d_k is a difference of iterates: its error is absolute (~ulp(x)), not relative
        np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)
        r = p.solve(b, None, 500, 0.0)  # configs[1]: fixed 500 iterations
        assert (r.status, r.iters) == (jb.MAX_ITER, 500)
        assert np.max(np.abs(r.x - xs)) <= 1e-12


# ------------------------------------------------------------------ early sweeps (in-place race guard)
def test_early_sweeps_match_one_by_one(jb):
    A, b, _ = dominant(1500, 1, scale=1.05)
    x0 = np.random.default_rng(2).uniform(-1, 1, 1500)
    with jb.Plan(A) as p:
        xo = x0.copy()
        for k in range(1, 9):
            xo = oracle.sweep_rows(A, 0, b, xo)
            r = p.solve(b, x0, k, 0.0)
            assert r.iters == k and rel_linf(r.x, xo) <= 1e-13, k


# ------------------------------------------------------------------ P3: sweep 1 from zero, bitwise
@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 33, 127, 257, 1000, 4099])
def test_p3_first_sweep_bitwise_ragged(jb, n):
    A, b, _ = dominant(n, n)
    st, x_o, it = oracle.jacobi(A, b, None, 1, 0.0)
    r = jb.solve(A, b, None, 1, 0.0)
    assert r.iters == 1 and np.array_equal(r.x, x_o)


# ------------------------------------------------------------------ ragged sizes, tol stops
@pytest.mark.parametrize("n", [1, 2, 5, 64, 255, 513, 2049, 5000])
def test_ragged_sizes_parity(jb, n):
    A, b, xs = dominant(n, 100 + n, scale=1.05)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 30, 0.0, nthreads=8, history=True)
    with jb.Plan(A) as p:
        r = p.solve(b, None, 30, 0.0, history=True)
        assert r.iters == 30 and rel_linf(r.x, x_o) <= TOL64
        st_o, x_o, it_o = oracle.jacobi(A, b, None, 1000, 1e-9, nthreads=8)
        r = p.solve(b, None, 1000, 1e-9)
        assert (r.status, r.iters) == (st_o, it_o)
        assert rel_linf(r.x, x_o) <= TOL64


def test_fp32_storage_parity(jb):
    for n in (1000, 3000):
        A, b, xs = dominant(n, 7 + n, scale=1.2, f32=True)
        st_o, x_o, it_o = oracle.jacobi(A, b, None, 25, 0.0, nthreads=8)
        r = jb.solve(A, b, None, 25, 0.0)
        assert r.iters == 25 and rel_linf(r.x, x_o) <= 1e-10  # self-check; official bar TOL32
        st_o, x_o, it_o = oracle.jacobi(A, b, None, 2000, 1e-6, nthreads=8)
        r = jb.solve(A, b, None, 2000, 1e-6)
        assert (r.status, r.iters) == (st_o, it_o) and rel_linf(r.x, x_o) <= TOL32
    cfg = g.GenConfig(2048, a_dtype=g.F32, diag_mode=g.DIAG_SCALE, diag_scale=1.2)  # c5 recipe, small n
    A, b, xs = g.host_system(cfg)
    st_o, x_o, it_o = oracle.jacobi(A, b, None, 2000, 1e-6, nthreads=8)
    r = jb.solve(A, b, None, 2000, 1e-6)
    assert (r.status, r.iters) == (st_o, it_o) and rel_linf(r.x, x_o) <= TOL32


# ------------------------------------------------------------------ invariances (bitwise)
def test_p12a_row_block_launches_bitwise(jb):
    A, b, _ = dominant(4096, 12, scale=1.05)
    with jb.Plan(A) as p:
        ref = p.solve(b, None, 15, 0.0, history=True)
        for nb in (2, 4, 8, 16):
            p.set_row_blocks(nb)
            r = p.solve(b, None, 15, 0.0, history=True)
            assert np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist), nb
        p.set_row_blocks(4)
        r1 = p.solve(b, None, 500, 1e-10)
        p.set_row_blocks(1)
        r2 = p.solve(b, None, 500, 1e-10)
        assert r1.iters == r2.iters and np.array_equal(r1.x, r2.x)


def test_p13_p11_determinism_split_and_batch(jb):
    A, b, _ = dominant(3000, 13, scale=1.02)
    with jb.Plan(A) as p:
        a = p.solve(b, None, 37, 0.0, history=True)
        a2 = p.solve(b, None, 37, 0.0, history=True)
        assert np.array_equal(a.x, a2.x) and np.array_equal(a.hist, a2.hist)  # P13
        h1 = p.solve(b, None, 20, 0.0, history=True)
        h2 = p.solve(b, h1.x, 17, 0.0, history=True)
        assert np.array_equal(h2.x, a.x) and np.array_equal(np.concatenate([h1.hist, h2.hist]), a.hist)  # P11
        for K in (4, 8, 64, 1024):
            p.set_batch(K)
            r = p.solve(b, None, 37, 0.0, history=True)
            assert r.iters == 37 and np.array_equal(r.x, a.x), K
            c = p.solve(b, None, 5000, 1e-11)
            p.set_batch(32)
            c32 = p.solve(b, None, 5000, 1e-11)
            assert (c.status, c.iters) == (c32.status, c32.iters) and np.array_equal(c.x, c32.x)


# ------------------------------------------------------------------ P14: divergent paper regime
@pytest.mark.parametrize("n", [8, 64, 512, 2000, 5000])  # cluster, persistent (2000), graph (5000) paths
def test_p14_divergence_nan_semantics(jb, n):
    rng = np.random.default_rng(14)
    A = rng.uniform(0, 1, (n, n))
    b = rng.uniform(0, 1, n)
    x0 = rng.uniform(0, 1, n)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, 1000, 1e-8, nthreads=16, history=True)
    with jb.Plan(A) as p:
        r = p.solve(b, x0, 1000, 1e-8, history=True)
    assert (r.status, r.iters) == (st_o, it_o) == (jb.MAX_ITER, 1000)
    bad_o = np.argmax(~np.isfinite(h_o))
    bad_g = np.argmax(~np.isfinite(r.hist))
    assert abs(int(bad_o) - int(bad_g)) <= 1 and (~np.isfinite(r.hist[bad_g:])).all()
    assert not np.isfinite(r.x).all() and not np.isfinite(x_o).all()


# ------------------------------------------------------------------ errors and edge cases
def test_errors_and_edges_on_gpu(jb):
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = np.array([3.0, 4.0])
    r = jb.solve(A, b, None, 1000, 1e-12)
    assert (r.status, r.iters) == (jb.CONVERGED, 33)  # P1 on the GPU
    Z = np.eye(6)
    Z[4, 4] = 0.0
    Z[2, 2] = 0.0
    with pytest.raises(jb.JacobiError) as e:
        jb.solve(Z, np.ones(6), None, 5, 0.0)
    assert e.value.status == jb.EZERODIAG and "i = 2" in str(e.value)
    An = np.eye(3)
    An[0, 2] = np.nan
    with pytest.raises(jb.JacobiError) as e:
        jb.solve(An, np.ones(3), None, 5, 0.0)
    assert e.value.status == jb.ENONFINITE
    with pytest.raises(jb.JacobiError) as e:
        jb.solve(np.eye(3), np.array([1.0, np.inf, 0.0]), None, 5, 0.0)
    assert e.value.status == jb.ENONFINITE
    x0 = np.array([0.25, -0.5])
    r = jb.solve(A, b, x0, 0, 1e-3)
    assert (r.status, r.iters) == (jb.MAX_ITER, 0) and np.array_equal(r.x, x0)
    r = jb.solve(A, b, None, 7, math.inf)
    assert (r.status, r.iters) == (jb.CONVERGED, 1)
    P5A = np.array([[4.0, -2, 1], [1, 5, -3], [2, 2, 6]])
    r = jb.solve(P5A, np.array([3.0, 2, 24]), np.array([1.0, 2, 3]), 10, 1e-300)
    assert (r.status, r.iters) == (jb.CONVERGED, 1) and np.array_equal(r.x, [1.0, 2.0, 3.0])  # P5


@pytest.mark.parametrize("n,f32", [(256, False), (2000, False), (5000, False), (3001, True), (9001, True)])
def test_p6_row_scaling_and_p4_diagonal_on_every_path(jb, n, f32):
    """Pins P6 and P4 on the CUDA path, at sizes that take the cluster (256),
    persistent (2000, fp32 3001) and graph (5000, fp32 9001) paths.
    P6: scaling row i of A and b_i by 2^e_i (PAPER.md:55 is homogeneous per row: every product, partial
    sum and the division scale exactly) leaves every iterate and every d_k bitwise unchanged — a row
    index off by one anywhere (b_i, a_ii, the diagonal mask, x_i^(k-1) of the epilogue) breaks it.
    P4: a diagonal system gives x = b / diag after sweep 1 and d_2 = 0, i.e. CONVERGED at k = 2."""
    A, b, _ = dominant(n, 600 + n, scale=1.1, f32=f32)
    rng = np.random.default_rng(n)
    s = np.ldexp(1.0, rng.integers(-20, 21, n))
    As = (A.astype(np.float64) * s[:, None]).astype(A.dtype)  # exact: powers of two, no over/underflow
    x0 = rng.uniform(-1, 1, n)
    with jb.Plan(A) as p, jb.Plan(As) as q:
        assert (p.info.persistent_ctas > 0) == (q.info.persistent_ctas > 0)
        r = p.solve(b, x0, 12, 0.0, history=True)
        rs = q.solve(b * s, x0, 12, 0.0, history=True)
    assert np.array_equal(r.x, rs.x) and np.array_equal(r.hist, rs.hist)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, 12, 0.0, nthreads=16, history=True)
    assert rel_linf(r.x, x_o) <= (TOL64 if not f32 else 1e-10)
    D = np.diag(np.diag(A)).astype(A.dtype)
    with jb.Plan(D) as p:
        r = p.solve(b, None, 50, 1e-300, history=True)
    assert (r.status, r.iters) == (jb.CONVERGED, 2)
    assert np.array_equal(r.x, b / np.diag(A).astype(np.float64)) and r.hist[1] == 0.0


def test_device_borrowed_A_and_device_solve(jb):
    import torch
    n = 3000
    A, b, xs = dominant(n, 21)
    dA = torch.empty((n, 3008), dtype=torch.float64, device="cuda")
    dA[:, n:] = float("nan")  # padding must never be read into a sum
    dA[:, :n] = torch.from_numpy(A).cuda()
    st_o, x_o, it_o = oracle.jacobi(A, b, None, 20, 0.0, nthreads=8)
    with jb.Plan(dA[:, :n], n=n) as p:
        assert p.info.a_borrowed == 1 and p.info.lda == 3008
        db = torch.from_numpy(b).cuda()
        dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        dxo = torch.empty(n, dtype=torch.float64, device="cuda")
        with pytest.raises(ValueError):  # the kernels write d_k into hist during the solve: too short = refused
            p.solve_device(db, dx0, dxo, 20, 0.0, hist=torch.empty(19, dtype=torch.float64, device="cuda"))
        hist = torch.empty(20, dtype=torch.float64, device="cuda")
        r = p.solve_device(db, dx0, dxo, 20, 0.0, hist=hist)
        assert r.iters == 20 and rel_linf(dxo.cpu().numpy(), x_o) <= TOL64
        r2 = p.solve(b, None, 20, 0.0, history=True)
        assert np.array_equal(r2.x, dxo.cpu().numpy()) and np.array_equal(r2.hist, hist.cpu().numpy())
        ms = p.time_sweeps(db, dx0, 3)
        assert ms.shape == (3,) and (ms > 0).all()


def test_bwprobe_sane(jb):
    gbs = jb.bwprobe(4 << 30, 3)
    assert 3000 < gbs < 9000


# ------------------------------------------------------------------ full-size configs (sampled parity)
def _device_system(jb, cfg):
    import torch
    n = cfg.n
    dt = torch.float32 if cfg.a_dtype == g.F32 else torch.float64
    dA = torch.empty((n, n), dtype=dt, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return dA, db


def test_c3_full_parity_and_shards(jb):
    """BASELINE.json configs[2] at full size (n = 16384, 2.1 GB, diag = 1.05 x row abs-sum): the tol
    1e-10 stop run against the full oracle — same status and iteration count, relative L-inf error
    <= 1e-10, d_k history — and the P = 2/4/8 row-block split of the same plan (P12a, the shards of
    the 1/2/4/8-GPU runs launched one after another on this GPU) bitwise equal to P = 1."""
    cfg = g.CONFIGS["c3"]
    A, b, xs = g.host_system(cfg)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 5000, 1e-10, nthreads=16, history=True)
    assert st_o == oracle.CONVERGED
    with jb.Plan(A) as p:
        r = p.solve(b, None, 5000, 1e-10, history=True)
        assert (r.status, r.iters) == (jb.CONVERGED, it_o)
        assert rel_linf(r.x, x_o) <= TOL64
        np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)
        # the margin of the decisive distance to tol is far above the GPU/oracle d difference (R20)
        assert h_o[it_o - 2] >= 1e-10 * 1.05 and h_o[it_o - 1] <= 1e-10 / 1.05
        assert _tie_margin_ok(r.hist, h_o, it_o, 1e-10)[0]
        for nb in (2, 4, 8):
            p.set_row_blocks(nb)
            q = p.solve(b, None, 5000, 1e-10, history=True)
            assert (q.status, q.iters) == (r.status, r.iters)
            assert np.array_equal(q.x, r.x) and np.array_equal(q.hist, r.hist), nb
        p.set_row_blocks(1)
        f = p.solve(b, None, 1000, 0.0)  # the fixed-1000 companion run the rates are quoted on
        assert (f.status, f.iters) == (jb.MAX_ITER, 1000)
        assert np.max(np.abs(f.x - xs)) <= 1e-12  # P8 planted solution


def slow_companion(n, seed, f32=False):
    return g.slow_companion(n, seed, f32)  # SURVEY.md Q21 / DESIGN.md R21 (jacobi_gen: input construction)


@pytest.mark.parametrize("n", [1500, 4096, 10007])
def test_slow_companion_iteration_count(jb, n):
    """A long tol run on the slow companion, on the persistent path (n = 1500, 4096)
    and the graph path (n = 10007, ragged): same status and iteration count as the oracle over
    ~370 sweeps of different summation orders (R20 margin checked), x within 1e-10, every d_k."""
    A, b, xs = slow_companion(n, 100 + n)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 5000, 1e-10, nthreads=16, history=True)
    assert st_o == oracle.CONVERGED and it_o > 300
    with jb.Plan(A) as p:
        r = p.solve(b, None, 5000, 1e-10, history=True)
    assert (r.status, r.iters) == (jb.CONVERGED, it_o), (r.iters, it_o)
    ok, delta = _tie_margin_ok(r.hist, h_o, it_o, 1e-10)
    assert ok, (delta, h_o[it_o - 2], h_o[it_o - 1])
    assert rel_linf(r.x, x_o) <= TOL64
    np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)
    assert np.max(np.abs(r.x - xs)) <= 1e-9  # converged to the planted solution (|x - x*| ~ d / (1 - rho))


def _twin_rows_check(cfg, dA, db, b_all, rows):
    """Device twin of the generator == host generator on sampled rows of A and on all of b (the two
    sides of every full-size parity test start from the same bits)."""
    assert np.array_equal(db.cpu().numpy(), b_all)
    for i in rows:
        Ar, _ = g.host_rows(cfg, int(i), int(i) + 1)
        assert np.array_equal(dA[int(i)].cpu().numpy(), Ar[0])


def _oracle_sweep_threaded(A, b, x, nthreads=16):
    """One application of PAPER.md:55 to every row with the oracle's oracle_sweep_rows, rows split over
    host threads (ctypes releases the GIL; per-row arithmetic is unchanged, so the bits are those of
    oracle.jacobi at any thread count — pins P11/P13)."""
    import threading
    n = A.shape[0]
    out = np.empty(n)
    bounds = [n * t // nthreads for t in range(nthreads + 1)]

    def run(t):
        r0, r1 = bounds[t], bounds[t + 1]
        if r1 > r0:
            out[r0:r1] = oracle.sweep_rows(A[r0:r1], r0, b[r0:r1], x)

    th = [threading.Thread(target=run, args=(t,)) for t in range(nthreads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def _tie_margin_ok(h_gpu, h_orc, it, tol):
    """DESIGN.md reading R20: the decisive distances sit farther from tol than the largest GPU/oracle
    difference of any d_k, so the equal iteration counts are a real agreement, not a tie."""
    delta = float(np.max(np.abs(np.asarray(h_gpu) - np.asarray(h_orc))))
    ok_last = h_orc[it - 1] < tol - delta
    ok_prev = it < 2 or h_orc[it - 2] >= tol + delta
    return ok_last and ok_prev, delta


def test_c4_full_parity_all_rows(jb, monkeypatch):
    """BASELINE.json configs[3] at full size in the bench's launch configuration (n = 65536, 34.4 GB,
    the dynamic-tile default kernel): against the oracle over the WHOLE system (PAPER.md:55 component
    equation, PAPER.md:59-66 loop) — every one of the 65536 entries after each of sweeps 1-8 (sweep 1
    bitwise: pin P3), after the 100 fixed sweeps at relative L-inf <= 1e-10, and all 100 distances d_k.
    The oracle's sweeps 1-8 are single-sweep runs chained through x0 (split runs are bitwise equal to
    one run: pin P11), so its history is the concatenation."""
    import torch
    cfg = g.CONFIGS["c4"]
    n = cfg.n
    A, b_all = g.host_rows(cfg, 0, n)  # oracle-side inputs: host generator
    dA, db = _device_system(jb, cfg)  # GPU-side inputs: device twin
    _twin_rows_check(cfg, dA, db, b_all, [0, 1, 4095, 32768, n - 2, n - 1])
    xo_orc = np.zeros(n)
    h_orc = []
    iterates = []
    for k in range(1, 9):  # one oracle sweep (oracle.sweep_rows, rows split over threads: pin P13)
        xn = _oracle_sweep_threaded(A, b_all, xo_orc)
        h_orc.append(oracle.maxnorm_dist(xn, xo_orc))
        xo_orc = xn
        iterates.append(xo_orc.copy())
    st, x100_orc, it, h = oracle.jacobi(A, b_all, xo_orc, 92, 0.0, nthreads=16, history=True)
    assert (st, it) == (oracle.MAX_ITER, 92)
    h_orc = np.concatenate([h_orc, h])
    del A
    with jb.Plan(dA) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_cta R4 U2 L2-policy dynamic"
        dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        dxo = torch.empty(n, dtype=torch.float64, device="cuda")
        for k in range(1, 9):
            r = p.solve_device(db, dx0, dxo, k, 0.0)
            assert (r.status, r.iters) == (jb.MAX_ITER, k)
            xk = dxo.cpu().numpy()
            if k == 1:
                assert np.array_equal(xk, iterates[0])  # P3: b / diag bitwise for any summation order
            assert rel_linf(xk, iterates[k - 1]) <= TOL64, k
        hist = torch.empty(100, dtype=torch.float64, device="cuda")
        r = p.solve_device(db, dx0, dxo, 100, 0.0, hist=hist)
        assert (r.status, r.iters) == (jb.MAX_ITER, 100)
        x100 = dxo.cpu().numpy()
        assert rel_linf(x100, x100_orc) <= TOL64
        np.testing.assert_allclose(hist.cpu().numpy(), h_orc, rtol=1e-9, atol=1e-14)
        assert np.max(np.abs(x100 - g.host_xstar(cfg))) <= 1e-12  # P8 planted solution
        r = p.solve_device(db, dx0, dxo, 3, 0.0)
        x3 = dxo.cpu().numpy()
    # the kernels the P = 2 / 4 / 8 ranks pick for their 32768 / 16384 / 8192-row blocks (the dynamic-tile
    # kernel at P = 2, the static L2-policy CTA kernel at P = 4 and 8), forced on the same borrowed A as
    # 2 / 4 / 8 row blocks of exactly those shapes: sweeps 1-3 bitwise equal to the P = 1 run (P12)
    for v, nbs in (("10", (2,)), ("7", (4, 8))):
        monkeypatch.setenv("JACOBI_SWEEP_VARIANT", v)
        with jb.Plan(dA) as p:
            assert p.info.variant == int(v)
            for nb in nbs:
                p.set_row_blocks(nb)
                q = p.solve_device(db, dx0, dxo, 3, 0.0)
                assert (q.status, q.iters) == (jb.MAX_ITER, 3)
                assert np.array_equal(dxo.cpu().numpy(), x3), (v, nb)
    monkeypatch.delenv("JACOBI_SWEEP_VARIANT")
    del dA
    torch.cuda.empty_cache()


def test_c5_full_parity_tol_run(jb, monkeypatch):
    """BASELINE.json configs[4] at full size (n = 131072, A stored fp32, 68.7 GB; diagonal = 1.2 x
    row abs-sum; tol 1e-6 or 2000): the whole-system oracle on the same fp32 values (widened exactly)
    must stop at the SAME iteration with the same status, x within the fp32-storage
    bar 1e-4 (self-checked at 1e-10: both sides accumulate the same fp32 values in fp64), the same
    distance history, and a decisive margin to tol larger than the GPU/oracle d_k difference (R20)."""
    import torch
    cfg = g.CONFIGS["c5"]
    n = cfg.n
    A, b_all = g.host_rows(cfg, 0, n)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b_all, None, 2000, 1e-6, nthreads=16, history=True)
    assert st_o == oracle.CONVERGED
    dA, db = _device_system(jb, cfg)
    _twin_rows_check(cfg, dA, db, b_all, [0, 1, 65535, n - 1])
    del A
    with jb.Plan(dA) as p:
        dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        dxo = torch.empty(n, dtype=torch.float64, device="cuda")
        hist = torch.empty(2000, dtype=torch.float64, device="cuda")
        r = p.solve_device(db, dx0, dxo, 2000, 1e-6, hist=hist)
        assert (r.status, r.iters) == (jb.CONVERGED, it_o)
        x = dxo.cpu().numpy()
        assert rel_linf(x, x_o) <= TOL32 and rel_linf(x, x_o) <= 1e-10
        h = hist.cpu().numpy()[:it_o]
        np.testing.assert_allclose(h, h_o, rtol=1e-9, atol=1e-14)
        ok, delta = _tie_margin_ok(h, h_o, it_o, 1e-6)
        assert ok, (h_o, delta)
        assert np.max(np.abs(x - g.host_xstar(cfg))) <= 1e-5  # planted solution, to the stop tolerance
        r = p.solve_device(db, dx0, dxo, 100, 0.0)  # the fixed-100 companion the rates are quoted on
        assert (r.status, r.iters) == (jb.MAX_ITER, 100)
        assert np.max(np.abs(dxo.cpu().numpy() - g.host_xstar(cfg))) <= 1e-12
    # the P = 2/4/8 shards' kernel (the group kernel a rank with 65536 / 32768 / 16384 rows picks):
    # forced on the same borrowed A, as one launch and as 2/4/8 row blocks of exactly the shard shapes,
    # bitwise equal to the P = 1 default run above (P12) — same stop iteration, x and d_k history
    monkeypatch.setenv("JACOBI_SWEEP_VARIANT", "12")
    with jb.Plan(dA) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_group R8 G4 x-smem"
        for nb in (1, 2, 4, 8):
            p.set_row_blocks(nb)
            dxq = torch.empty(n, dtype=torch.float64, device="cuda")
            hq = torch.empty(2000, dtype=torch.float64, device="cuda")
            q = p.solve_device(db, dx0, dxq, 2000, 1e-6, hist=hq)
            assert (q.status, q.iters) == (jb.CONVERGED, it_o), nb
            assert np.array_equal(dxq.cpu().numpy(), x) and np.array_equal(hq.cpu().numpy()[:it_o], h), nb
    del dA
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ kernel variants (same bits by design)
@pytest.mark.parametrize("n,f32", [(3000, False), (8190, False), (16384, False), (16384, True)])
def test_all_sweep_variants_bitwise_identical(jb, n, f32, monkeypatch):
    """Every sweep-kernel variant (item kernel with R in {2,4,8}, CTA-cooperative kernel) must give
    identical bits: the per-row summation order depends only on column indices (R10)."""
    A, b, _ = dominant(n, 31 + n, scale=1.05, f32=f32)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 12, 0.0, nthreads=16, history=True)
    ref = None
    with jb.Plan(A) as p:
        nvar = p.info.num_variants  # the fused-exchange instance is never selected by JACOBI_SWEEP_VARIANT
    assert nvar >= 11
    for v in range(nvar):
        monkeypatch.setenv("JACOBI_SWEEP_VARIANT", str(v))
        with jb.Plan(A) as p:
            assert p.info.num_variants == nvar
            r = p.solve(b, None, 12, 0.0, history=True)
            c = p.solve(b, None, 500, 1e-11)
            if n == 8190 and v in (2, 3, 7, 8, 9, 10, 12):
                for nb in (2, 3, 5):  # P12a through the CTA kernel, ragged rows per CTA
                    p.set_row_blocks(nb)
                    rb = p.solve(b, None, 12, 0.0, history=True)
                    assert np.array_equal(rb.x, r.x) and np.array_equal(rb.hist, r.hist), (v, nb)
                p.set_row_blocks(1)
        assert rel_linf(r.x, x_o) <= TOL64
        if ref is None:
            ref = (r, c)
        assert np.array_equal(r.x, ref[0].x) and np.array_equal(r.hist, ref[0].hist), v
        assert (c.status, c.iters) == (ref[1].status, ref[1].iters) and np.array_equal(c.x, ref[1].x), v


# ------------------------------------------------------------------ NEXT-2: Euclidean stop rule
def test_l2_norm_parity_and_pins(jb):
    A2 = np.array([[2.0, 1.0], [1.0, 3.0]])
    b2 = np.array([3.0, 4.0])
    with jb.Plan(A2) as p:
        p.set_norm("l2")
        r = p.solve(b2, None, 1000, 1e-12, history=True)
    assert (r.status, r.iters) == (jb.CONVERGED, 33)  # closed form: d_32 = 5*6^-16 >= tol > d_33
    assert r.hist[1] == pytest.approx(5 / 6, rel=1e-12) and r.hist[0] == pytest.approx(math.sqrt(145) / 6, rel=1e-12)
    for n, scale in ((300, 1.02), (3000, 1.02), (8192, 1.05)):
        A, b, _ = dominant(n, 41 + n, scale=scale)
        st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 3000, 1e-10, nthreads=16, history=True, norm="l2")
        st_m, _, it_m = oracle.jacobi(A, b, None, 3000, 1e-10, nthreads=16, norm="max")
        with jb.Plan(A) as p:
            p.set_norm("l2")
            r = p.solve(b, None, 3000, 1e-10, history=True)
            assert (r.status, r.iters) == (st_o, it_o) and rel_linf(r.x, x_o) <= TOL64
            np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)
            if n == 8192:  # P12a with the L2 reduction: row blocks that are multiples of 256 rows
                for nb in (2, 4, 8):
                    p.set_row_blocks(nb)
                    rb = p.solve(b, None, 3000, 1e-10, history=True)
                    assert rb.iters == r.iters and np.array_equal(rb.x, r.x) and np.array_equal(rb.hist, r.hist)
                p.set_row_blocks(1)
            p.set_norm("max")
            rm = p.solve(b, None, 3000, 1e-10)
            assert rm.iters == it_m <= r.iters  # ||.||_2 >= ||.||_inf: never stops earlier
    # divergent paper regime: NaN/Inf-sticky with the L2 sum too
    rng = np.random.default_rng(14)
    A = rng.uniform(0, 1, (64, 64))
    with jb.Plan(A) as p:
        p.set_norm("l2")
        r = p.solve(rng.uniform(0, 1, 64), None, 500, 1e-8, history=True)
    assert (r.status, r.iters) == (jb.MAX_ITER, 500) and not np.isfinite(r.hist[-1])


# ------------------------------------------------------------------ distributed plan (NCCL path), one rank
def test_dist_plan_single_rank_matches_plain_plan(jb):
    """jacobi_dist_plan_create with nranks = 1 runs the captured NCCL allgather / u64 max-allreduce /
    L2 block allgather path on one GPU; it must equal the plain plan bitwise (pin P12 at P = 1)."""
    import torch
    n = 4096
    A, b, _ = dominant(n, 77, scale=1.05)
    uid = jb.nccl_unique_id()
    orc = oracle.jacobi(A, b, None, 60, 1e-11, nthreads=16, history=True)
    orc2 = oracle.jacobi(A, b, None, 60, 1e-11, nthreads=16, history=True, norm="l2")
    with jb.Plan(A) as p0:
        ref = p0.solve(b, None, 60, 1e-11, history=True)
        p0.set_norm("l2")
        ref2 = p0.solve(b, None, 60, 1e-11, history=True)
    dA = torch.from_numpy(A).cuda()
    with jb.Plan(dA, n=n, dist=(uid, 0, 1)) as p:
        inf = p.info
        assert (inf.rank, inf.nranks, inf.rows, inf.row0) == (0, 1, n, 0)
        r = p.solve(b, None, 60, 1e-11, history=True)
        match_oracle(r, orc)
        assert (r.status, r.iters) == (ref.status, ref.iters)
        assert np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist)
        p.set_norm("l2")
        r2 = p.solve(b, None, 60, 1e-11, history=True)
        match_oracle(r2, orc2)
        assert (r2.status, r2.iters) == (ref2.status, ref2.iters) and np.array_equal(r2.x, ref2.x)
        db = torch.from_numpy(b).cuda()
        ms = p.time_sweeps(db, torch.zeros(n, dtype=torch.float64, device="cuda"), 3)
        assert (ms > 0).all()
    Z = A.copy()
    Z[5, 5] = 0.0
    with pytest.raises(jb.JacobiError) as e:
        jb.Plan(Z, dist=(jb.nccl_unique_id(), 0, 1))
    assert e.value.status == jb.EZERODIAG and "i = 5" in str(e.value)


# ------------------------------------------------------------------ NEXT-3: small-n cluster-resident solver
@pytest.mark.parametrize("n,f32", [(1, False), (2, False), (37, False), (129, False), (256, False), (300, True),
                                   (511, True), (600, False), (640, False)])
def test_small_n_cluster_path_bitwise(jb, n, f32, monkeypatch):
    """The one-launch cluster solver (A in shared memory, x through DSMEM) must reproduce the sweep
    kernels bit for bit: iterates, histories, stop iterations, both norms, and > 4096-sweep runs."""
    A, b, _ = dominant(n, 5 + n, scale=1.02 if n > 1 else None, f32=f32)
    x0 = np.random.default_rng(n).uniform(-1, 1, n)
    runs = [(25, 0.0, "max"), (3000, 1e-12, "max"), (3000, 1e-12, "l2"), (4200, 0.0, "max")]
    res = {}
    monkeypatch.setenv("JACOBI_PERSIST", "0")  # cluster vs graph of sweep kernels (persistent path: own tests)
    for small in ("1", "0"):
        monkeypatch.setenv("JACOBI_SMALL_N", small)
        with jb.Plan(A) as p:
            assert (p.info.cluster_ctas > 0) == (small == "1"), p.info.cluster_ctas
            for mi, tol, norm in runs:
                p.set_norm(norm)
                res[(small, mi, tol, norm)] = p.solve(b, x0, mi, tol, history=True)
    for mi, tol, norm in runs:
        r1, r0 = res[("1", mi, tol, norm)], res[("0", mi, tol, norm)]
        assert (r1.status, r1.iters) == (r0.status, r0.iters), (mi, tol, norm)
        assert np.array_equal(r1.x, r0.x) and np.array_equal(r1.hist, r0.hist), (mi, tol, norm)
    st_o, x_o, it_o = oracle.jacobi(A, b, x0, 3000, 1e-12)
    r = res[("1", 3000, 1e-12, "max")]
    assert (r.status, r.iters) == (st_o, it_o) and rel_linf(r.x, x_o) <= TOL64


# ------------------------------------------------------------------ NEXT-4: column-wise distribution (§3.2)
def test_colwise_emulated_slabs_and_single_rank(jb):
    """Column slabs: row sums of each n x m slab from that slab's x slice, summed over
    slabs, then the epilogue.  1-GPU emulation with P slabs vs the oracle (tolerance: the slab sums
    re-associate the chunk sums), and the NCCL column-wise plan with one rank (bitwise = row-wise)."""
    import torch
    for n, scale, f32, Ps in ((4096, 1.05, False, (2, 4, 8)), (3000, 1.02, False, (3, 5)), (8192, 1.2, True, (2, 8))):
        A, b, _ = dominant(n, 91 + n, scale=scale, f32=f32)
        st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 3000, 1e-10, nthreads=16, history=True)
        with jb.Plan(A) as p:
            ref = p.solve(b, None, 3000, 1e-10, history=True)
            with pytest.raises(jb.JacobiError):
                p.set_col_blocks(7)  # 7 does not divide n into 8-aligned slabs
            for P in Ps:
                p.set_col_blocks(P)
                r = p.solve(b, None, 3000, 1e-10, history=True)
                assert (r.status, r.iters) == (st_o, it_o), (n, P)
                assert rel_linf(r.x, x_o) <= TOL64
                np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)
                p.set_norm("l2")
                rl = p.solve(b, None, 3000, 1e-10)
                p.set_norm("max")
                assert rl.iters >= r.iters and rel_linf(rl.x, x_o) <= 1e-9
            p.set_col_blocks(1)
            r1 = p.solve(b, None, 3000, 1e-10, history=True)
            assert np.array_equal(r1.x, ref.x) and np.array_equal(r1.hist, ref.hist)
        dA = torch.from_numpy(A).cuda()
        with jb.Plan(dA, n=n, dist=(jb.nccl_unique_id(), 0, 1), layout="cols") as p:
            rc = p.solve(b, None, 3000, 1e-10, history=True)
            match_oracle(rc, (st_o, x_o, it_o, h_o))
            assert (rc.status, rc.iters) == (ref.status, ref.iters)
            assert np.array_equal(rc.x, ref.x) and np.array_equal(rc.hist, ref.hist)


# ------------------------------------------------------------------ NEXT-1: fused NVLink exchange (emulated ranks)
def test_fused_exchange_emulated_ranks_bitwise(jb):
    """P ranks emulated on one GPU (per-rank x copies, slots and arrival counters; the ranks' sweep
    kernels push x_i^(k) into every copy, fold max|dx| into every slot with atomics and bump every
    counter; the next sweep waits on its own counter).  Must equal the plain plan bit for bit."""
    import torch
    for n, scale in ((8192, 1.05), (16384, 1.02)):
        A, b, _ = dominant(n, 111 + n, scale=scale)
        x0 = np.random.default_rng(n).uniform(-1, 1, n)
        orc = oracle.jacobi(A, b, x0, 40, 0.0, nthreads=16, history=True)
        orc2 = oracle.jacobi(A, b, x0, 3000, 1e-11, nthreads=16, history=True)
        with jb.Plan(A) as p:
            ref = p.solve(b, x0, 40, 0.0, history=True)
            ref2 = p.solve(b, x0, 3000, 1e-11, history=True)
        for P in (1, 2, 4, 8):
            with jb.Plan(A) as p:
                p.set_p2p_emulation(P)
                for K in (4, 32):
                    p.set_batch(K)
                    r = p.solve(b, x0, 40, 0.0, history=True)
                    match_oracle(r, orc)
                    assert r.iters == 40 and np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist), (n, P, K)
                    r2 = p.solve(b, x0, 3000, 1e-11, history=True)
                    match_oracle(r2, orc2)
                    assert (r2.status, r2.iters) == (ref2.status, ref2.iters) and np.array_equal(r2.x, ref2.x), (n, P)
                with pytest.raises(jb.JacobiError):
                    p.set_norm("l2")  # max norm only
    # the real IPC path with a single rank (own handles only)
    A, b, _ = dominant(8192, 5, scale=1.05)
    orc = oracle.jacobi(A, b, None, 3000, 1e-11, nthreads=16, history=True)
    with jb.Plan(A) as p0:
        ref = p0.solve(b, None, 3000, 1e-11, history=True)
    dA = torch.from_numpy(A).cuda()
    with jb.Plan(dA, n=8192, dist=(jb.nccl_unique_id(), 0, 1)) as p:
        p.ipc_attach(p.ipc_export())
        r = p.solve(b, None, 3000, 1e-11, history=True)
        match_oracle(r, orc)
        assert (r.status, r.iters) == (ref.status, ref.iters) and np.array_equal(r.x, ref.x)
        assert np.array_equal(r.hist, ref.hist)


def test_slabs_and_row_blocks_every_sweep_on_slow_companion(jb):
    """NEXT-4's column slabs (P = 2/4/8 slabs emulated on one GPU) and the row-block
    split (P12a) over 120 sweeps of the slow companion, far from convergence: every d_k and
    x against the oracle (slabs re-associate the chunk sums: tolerance), row blocks bitwise = P = 1."""
    n = 8192
    A, b, _ = slow_companion(n, 8193)
    x0 = np.random.default_rng(6).uniform(-1, 1, n)
    orc = oracle.jacobi(A, b, x0, 120, 0.0, nthreads=16, history=True)
    with jb.Plan(A) as p:
        ref = p.solve(b, x0, 120, 0.0, history=True)
        match_oracle(ref, orc)
        for P in (2, 4, 8):
            p.set_col_blocks(P)
            match_oracle(p.solve(b, x0, 120, 0.0, history=True), orc)
        p.set_col_blocks(1)
        for P in (2, 4, 8):
            p.set_row_blocks(P)
            r = p.solve(b, x0, 120, 0.0, history=True)
            assert np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist), P


@pytest.mark.parametrize("variant", [12, 13])
def test_slab_kernels_every_sweep_on_slow_companion(jb, monkeypatch, variant):
    """The kernels a rank's narrow column slab runs (slab_variant: the group kernel for 4-15 chunks,
    the item kernel R4 U2 with the L2 policy for 2-3), forced onto the 1-GPU slab emulation: every d_k
    and x against the oracle over 120 sweeps of the slow companion, P = 2/4/8 slabs."""
    monkeypatch.setenv("JACOBI_SWEEP_VARIANT", str(variant))
    n = 8192
    A, b, _ = slow_companion(n, 8194)
    x0 = np.random.default_rng(7).uniform(-1, 1, n)
    orc = oracle.jacobi(A, b, x0, 120, 0.0, nthreads=16, history=True)
    with jb.Plan(A) as p:
        for P in (2, 4, 8):
            p.set_col_blocks(P)
            match_oracle(p.solve(b, x0, 120, 0.0, history=True), orc)


@pytest.mark.parametrize("persist", ["0", "1"])
def test_fused_exchange_every_sweep_on_slow_companion(jb, monkeypatch, persist):
    """NEXT-1's protocol pinned per sweep: P = 2/4/8 emulated ranks pushing
    x_i^(k) into every rank's copy (graph kernels, and the persistent push solver) over 120 sweeps of the
    slow companion, far from convergence — a missed or late push leaves stale x_j^(k-1) in a rank's copy,
    an error of order d_k that decays only by 1/1.05 per sweep — every d_k and x against the oracle."""
    monkeypatch.setenv("JACOBI_PERSIST", persist)
    n = 8192
    A, b, _ = slow_companion(n, 8192)
    x0 = np.random.default_rng(5).uniform(-1, 1, n)
    orc = oracle.jacobi(A, b, x0, 120, 0.0, nthreads=16, history=True)
    assert orc[3][-1] > 1e-6  # still far from converged (d_120 ~ 1e-5)
    for P in (2, 4, 8):
        with jb.Plan(A) as p:
            p.set_p2p_emulation(P)
            assert (p.info.persistent_ctas > 0) == (persist == "1")
            r = p.solve(b, x0, 120, 0.0, history=True)
        match_oracle(r, orc)


def test_fused_exchange_silent_peer_faults_instead_of_hanging(jb, monkeypatch):
    """A rank whose kernels never signal (fault injection: virtual rank 1 of 2 is never launched)
    must not hang its peers: the next sweep's wait for the signals is bounded (JACOBI_PEER_WAIT_MS),
    the plan is marked faulted, every later sweep is a no-op and the solve returns JACOBI_ECUDA."""
    import time
    A, b, _ = dominant(8192, 17, scale=1.05)
    monkeypatch.setenv("JACOBI_PEER_WAIT_MS", "300")
    monkeypatch.setenv("JACOBI_P2P_EMUL_DROP", "1")
    with jb.Plan(A) as p:
        p.set_p2p_emulation(2)
        t0 = time.perf_counter()
        with pytest.raises(jb.JacobiError) as ei:
            p.solve(b, None, 40, 0.0)
        assert ei.value.status == jb.ECUDA and "peer" in str(ei.value)
        assert time.perf_counter() - t0 < 30.0
    monkeypatch.delenv("JACOBI_P2P_EMUL_DROP")
    with jb.Plan(A) as p:  # the device is healthy afterwards
        p.set_p2p_emulation(2)
        assert p.solve(b, None, 40, 0.0).iters == 40


# ------------------------------------------------------------------ stream ordering of borrowed inputs
def test_null_stream_plan_sees_default_stream_writes(jb):
    """A plan created with no stream reads a borrowed device A that the caller has just written on
    torch's default (legacy) stream: its own stream is a blocking one, so the generator's writes
    are complete before the setup kernels read a_ii (with a non-blocking stream this raced and
    reported EZERODIAG on rows the generator had not reached yet)."""
    import torch
    cfg = g.GenConfig(16384, diag_mode=g.DIAG_SCALE, diag_scale=1.05)
    for _ in range(3):
        dA = torch.empty((cfg.n, cfg.n), dtype=torch.float64, device="cuda")
        db = torch.empty(cfg.n, dtype=torch.float64, device="cuda")
        g.device_rows(cfg, 0, cfg.n, dA.data_ptr(), cfg.n, db.data_ptr(), 0)  # legacy default stream
        with jb.Plan(dA, n=cfg.n) as p:  # no stream, no synchronize in between
            r = p.solve(db.cpu().numpy(), None, 1, 0.0)
        d, bh = g.host_diag_b(cfg, 0, cfg.n)
        assert np.array_equal(r.x, bh / d)  # P3: sweep 1 from x0 = 0 is b / diag bitwise
        del dA, db
        torch.cuda.empty_cache()


def test_enomem_on_oversized_plan_then_healthy(jb):
    """A plan whose A cannot fit in HBM (n = 200000 fp64: 320 GB) fails with JACOBI_ENOMEM at the
    device allocation (before any copy from the host pointer), releases what it allocated, and the
    device stays usable."""
    import ctypes
    h = ctypes.c_void_p()
    dummy = np.zeros(8)
    st = jb._lib.jacobi_plan_create(ctypes.byref(h), 200000, jb.F64, dummy.ctypes.data, 200000, 0, None)
    assert st == jb.ENOMEM and "out of memory" in jb.last_error().lower() and not h.value
    A, b, _ = dominant(512, 3, scale=1.05)
    with jb.Plan(A) as p:
        assert p.solve(b, None, 10, 0.0).iters == 10


@pytest.mark.parametrize("n,seed,max_iter,tol", [(18950, 1, 6, 0.0), (20001, 2, 40, 1e-9), (24575, 3, 5, 0.0)])
def test_dynamic_tile_default_sizes_vs_oracle(jb, n, seed, max_iter, tol):
    """Ragged sizes where the default sweep kernel takes its tiles dynamically: same
    status and iteration count as the oracle, relative L-inf error <= 1e-10."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05 * rng.choice([-1.0, 1.0], n))
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-1, 1, n)
    st_o, x_o, it_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=16)
    with jb.Plan(A) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_cta R4 U2 L2-policy dynamic"
        r = p.solve(b, x0, max_iter, tol)
    assert (r.status, r.iters) == (st_o, it_o)
    assert rel_linf(r.x, x_o) <= TOL64


def test_dynamic_tile_every_sweep_on_slow_companion(jb):
    """The dynamic-tile kernel (tiles claimed from a launch-wide counter, reset once per launch) over
    150 sweeps of a system that does not converge within them (R21's slow companion, rho(T) = 1/1.05):
    a tile dropped or done twice in any sweep leaves an error of order d_k that decays only by 1/1.05 per
    sweep, so every d_k and the final x against the oracle pin every sweep — unlike
    a fast-converging system, where Jacobi heals such an error before the last iterate."""
    n = 20001
    A, b, _ = slow_companion(n, 20001)
    x0 = np.random.default_rng(3).uniform(-1, 1, n)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, 150, 0.0, nthreads=16, history=True)
    with jb.Plan(A) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_cta R4 U2 L2-policy dynamic"
        r = p.solve(b, x0, 150, 0.0, history=True)
    assert (r.status, r.iters) == (st_o, it_o) == (jb.MAX_ITER, 150)
    assert h_o[-1] > 1e-6  # still far from converged: no healing
    assert rel_linf(r.x, x_o) <= TOL64
    np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


def test_group_kernel_every_sweep_on_slow_companion(jb):
    """The same every-sweep pin for the fp32 group kernel (the c5-shard default below 512 rows per SM):
    60 sweeps of the slow companion stored in fp32, n = 33001 (ragged), still far from converged."""
    n = 33001
    A, b, _ = slow_companion(n, 33001, f32=True)
    x0 = np.random.default_rng(4).uniform(-1, 1, n)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, 60, 0.0, nthreads=16, history=True)
    with jb.Plan(A) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_group R8 G4 x-smem"
        r = p.solve(b, x0, 60, 0.0, history=True)
    assert (r.status, r.iters) == (st_o, it_o) == (jb.MAX_ITER, 60)
    assert h_o[-1] > 1e-4
    assert rel_linf(r.x, x_o) <= 1e-10  # fp32 storage, fp64 arithmetic on both sides: self-check bar
    np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("n,seed,max_iter,tol", [(33001, 4, 5, 0.0), (40000, 5, 60, 1e-9)])
def test_group_kernel_default_sizes_vs_oracle(jb, n, seed, max_iter, tol):
    """fp32 A with >= 16 column chunks and fewer than 512 rows per SM: the default is the group kernel
    (4 warps per 8-row tile, chunk sums folded in ascending order).  Ragged n (a partial
    last chunk and tile): same status and iteration count as the oracle on the same fp32 values
    (PAPER.md:59-66), relative L-inf error <= 1e-10 (both sides accumulate in fp64)."""
    rng = np.random.default_rng(seed)
    A = rng.random((n, n), dtype=np.float32)
    A *= 2
    A -= 1
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, (np.abs(A).sum(1, dtype=np.float64) * 1.05).astype(np.float32))
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-1, 1, n)
    st_o, x_o, it_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=16)
    with jb.Plan(A) as p:
        assert jb.variant_name(p.info.variant) == "k_sweep_group R8 G4 x-smem"
        r = p.solve(b, x0, max_iter, tol)
    assert (r.status, r.iters) == (st_o, it_o)
    assert rel_linf(r.x, x_o) <= TOL64


@pytest.mark.parametrize("n,f32", [(300, True), (149, False), (600, True)])
def test_group_kernel_few_rows_per_cta(jb, n, f32, monkeypatch):
    """The group kernel (variant 12) on the graph path with fewer rows per CTA than groups (n = 149 / 300:
    1-2 rows per CTA, so some of a CTA's 4 groups own no tile and the x ring counts only the others):
    bitwise equal to the row-panel kernel (variant 6) and to the item kernel, within 1e-10 of the oracle."""
    A, b, _ = dominant(n, 900 + n, scale=1.05, f32=f32)
    orc = oracle.jacobi(A, b, None, 30, 1e-11, nthreads=16, history=True)
    monkeypatch.setenv("JACOBI_SMALL_N", "0")
    monkeypatch.setenv("JACOBI_PERSIST", "0")
    out = {}
    for v in ("12", "6", "0"):
        monkeypatch.setenv("JACOBI_SWEEP_VARIANT", v)
        with jb.Plan(A) as p:
            assert p.info.variant == int(v), (v, p.info.variant)
            out[v] = p.solve(b, None, 30, 1e-11, history=True)
    match_oracle(out["12"], orc)
    for v in ("6", "0"):
        assert np.array_equal(out[v].x, out["12"].x) and np.array_equal(out[v].hist, out["12"].hist), v


def test_time_shard_hook(jb):
    """jacobi_plan_time_shard (per-GPU shard measurement): runs the three row-block modes and the column
    slab mode (NEXT-4) of a rank,
    reports the variant its plan would pick, rejects bad arguments, and leaves the plan usable (the
    next solve still matches the oracle)."""
    import torch
    n = 8192
    A, b, _ = dominant(n, 404, scale=1.05)
    dA = torch.from_numpy(A).cuda()
    db = torch.from_numpy(b).cuda()
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    with jb.Plan(dA, n=n) as p:
        for P, r in ((1, 0), (4, 3), (8, 5)):
            for mode in ("graph", "persistent", "persistent-push", "colslab"):
                ms, v = p.time_shard(db, dx0, P, r, 8, mode)
                assert 0 < ms < 50, (P, r, mode, ms)
                if mode in ("graph", "colslab"):
                    assert jb.variant_name(v).startswith("k_sweep")
        with pytest.raises(jb.JacobiError) as e:
            p.time_shard(db, dx0, 2048, 0, 8, "colslab")  # slabs of 4 columns: not a multiple of 8
        assert e.value.status == jb.EINVAL
        for bad in ((3, 0), (4, 4), (0, 0)):  # 3 does not divide 8192; rank out of range; no ranks
            with pytest.raises(jb.JacobiError) as e:
                p.time_shard(db, dx0, bad[0], bad[1], 8, "graph")
            assert e.value.status == jb.EINVAL
        with pytest.raises(jb.JacobiError):
            p.time_shard(db, dx0, 2, 0, 5000, "graph")  # more than 4096 sweeps
        orc = oracle.jacobi(A, b, None, 30, 1e-11, nthreads=16, history=True)
        match_oracle(p.solve(b, None, 30, 1e-11, history=True), orc)


def test_fused_exchange_dynamic_tiles(jb):
    """A rank with >= 32 four-row tiles per CTA runs the dynamic-tile fused-exchange kernel (variant 11):
    bitwise equal to the plain plan and matching the oracle, as one emulated rank and as the real IPC
    path with one rank; two emulated ranks of the same system take the static fused kernel (4)."""
    import torch
    n = 20480
    rng = np.random.default_rng(2048)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05)
    b = rng.uniform(-1, 1, n)
    orc = oracle.jacobi(A, b, None, 200, 1e-11, nthreads=16, history=True)
    with jb.Plan(A) as p0:
        ref = p0.solve(b, None, 200, 1e-11, history=True)
    for P, want in ((1, 11), (2, 4)):
        with jb.Plan(A) as p:
            p.set_p2p_emulation(P)
            assert p.info.variant == want, (P, p.info.variant)
            r = p.solve(b, None, 200, 1e-11, history=True)
            match_oracle(r, orc)
            assert np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist)
    dA = torch.from_numpy(A).cuda()
    with jb.Plan(dA, n=n, dist=(jb.nccl_unique_id(), 0, 1)) as p:
        p.ipc_attach(p.ipc_export())
        assert p.info.variant == 11
        r = p.solve(b, None, 200, 1e-11, history=True)
        match_oracle(r, orc)
        assert np.array_equal(r.x, ref.x)


def test_device_while_loop_matches_host_polled_batches(jb, monkeypatch):
    """The device-side while loop over graph batches (conditional graph node) and the
    host-polled batches give the same bits, statuses and iteration counts for fixed runs, tol stops
    inside and at the end of a batch, max_iter not a multiple of the batch, and both norms."""
    n = 6000
    A, b, _ = dominant(n, 909, scale=1.05)
    x0 = np.random.default_rng(9).uniform(-1, 1, n)
    runs = [(37, 0.0, "max"), (5000, 1e-10, "max"), (5000, 1e-10, "l2"), (8, 0.0, "max"), (1, 0.0, "max")]
    out = {}
    for w in ("1", "0"):
        monkeypatch.setenv("JACOBI_GRAPH_WHILE", w)
        monkeypatch.setenv("JACOBI_PERSIST", "0")
        with jb.Plan(A) as p:
            for K in (4, 8):
                p.set_batch(K)
                for mi, tol, norm in runs:
                    p.set_norm(norm)
                    out[(w, K, mi, tol, norm)] = p.solve(b, x0, mi, tol, history=True)
    for K in (4, 8):
        for mi, tol, norm in runs:
            r, q = out[("1", K, mi, tol, norm)], out[("0", K, mi, tol, norm)]
            assert (r.status, r.iters) == (q.status, q.iters), (K, mi, tol, norm)
            assert np.array_equal(r.x, q.x) and np.array_equal(r.hist, q.hist), (K, mi, tol, norm)
    orc = oracle.jacobi(A, b, x0, 5000, 1e-10, nthreads=16, history=True)
    match_oracle(out[("1", 8, 5000, 1e-10, "max")], orc)
