"""GPU: the persistent grid solver (k_solve_gridsync — the sweeps of a launch in one cooperative
kernel, grid barrier between sweeps; NEXT-3 for mid-size n) against the graph-of-sweep-kernels path
and the oracle.

Each sweep runs the body of k_sweep_cta (same work split and summation order), so every iterate,
every d_k and the iteration count must be bitwise identical to the graph path (R10), and
within the north-star tolerance of the oracle (stop rule PAPER.md:61-66).
"""
import numpy as np
import pytest

import jacobi_gen as g
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def jb():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1403_5805_b200 as jb
    return jb


def dominant(n, seed, scale=None, f32=False):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    rs = np.abs(A).sum(1)
    d = rs * scale if scale else rs + rng.uniform(1, 2, n)
    np.fill_diagonal(A, d * rng.choice([-1.0, 1.0], n))
    if f32:
        A = A.astype(np.float32)
    xs = rng.uniform(-1, 1, n)
    return A, A.astype(np.float64) @ xs, xs


def solve_both(jb, monkeypatch, A, b, max_iter, tol, x0=None):
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("JACOBI_PERSIST", mode)
        with jb.Plan(A) as p:
            assert (p.info.persistent_ctas > 0) == (mode == "1"), p.info.persistent_ctas
            out[mode] = p.solve(b, x0, max_iter, tol, history=True)
    return out["1"], out["0"]


def rel_linf(x, ref):
    den = np.max(np.abs(ref))
    err = np.max(np.abs(np.asarray(x) - ref))
    return err / den if den > 0 else err


def match_oracle(r, orc, tol=1e-10):
    """Status, iteration count, x (relative L-inf <= 1e-10) and the d_k history against the oracle."""
    st_o, x_o, it_o, h_o = orc
    assert (r.status, r.iters) == (st_o, it_o), (r.status, r.iters, st_o, it_o)
    assert rel_linf(r.x, x_o) <= tol
    if r.hist is not None:
        np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


def same(r, q):
    return ((r.status, r.iters) == (q.status, q.iters) and np.array_equal(r.x, q.x)
            and np.array_equal(r.hist, q.hist, equal_nan=True))


# several tiles per CTA with a ragged last tile; a ragged column tail; fewer than 8 rows per CTA;
# fewer and more than 16 column chunks; fp32 A storage.
@pytest.mark.parametrize("n,f32", [(700, False), (1000, False), (3001, False), (4096, False), (9000, False),
                                   (2049, True), (5003, True)])
def test_gridsync_bitwise_vs_graph_and_oracle(jb, monkeypatch, n, f32):
    A, b, xs = dominant(n, 7 + n, scale=1.05, f32=f32)
    r, q = solve_both(jb, monkeypatch, A, b, 25, 0.0)
    assert same(r, q)
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, None, 25, 0.0, nthreads=16, history=True)
    assert r.iters == it_o == 25
    assert np.max(np.abs(r.x - x_o)) / np.max(np.abs(x_o)) <= 1e-10
    np.testing.assert_allclose(r.hist, h_o, rtol=1e-9, atol=1e-14)


@pytest.mark.parametrize("n", [1000, 4096, 6000])
def test_gridsync_fixed_count_without_history(jb, monkeypatch, n):
    """Fixed-count runs without a history skip the distance read between sweeps in every CTA (tol = 0
    never satisfies d_k < tol): the iterates must not change — bitwise equal to the graph
    path, and to the same run with a history (which CTA 0 records)."""
    A, b, _ = dominant(n, 17 + n, scale=1.05)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("JACOBI_PERSIST", mode)
        with jb.Plan(A) as p:
            assert (p.info.persistent_ctas > 0) == (mode == "1")
            out[mode] = (p.solve(b, None, 60, 0.0), p.solve(b, None, 60, 0.0, history=True))
    for r in out["1"] + out["0"]:
        assert (r.status, r.iters) == (jb.MAX_ITER, 60)
        assert np.array_equal(r.x, out["0"][0].x)
    assert np.array_equal(out["1"][1].hist, out["0"][1].hist)


def test_gridsync_c2_config(jb, monkeypatch):
    """BASELINE.json configs[1]: n = 4096, fixed 500 iterations (the default path for c2)."""
    A, b, xs = g.host_system(g.CONFIGS["c2"])
    r, q = solve_both(jb, monkeypatch, A, b, 500, 0.0)
    assert same(r, q) and (r.status, r.iters) == (jb.MAX_ITER, 500)
    assert np.max(np.abs(r.x - xs)) <= 1e-12  # P8 planted solution


def test_gridsync_stop_rule_segments_split(jb, monkeypatch):
    """tol stop inside a launch (strict <), max_iter exhausted across several
    kMaxSweepsPerLaunch = 4096-sweep launches, max_iter = 1 (P3), split runs (P11), determinism (P13)."""
    A, b, _ = dominant(2048, 11, scale=1.05)
    r, q = solve_both(jb, monkeypatch, A, b, 5000, 1e-11)
    assert same(r, q) and r.status == jb.CONVERGED
    st_o, x_o, it_o = oracle.jacobi(A, b, None, 5000, 1e-11, nthreads=16)
    assert (r.status, r.iters) == (st_o, it_o)
    r, q = solve_both(jb, monkeypatch, A, b, 9000, 0.0)  # three launches: 4096 + 4096 + 808
    assert same(r, q) and r.iters == 9000
    r, q = solve_both(jb, monkeypatch, A, b, 1, 0.0)
    assert same(r, q) and np.array_equal(r.x, b / np.diag(A))
    monkeypatch.setenv("JACOBI_PERSIST", "1")
    with jb.Plan(A) as p:
        assert p.info.persistent_ctas > 0
        r12 = p.solve(b, None, 12, 0.0)
        r5 = p.solve(b, None, 5, 0.0)
        r7 = p.solve(b, r5.x, 7, 0.0)
        assert np.array_equal(r12.x, r7.x)
        assert np.array_equal(p.solve(b, None, 12, 0.0).x, r12.x)
        p.set_norm("l2")  # the Euclidean rule runs in the persistent solver too (m <= 16384)
        assert p.info.persistent_ctas > 0
        p.set_norm("max")
        p.set_row_blocks(4)  # P12a emulation runs on the graph path, same bits
        assert p.info.persistent_ctas == 0 and np.array_equal(p.solve(b, None, 12, 0.0).x, r12.x)


def test_gridsync_nan_sticky(jb, monkeypatch):
    """The paper's raw regime (A, b ~ U[0,1]) diverges: max|dx| becomes NaN and stays
    NaN, nothing converges, both paths run to max_iter with the same NaN pattern."""
    rng = np.random.default_rng(3)
    n = 1024
    A = rng.uniform(0, 1, (n, n))
    b = rng.uniform(0, 1, n)
    r, q = solve_both(jb, monkeypatch, A, b, 300, 1e-6)
    assert (r.status, r.iters) == (q.status, q.iters) == (jb.MAX_ITER, 300)
    assert np.array_equal(np.isnan(r.x), np.isnan(q.x))
    assert np.array_equal(r.hist, q.hist, equal_nan=True)


def test_gridsync_device_borrowed(jb, monkeypatch):
    """Borrowed device A and device solve, as bench.py and the size sweep use the path."""
    import torch
    A, b, _ = dominant(3000, 21, scale=1.05)
    monkeypatch.setenv("JACOBI_PERSIST", "1")
    dA = torch.from_numpy(A).cuda()
    db = torch.from_numpy(b).cuda()
    dx0 = torch.zeros(3000, dtype=torch.float64, device="cuda")
    xo = torch.empty_like(dx0)
    with jb.Plan(dA, n=3000) as p:
        assert p.info.persistent_ctas > 0
        r = p.solve_device(db, dx0, xo, 60, 0.0)
    monkeypatch.setenv("JACOBI_PERSIST", "0")
    with jb.Plan(A) as p:
        q = p.solve(b, None, 60, 0.0)
    assert r.iters == q.iters == 60 and np.array_equal(xo.cpu().numpy(), q.x)


@pytest.mark.parametrize("n,f32", [(2048, False), (4096, False), (6144, False), (16384, False), (40000, False),
                                   (8192, True)])
def test_l2_keep_share_rule(jb, n, f32, monkeypatch):
    """L2-resident share of A: per mille of the block's work units kept with evict_last =
    floor(1000 x budget x L2 / A bytes), capped at 1000 (A within the budget is kept whole) and 0 below
    20 (less than 2 % is not worth it); budget = 0.55 of the L2, JACOBI_L2_BUDGET / JACOBI_L2_KEEP override.
    The same rule gives a rank's share from its m x n block (jacobi_plan_time_shard)."""
    import torch
    monkeypatch.delenv("JACOBI_L2_KEEP", raising=False)
    monkeypatch.delenv("JACOBI_L2_BUDGET", raising=False)
    L2 = torch.cuda.get_device_properties(0).L2_cache_size
    dA = torch.eye(n, dtype=torch.float32 if f32 else torch.float64, device="cuda") * 2.0
    a_bytes = n * n * (4 if f32 else 8)
    want = min(1000, int(1000 * 0.55 * L2 / a_bytes))
    want = 0 if want < 20 else want
    with jb.Plan(dA, n=n) as p:
        assert p.info.l2_keep_permille == want, (n, p.info.l2_keep_permille, want)
    monkeypatch.setenv("JACOBI_L2_BUDGET", "0.25")
    with jb.Plan(dA, n=n) as p:
        w = min(1000, int(1000 * 0.25 * L2 / a_bytes))
        assert p.info.l2_keep_permille == (0 if w < 20 else w)
    monkeypatch.setenv("JACOBI_L2_KEEP", "333")
    with jb.Plan(dA, n=n) as p:
        assert p.info.l2_keep_permille == 333


@pytest.mark.parametrize("n,f32,path", [(256, False, "cluster"), (512, False, "cluster"), (600, False, "grid"),
                                        (512, True, "cluster"), (576, True, "grid"), (600, True, "grid"), (3072, False, "grid"),
                                        (4096, False, "grid"), (8192, False, "graph")])
def test_default_path_by_size(jb, n, f32, path, monkeypatch):
    """Default solver path by size (measured crossovers): the cluster solver for small n,
    the persistent grid solver for mid-size A, the graph of sweep kernels beyond; the Euclidean rule
    keeps the persistent solver up to 16384 rows."""
    monkeypatch.delenv("JACOBI_PERSIST", raising=False)
    monkeypatch.delenv("JACOBI_SMALL_N", raising=False)
    A = np.eye(n, dtype=np.float32 if f32 else np.float64) * 2.0
    with jb.Plan(A) as p:
        inf = p.info
        got = "cluster" if inf.cluster_ctas else ("grid" if inf.persistent_ctas else "graph")
        assert got == path, (n, f32, got)
        p.set_norm("l2")
        assert (p.info.persistent_ctas > 0) == (path == "grid")


@pytest.mark.parametrize("n", [256, 1000, 8192])  # cluster, persistent and graph paths
def test_device_solve_x_out_aliases_x0(jb, n, monkeypatch):
    """include/jacobi.h: x_out may alias x0 (inputs are copied in before any write), on every path;
    and x_out is untouched when the solve fails (non-finite b -> ENONFINITE)."""
    import torch
    monkeypatch.delenv("JACOBI_PERSIST", raising=False)
    A, b, _ = dominant(n, 41 + n, scale=1.05)
    dA = torch.from_numpy(A).cuda()
    db = torch.from_numpy(b).cuda()
    x0 = np.random.default_rng(n).uniform(-1, 1, n)
    with jb.Plan(dA, n=n) as p:
        ref_x = torch.empty(n, dtype=torch.float64, device="cuda")
        r = p.solve_device(db, torch.from_numpy(x0).cuda(), ref_x, 30, 0.0)
        io = torch.from_numpy(x0).cuda()
        q = p.solve_device(db, io, io, 30, 0.0)  # x_out is x0
        assert (q.status, q.iters) == (r.status, r.iters) and torch.equal(io, ref_x)
        bad = db.clone()
        bad[n // 2] = float("nan")
        keep = io.clone()
        with pytest.raises(jb.JacobiError) as ei:
            p.solve_device(bad, io, io, 30, 0.0)
        assert ei.value.status == jb.ENONFINITE and torch.equal(io, keep)


@pytest.mark.parametrize("n,f32", [(700, False), (4096, False), (3001, True)])
def test_gridsync_euclidean_rule_bitwise(jb, monkeypatch, n, f32):
    """The paper's Euclidean stop rule in the persistent solver: every CTA reduces all
    rows' dx^2 in the order of k_l2_partials/k_l2_final, so histories, stop iterations and iterates
    equal the graph path's bit for bit, and the stop iteration matches the oracle's Euclidean rule."""
    A, b, _ = dominant(n, 3 + n, scale=1.05, f32=f32)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("JACOBI_PERSIST", mode)
        with jb.Plan(A) as p:
            p.set_norm("l2")
            assert (p.info.persistent_ctas > 0) == (mode == "1")
            out[mode] = (p.solve(b, None, 40, 0.0, history=True), p.solve(b, None, 5000, 1e-11, history=True))
    for r, q in zip(out["1"], out["0"]):
        assert same(r, q)
    st_o, x_o, it_o = oracle.jacobi(A, b, None, 5000, 1e-11, nthreads=16, norm="l2")
    assert (out["1"][1].status, out["1"][1].iters) == (st_o, it_o)


def test_persistent_fused_exchange_emulated_ranks_bitwise(jb, monkeypatch):
    """NEXT-1 x NEXT-3: the persistent solver over P ranks with the fused exchange (each rank's CTAs
    push x_i^(k) into every rank's x copy, fold max|dx| into every rank's slot, bump every rank's
    counter; the next sweep waits on its own counter), emulated as P CTA groups of one cooperative
    launch, must equal the plain plan bit for bit — fixed runs, tol stops, runs over several launch
    segments — and so must the real IPC path with one rank."""
    import torch
    monkeypatch.setenv("JACOBI_PERSIST", "1")
    for n, scale in ((8192, 1.05), (4096, 1.02)):  # >= 16 column chunks (the fused-exchange plans need it)
        A, b, _ = dominant(n, 211 + n, scale=scale)
        x0 = np.random.default_rng(n).uniform(-1, 1, n)
        orc = oracle.jacobi(A, b, x0, 40, 0.0, nthreads=16, history=True)
        orc2 = oracle.jacobi(A, b, x0, 3000, 1e-11, nthreads=16, history=True)
        monkeypatch.setenv("JACOBI_PERSIST", "0")
        with jb.Plan(A) as p:
            ref = p.solve(b, x0, 40, 0.0, history=True)
            ref2 = p.solve(b, x0, 3000, 1e-11, history=True)
            ref3 = p.solve(b, x0, 4200, 0.0)
        monkeypatch.setenv("JACOBI_PERSIST", "1")
        for P in (1, 2, 4, 8):
            with jb.Plan(A) as p:
                p.set_p2p_emulation(P)
                assert p.info.persistent_ctas > 0
                r = p.solve(b, x0, 40, 0.0, history=True)
                match_oracle(r, orc)
                assert r.iters == 40 and np.array_equal(r.x, ref.x) and np.array_equal(r.hist, ref.hist), (n, P)
                r2 = p.solve(b, x0, 3000, 1e-11, history=True)
                match_oracle(r2, orc2)
                assert (r2.status, r2.iters) == (ref2.status, ref2.iters) and np.array_equal(r2.x, ref2.x), (n, P)
                assert np.array_equal(r2.hist, ref2.hist)
                if P in (1, 8):
                    r3 = p.solve(b, x0, 4200, 0.0)  # two launch segments
                    assert r3.iters == 4200 and np.array_equal(r3.x, ref3.x), (n, P)
    A, b, _ = dominant(8192, 5, scale=1.05)
    orc = oracle.jacobi(A, b, None, 3000, 1e-11, nthreads=16, history=True)
    monkeypatch.setenv("JACOBI_PERSIST", "0")
    with jb.Plan(A) as p0:
        ref = p0.solve(b, None, 3000, 1e-11, history=True)
    monkeypatch.setenv("JACOBI_PERSIST", "1")
    dA = torch.from_numpy(A).cuda()
    with jb.Plan(dA, n=8192, dist=(jb.nccl_unique_id(), 0, 1)) as p:
        p.ipc_attach(p.ipc_export())
        assert p.info.persistent_ctas > 0
        r = p.solve(b, None, 3000, 1e-11, history=True)
        match_oracle(r, orc)
        assert (r.status, r.iters) == (ref.status, ref.iters) and np.array_equal(r.x, ref.x)
        assert np.array_equal(r.hist, ref.hist)


def test_distinct_plans_on_distinct_threads(jb, monkeypatch):
    """include/jacobi.h threading rule: distinct plans may run concurrently on distinct host threads
    (each on its own stream).  Two plans on different paths (cluster, persistent, graph) solved from
    three threads at once give the same bits as solved alone."""
    import threading
    monkeypatch.delenv("JACOBI_PERSIST", raising=False)
    systems = [dominant(n, 500 + n, scale=1.05) for n in (256, 2048, 8192)]
    alone = []
    for A, b, _ in systems:
        with jb.Plan(A) as p:
            alone.append(p.solve(b, None, 60, 0.0).x)
    plans = [jb.Plan(A) for A, _, _ in systems]
    out = [None] * len(systems)
    errs = []

    def run(i):
        try:
            for _ in range(3):
                out[i] = plans[i].solve(systems[i][1], None, 60, 0.0).x
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(systems))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for p in plans:
        p.close()
    assert not errs, errs
    for i in range(len(systems)):
        assert np.array_equal(out[i], alone[i]), i


def test_dynamic_tile_plans_concurrently(jb, monkeypatch):
    """Dynamic tile assignment (variant 10; DESIGN.md §6 tail paragraph): each plan owns its tile
    counters, so two plans claiming tiles at once on different streams give the bits each gives
    alone, and the counters reset themselves between launches (many sweeps, several solves)."""
    import threading
    monkeypatch.delenv("JACOBI_PERSIST", raising=False)
    monkeypatch.setenv("JACOBI_PERSIST", "0")
    monkeypatch.setenv("JACOBI_SWEEP_VARIANT", "10")
    systems = [dominant(n, 700 + n, scale=1.05) for n in (4096, 6000)]
    alone = []
    for A, b, _ in systems:
        with jb.Plan(A) as p:
            assert jb.variant_name(p.info.variant) == "k_sweep_cta R4 U2 L2-policy dynamic"
            alone.append(p.solve(b, None, 45, 0.0).x)
    monkeypatch.delenv("JACOBI_SWEEP_VARIANT")
    with jb.Plan(systems[0][0]) as p:  # the static default of this size: same bits
        assert np.array_equal(p.solve(systems[0][1], None, 45, 0.0).x, alone[0])
    monkeypatch.setenv("JACOBI_SWEEP_VARIANT", "10")
    plans = [jb.Plan(A) for A, _, _ in systems]
    out, errs = [None] * len(systems), []

    def run(i):
        try:
            for _ in range(3):
                out[i] = plans[i].solve(systems[i][1], None, 45, 0.0).x
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(systems))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for p in plans:
        p.close()
    assert not errs, errs
    for i in range(len(systems)):
        assert np.array_equal(out[i], alone[i]), i
