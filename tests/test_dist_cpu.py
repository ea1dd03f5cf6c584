"""Multi-process (world_size 2, gloo, CPU) checks of the N > 1 path's host logic.

1. paper_1403_5805_b200.dist.bootstrap: every rank gets the same NCCL unique id and its row block
   (PAPER.md:72), and an indivisible n fails identically on every rank.
2. The exchange protocol of the distributed sweep, run with the oracle as the
   per-rank compute: rank r updates rows [r*m, (r+1)*m) (oracle.sweep_rows), the new
   slices are allgathered, and d_k is the max-allreduce of the u64 bit pattern of max|dx| (sign
   cleared; NaN-sticky).  The result must equal the single-process oracle bitwise, including the
   stop iteration — the property (pin P12) the CUDA plan relies on.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits_max(local_dx):
    u = local_dx.view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)
    return int(u.max()) if u.size else 0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1403_5805_b200 as jb
        from paper_1403_5805_b200.dist import bootstrap

        out = {}
        uid, r, w, row0, rows = bootstrap(96)
        out["uid"] = uid
        out["part"] = (r, w, row0, rows)
        try:
            bootstrap(97)
            out["indiv"] = None
        except jb.JacobiError as e:
            out["indiv"] = e.status

        # the library's distributed plan entry points, world_size 2 (no GPU here): argument validation
        # before any CUDA call, EINDIVISIBLE on every rank, and ECUDA — never a CPU fallback — once the
        # arguments are valid (paper_1403_5805_b200.dist.dist_plan -> jacobi_dist_plan_create)
        import ctypes
        from paper_1403_5805_b200.dist import dist_plan
        blk = np.eye(96)[row0:row0 + rows] * 2.0
        try:
            dist_plan(np.zeros((rows + 1, 96)), 96)
            out["shape"] = None
        except ValueError as e:
            out["shape"] = "ValueError" if "rows" in str(e) else str(e)
        try:
            dist_plan(np.eye(97)[:48], 97)
            out["dp_indiv"] = None
        except jb.JacobiError as e:
            out["dp_indiv"] = e.status
        try:
            dist_plan(blk, 96)
            out["dp_nogpu"] = None
        except jb.JacobiError as e:
            out["dp_nogpu"] = e.status
        h = ctypes.c_void_p()
        ub = ctypes.create_string_buffer(bytes(uid), 128)
        out["einval"] = [
            jb._lib.jacobi_dist_plan_create(ctypes.byref(h), ub, 2, 2, 96, jb.F64, blk.ctypes.data, 96, 0, None),
            jb._lib.jacobi_dist_plan_create(ctypes.byref(h), None, r, w, 96, jb.F64, blk.ctypes.data, 96, 0, None),
            jb._lib.jacobi_dist_plan_create(ctypes.byref(h), ub, r, w, 96, 7, blk.ctypes.data, 96, 0, None),
            jb._lib.jacobi_dist_plan_create(ctypes.byref(h), ub, r, w, 96, jb.F64, blk.ctypes.data, 95, 0, None),
            jb._lib.jacobi_dist_plan_create_colwise(ctypes.byref(h), ub, r, w, 100, jb.F64, blk.ctypes.data, 100, 0,
                                                    None),
        ]

        # distributed Jacobi protocol with the oracle as the per-rank compute
        rng = np.random.default_rng(5)
        n = 96
        A = rng.uniform(-1, 1, (n, n))
        np.fill_diagonal(A, 0)
        np.fill_diagonal(A, np.abs(A).sum(1) * 1.05)
        b = rng.uniform(-1, 1, n)
        x = np.zeros(n)
        hist = []
        for k in range(1, 500):
            xn_local = oracle.sweep_rows(A[row0:row0 + rows], row0, b[row0:row0 + rows], x)
            d_local = _bits_max(np.abs(xn_local - x[row0:row0 + rows]))
            gathered = [torch.empty(rows, dtype=torch.float64) for _ in range(w)]
            dist.all_gather(gathered, torch.from_numpy(xn_local))
            d = torch.tensor([d_local], dtype=torch.int64)  # bit patterns < 2^63: int64 max == u64 max
            dist.all_reduce(d, op=dist.ReduceOp.MAX)
            x = torch.cat(gathered).numpy().copy()
            dk = np.array([d.item()], dtype=np.uint64).view(np.float64)[0]
            hist.append(dk)
            if dk < 1e-12:
                break
        out["x"], out["k"], out["hist"] = x, k, np.array(hist)

        # column-wise protocol (jacobi_dist_plan_create_colwise): rank r keeps only
        # its x slice; row sums of its n x m column slab for ALL rows, reduce-scatter (sum) -> its rows
        c0, c1 = row0, row0 + rows
        xs_own = np.zeros(rows)
        for kc in range(1, 500):
            xfull = np.zeros(n)
            xfull[c0:c1] = xs_own  # only the own slice is ever read below
            slab = A[:, c0:c1].copy()
            idx = np.arange(c0, c1)
            slab[idx, idx - c0] = 0.0  # j != i
            part = torch.from_numpy(slab @ xfull[c0:c1])
            dist.all_reduce(part)  # sum; each rank keeps its rows = reduce-scatter
            s_own = part.numpy()[c0:c1]
            xn_own = (b[c0:c1] - s_own) / np.diag(A)[c0:c1]
            d = torch.tensor([_bits_max(np.abs(xn_own - xs_own))], dtype=torch.int64)
            dist.all_reduce(d, op=dist.ReduceOp.MAX)
            xs_own = xn_own
            if np.array([d.item()], dtype=np.uint64).view(np.float64)[0] < 1e-12:
                break
        gathered = [torch.empty(rows, dtype=torch.float64) for _ in range(w)]
        dist.all_gather(gathered, torch.from_numpy(xs_own))
        out["xc"], out["kc"] = torch.cat(gathered).numpy().copy(), kc
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_bootstrap_uid_and_partition(results):
    import paper_1403_5805_b200 as jb
    assert results[0]["uid"] == results[1]["uid"] and len(results[0]["uid"]) == 128
    assert results[0]["part"] == (0, 2, 0, 48) and results[1]["part"] == (1, 2, 48, 48)
    assert results[0]["indiv"] == results[1]["indiv"] == jb.EINDIVISIBLE


def test_library_dist_plan_validation_world2(results):
    """jacobi_dist_plan_create through the binding on 2 gloo ranks without a GPU: a wrong block shape is
    refused by the binding, P not dividing n is EINDIVISIBLE on both ranks, bad arguments
    are EINVAL before any CUDA call, and valid arguments end in ECUDA (there is no CPU fallback)."""
    import paper_1403_5805_b200 as jb
    for r in (0, 1):
        o = results[r]
        assert o["shape"] == "ValueError"
        assert o["dp_indiv"] == jb.EINDIVISIBLE
        assert o["dp_nogpu"] == jb.ECUDA
        # rank out of range, NULL uid, bad dtype, lda < n -> EINVAL; column slabs of 50 columns -> EINVAL
        # (a multiple of 8 is required), or EINDIVISIBLE first when P does not divide n
        assert o["einval"][:4] == [jb.EINVAL] * 4
        assert o["einval"][4] == jb.EINVAL


def test_exchange_protocol_matches_serial_oracle_bitwise(results):
    import oracle
    rng = np.random.default_rng(5)
    n = 96
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05)
    b = rng.uniform(-1, 1, n)
    st, x, it, h = oracle.jacobi(A, b, None, 499, 1e-12, history=True)
    for r in (0, 1):
        assert results[r]["k"] == it
        assert np.array_equal(results[r]["x"], x)
        assert np.array_equal(results[r]["hist"], h)


def test_colwise_protocol_matches_serial_oracle(results):
    """Column-wise exchange: the reduce-scatter of slab row sums plus the owned-slice update is the
    Jacobi sweep (within rounding: the slab sums re-associate the row sum), same stop iteration."""
    import oracle
    rng = np.random.default_rng(5)
    n = 96
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05)
    b = rng.uniform(-1, 1, n)
    st, x, it = oracle.jacobi(A, b, None, 499, 1e-12)
    for r in (0, 1):
        assert results[r]["kc"] == it
        assert np.max(np.abs(results[r]["xc"] - x)) <= 1e-12 * np.max(np.abs(x))
