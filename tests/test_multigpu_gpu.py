"""GPU, P >= 2 processes (one per GPU): every distributed exchange of the library against the 1-GPU
plan and the oracle (skipped when fewer than 2 GPUs are visible).

Row blocks (§3) with the NCCL allgather + max allreduce, the fused
NVLink push exchange (NEXT-1) in the graph path and in the persistent solver,
and column slabs with a reduce-scatter (NEXT-4), for P = 2 .. min(8, #GPUs), on the
c3 recipe (n = 16384, diagonal 1.05 x row abs-sum), a ragged n = 13440 (26.25 column chunks,
divisible by 2..8) and the slow companion (n = 8400, rho(T) = 1/1.05: no self-healing of a missed
exchange within the 30-sweep run, ~370 sweeps for the tol run).  Row-block results must be bitwise equal to the 1-GPU plan (pin P12(b): the
per-row summation order depends only on column indices) and match the oracle (status, iteration count,
x at relative L-inf <= 1e-10, d_k history); column slabs match the oracle within the same tolerance.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import jacobi_gen as g
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SYSTEMS = (("c3", 16384, 1.05), ("ragged", 13440, 1.05), ("slow", 8400, 0.0))  # slow: SURVEY.md Q21
RUNS = ((30, 0.0), (3000, 1e-10))


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _rel(x, ref):
    return np.max(np.abs(x - ref)) / np.max(np.abs(ref))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_multi_gpu_exchanges_vs_one_gpu_and_oracle(P, tmp_path):
    """P = 1 runs the same harness as one torchrun process on one GPU (NCCL communicator of one rank,
    IPC handles of its own buffers): it checks the launcher, the worker and the comparisons wherever
    the multi-GPU cases skip."""
    ng = _gpus()
    if ng < 1:
        pytest.skip("needs a GPU")
    if P > min(8, ng):
        pytest.skip(f"P = {P} needs {P} GPUs ({ng} visible)")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    systems = [sp for sp in SYSTEMS if sp[1] % P == 0]
    out = tmp_path / f"dist_P{P}.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "dist_worker.py"), str(out)]
    cmd += [f"{nm}:{n}:{sc}" for nm, n, sc in systems]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    res = dict(np.load(out))
    import paper_1403_5805_b200 as jb
    for name, n, scale in systems:
        if name == "slow":  # far from convergence after 30 sweeps: a missed exchange cannot self-heal
            A, b, _ = g.slow_companion(n, 7)  # tests/dist_worker.py SLOW_SEED
        else:
            cfg = g.GenConfig(n, seed=3, diag_mode=g.DIAG_SCALE, diag_scale=scale)
            A, b, _ = g.host_system(cfg)
        with jb.Plan(A) as p1:
            one = {(mi, tol): p1.solve(b, None, mi, tol, history=True) for mi, tol in RUNS}
        orc = {(mi, tol): oracle.jacobi(A, b, None, mi, tol, nthreads=16, history=True) for mi, tol in RUNS}
        for mode in ("nccl", "p2p", "p2p_persist", "cols"):
            if mode == "cols" and (n // P) % 8 != 0:
                continue
            assert f"{name}/{mode}/error" not in res, (P, name, mode, str(res.get(f"{name}/{mode}/error")))
            if mode == "p2p_persist":
                assert int(res[f"{name}/{mode}/persistent"]) > 0
            for mi, tol in RUNS:
                key = f"{name}/{mode}/{mi}/{tol:g}"
                x, (st, it), h = res[key + "/x"], res[key + "/it"], res[key + "/hist"]
                st_o, x_o, it_o, h_o = orc[(mi, tol)]
                assert (st, it) == (st_o, it_o), (P, key)
                assert _rel(x, x_o) <= 1e-10, (P, key)
                np.testing.assert_allclose(h, h_o, rtol=1e-9, atol=1e-14)
                if mode != "cols":  # P12(b): bitwise independent of the rank count
                    o = one[(mi, tol)]
                    assert (st, it) == (o.status, o.iters) and np.array_equal(x, o.x) and np.array_equal(h, o.hist), \
                        (P, key)


def test_bench_distributed_path_on_one_rank():
    """bench.py's N > 1 code path (distributed plan with the NCCL exchange as the headline, then the
    fused-exchange side leg behind its votes and watchdog) taken at N = 1 with --force-dist, on the
    small c2 workload: one JSON line, planted solution reached, a fused-exchange value."""
    import json
    if _gpus() < 1:
        pytest.skip("needs a GPU")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c2", "--force-dist", "--steps", "2",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT, env={k: v for k, v in os.environ.items()
                                                    if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and "NCCL" in d["config"]["parallelism"] and d["value"] > 0
    assert d["check"]["planted_max_abs_err"] <= 1e-12
    fx = d["fused_exchange"]
    assert "error" not in fx and fx["value"] > 0, fx
