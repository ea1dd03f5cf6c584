"""One rank of the multi-GPU parity run (launched by tests/test_multigpu_gpu.py under
torch.distributed.run, one process per GPU).  Not a test module itself.

Each rank builds its block of the system with the generator's device twin and solves it through the
C-ABI with every distributed exchange the library has:
  nccl        row blocks + NCCL allgather / max-allreduce per sweep
  p2p         row blocks + fused NVLink push exchange in the sweep kernel (NEXT-1)
  p2p_persist the same exchange inside the persistent cooperative solver (JACOBI_PERSIST=1)
  cols        column slabs + NCCL reduce-scatter (NEXT-4)
Rank 0 writes every result (x, iters, status, d_k history, or the error) to an .npz file.

python -m torch.distributed.run --nproc-per-node P tests/dist_worker.py OUT.npz name:n:scale ...
(name "slow": the slow companion of jacobi_gen, scale unused)
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402
from paper_1403_5805_b200.dist import dist_plan  # noqa: E402

RUNS = ((30, 0.0), (3000, 1e-10))
MODES = ("nccl", "p2p", "p2p_persist", "cols")


SLOW_SEED = 7  # the "slow" system: jacobi_gen.slow_companion(n, SLOW_SEED)


def block(cfg, rank, world, layout, stream, host=None):
    n = cfg.n
    row0, m = jb.partition(n, world, rank)
    db = torch.empty(m, dtype=torch.float64, device="cuda")
    if host is not None:  # a host-built system (A, b): this rank's rows or column slab
        A, b = host
        dA = torch.from_numpy(np.ascontiguousarray(A[row0:row0 + m] if layout == "rows" else A[:, row0:row0 + m]))
        db.copy_(torch.from_numpy(b[row0:row0 + m]))
        return dA.cuda(), db
    if layout == "rows":
        dA = torch.empty((m, n), dtype=torch.float64, device="cuda")
        g.device_rows(cfg, row0, row0 + m, dA.data_ptr(), n, db.data_ptr(), stream)
    else:  # the n x m column slab [row0, row0 + m) of all rows
        full = torch.empty((n, n), dtype=torch.float64, device="cuda")
        bf = torch.empty(n, dtype=torch.float64, device="cuda")
        g.device_rows(cfg, 0, n, full.data_ptr(), n, bf.data_ptr(), stream)
        torch.cuda.synchronize()
        dA = full[:, row0:row0 + m].contiguous()
        db.copy_(bf[row0:row0 + m])
        del full, bf
    torch.cuda.synchronize()
    return dA, db


def main():
    out_path, specs = sys.argv[1], sys.argv[2:]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream().cuda_stream
    res = {}
    for spec in specs:
        name, n, scale = spec.split(":")
        cfg = g.GenConfig(int(n), seed=3, diag_mode=g.DIAG_SCALE, diag_scale=float(scale))
        host = g.slow_companion(int(n), SLOW_SEED)[:2] if name == "slow" else None
        for mode in MODES:
            os.environ["JACOBI_PERSIST"] = "1" if mode == "p2p_persist" else "0"
            layout = "cols" if mode == "cols" else "rows"
            if mode == "cols" and (cfg.n // world) % 8 != 0:
                continue  # column slabs must be a multiple of 8 columns (jacobi.h)
            dA, db = block(cfg, rank, world, layout, stream, host)
            try:
                with dist_plan(dA, cfg.n, stream=stream, layout=layout, p2p=mode.startswith("p2p")) as p:
                    info = p.info
                    res[f"{name}/{mode}/persistent"] = np.array(info.persistent_ctas)
                    for max_iter, tol in RUNS:
                        r = p.solve(db.cpu().numpy(), None, max_iter, tol, history=True)
                        key = f"{name}/{mode}/{max_iter}/{tol:g}"
                        res[key + "/x"] = r.x
                        res[key + "/it"] = np.array([r.status, r.iters])
                        res[key + "/hist"] = r.hist
            except Exception as ex:  # recorded; the test reports it
                res[f"{name}/{mode}/error"] = np.array(str(ex))
            del dA, db
            torch.cuda.empty_cache()
            dist.barrier()
    if rank == 0:
        np.savez(out_path, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
