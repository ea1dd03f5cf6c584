"""Per-GPU sweep-kernel rate of a P-way row-block shard, measured on one GPU.

A P-rank run gives every GPU the rows [r*n/P, (r+1)*n/P) of A.  With jacobi_plan_set_row_blocks(P) a
single-GPU plan launches exactly those P shard kernels one after another (same rows per CTA, same
grid, same kernel as rank r would run; bitwise-identical results, test P12a), so the per-shard kernel
time is (time of the P launches) / P.  The exchange (NCCL allgather + max allreduce, or the fused
NVLink push) is NOT included: this isolates the compute side of the strong-scaling runs.

python probes/shard_rates.py c3|c4 [variants]   -> one JSON line per (P, variant)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
variants = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [None]
cfg = g.CONFIGS[name]
n = cfg.n
stream = torch.cuda.Stream()
dA = torch.empty((n, n), dtype=torch.float32 if cfg.a_dtype == g.F32 else torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
esz = 4 if cfg.a_dtype == g.F32 else 8
for v in variants:
    if v is None:
        os.environ.pop("JACOBI_SWEEP_VARIANT", None)
    else:
        os.environ["JACOBI_SWEEP_VARIANT"] = str(v)
    with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
        for P in (1, 2, 4, 8):
            p.set_row_blocks(P)
            ms = p.time_sweeps(db, dx0, 12)
            per = float(np.median(ms[2:])) / P
            m = n // P
            bytes_shard = m * n * esz + 8 * n + 16 * m
            inf = p.info
            print(json.dumps({"config": name, "P": P, "rows_per_gpu": m, "variant": jb.variant_name(inf.variant),
                              "shard_kernel_us": per * 1e3, "gbs_per_gpu": bytes_shard / (per * 1e-3) / 1e9,
                              "projected_it_s_kernel_only": 1e3 / per}), flush=True)
