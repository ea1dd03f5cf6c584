"""Per-GPU sweep rate of a P-way row-block shard, measured on one GPU (exchange excluded).

A P-rank run gives every GPU the rows [r*n/P, (r+1)*n/P) of A.  jacobi_plan_time_shard times the
sweeps of exactly that block with the kernel variant, grid and L2-resident share rank r's plan would
choose (they depend on the m x n block's shape only), in three forms:
  graph            a CUDA graph of sweep kernels (the graph path: what a rank runs between NCCL calls)
  persistent       the persistent grid solver on the shard (grid barrier per sweep)
  persistent-push  the persistent fused-exchange kernel of a rank, peer set reduced to this GPU
GB/s = algorithmic bytes of the shard per sweep (m*n*s_A + 8n + 16m) / time.

python probes/shard_rates.py c3|c4|c5 [P list] [modes] [sweeps]  -> one JSON line per (P, mode)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
Ps = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["graph", "persistent-push"]
sweeps = int(sys.argv[4]) if len(sys.argv) > 4 else 40
cfg = g.CONFIGS[name]
n = cfg.n
stream = torch.cuda.Stream()
dA = torch.empty((n, n), dtype=torch.float32 if cfg.a_dtype == g.F32 else torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
esz = 4 if cfg.a_dtype == g.F32 else 8
with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
    for P in Ps:
        for mode in modes:
            try:
                ms, v = p.time_shard(db, dx0, P, 0, sweeps, mode)
            except jb.JacobiError as e:
                print(json.dumps({"config": name, "P": P, "mode": mode, "error": str(e)}), flush=True)
                continue
            m = n // P
            by = m * n * esz + 8 * n + 16 * m
            print(json.dumps({"config": name, "P": P, "rows_per_gpu": m, "mode": mode,
                              "variant": jb.variant_name(v) if v >= 0 else mode, "sweeps": sweeps,
                              "shard_us": ms * 1e3, "gbs_per_gpu": by / (ms * 1e-3) / 1e9}), flush=True)
