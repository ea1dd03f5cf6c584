"""One P-way row-block shard timed alone: the sweep kernels of rows [0, n/P) of config c3/c4/c5.

python probes/shard_once.py c3 8 [sweeps]  -> one JSON line (per-launch event times of the shard
kernel only: jacobi_plan_set_row_blocks(P) launches the P shards; the ncu launch list of this
command gives each launch's device time without the host gaps between launches).
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
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
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
    p.set_row_blocks(P)
    ms = p.time_sweeps(db, dx0, sweeps)
    per = float(np.median(ms[1:])) / P
    m = n // P
    by = m * n * esz + 8 * n + 16 * m
    print(json.dumps({"config": name, "P": P, "variant": jb.variant_name(p.info.variant), "shard_us": per * 1e3,
                      "gbs": by / (per * 1e-3) / 1e9}), flush=True)
