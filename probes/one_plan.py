"""Profiling target: one plan, a few individually timed sweeps (jacobi_plan_time_sweeps).

python probes/one_plan.py N f64|f32 [sweeps] [variant]
Short enough to run under `ncu --set full -k regex:k_sweep -s 2 -c 1`.  The system is the seeded
generator's (off-diagonals U[-1,1], diag = 1.2 * rowabs) written on the device.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402

n = int(sys.argv[1])
f32 = len(sys.argv) > 2 and sys.argv[2] == "f32"
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
if len(sys.argv) > 4:
    os.environ["JACOBI_SWEEP_VARIANT"] = sys.argv[4]
import paper_1403_5805_b200 as jb  # noqa: E402

cfg = g.GenConfig(n, a_dtype=g.F32 if f32 else g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
dA = torch.empty((n, n), dtype=torch.float32 if f32 else torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
    inf = p.info
    ms = p.time_sweeps(db, dx0, sweeps)
    print(json.dumps({"n": n, "dtype": "f32" if f32 else "f64", "variant": inf.variant, "ms": list(ms),
                      "gbs_best": inf.bytes_per_sweep / min(ms) / 1e6}))
