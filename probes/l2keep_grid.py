"""L2 residency of the persistent grid solver vs the kept share of A (JACOBI_L2_KEEP, per mille).

python probes/l2keep_grid.py n keep1,keep2,... [sweeps]   -> one JSON line per keep value
One process, one plan per keep value (the library reads JACOBI_L2_KEEP at plan creation), so a single
`ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum ... -k
regex:gridsync` run captures every setting.  System: the seeded generator (diag = 1.2 x row abs-sum).
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

n = int(sys.argv[1])
keeps = [int(v) for v in sys.argv[2].split(",")]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
stream = torch.cuda.Stream()
cfg = g.GenConfig(n, a_dtype=g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
xo = torch.empty(n, dtype=torch.float64, device="cuda")
for keep in keeps:
    os.environ["JACOBI_L2_KEEP"] = str(keep)
    with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
        p.solve_device(db, dx0, xo, sweeps, 0.0)  # warm
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.solve_device(db, dx0, xo, sweeps, 0.0)
        e1.record(stream)
        e1.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / sweeps
        print(json.dumps({"n": n, "keep": keep, "us_per_sweep": round(us, 3),
                          "persistent": p.info.persistent_ctas}), flush=True)
