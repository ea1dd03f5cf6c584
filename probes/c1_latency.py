"""c1 (n = 256) latency probe: per-solve wall time of the cluster path vs the graph path."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

cfg = g.CONFIGS["c1"]
A, b, xs = g.host_system(cfg)
dA = torch.from_numpy(A).cuda()
db = torch.from_numpy(b).cuda()
dx0 = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
xo = torch.empty_like(dx0)
for small in ("1", "0"):
    os.environ["JACOBI_SMALL_N"] = small
    with jb.Plan(dA, n=cfg.n) as p:
        for mi, tol in ((200, 0.0), (2000, 0.0), (200, 1e-12)):
            p.solve_device(db, dx0, xo, mi, tol)
            t0 = time.perf_counter()
            reps = 20
            for _ in range(reps):
                r = p.solve_device(db, dx0, xo, mi, tol)
            el = (time.perf_counter() - t0) / reps
            print(json.dumps({"path": "cluster" if small == "1" else "graph", "cluster_ctas": p.info.cluster_ctas,
                              "max_iter": mi, "tol": tol, "iters": r.iters, "solve_us": el * 1e6,
                              "us_per_sweep": el * 1e6 / r.iters}), flush=True)
