"""Per-CTA timeline of four consecutive sweeps inside the persistent grid solver (probe build:
nvcc ... -DJACOBI_SM_TIMING -> probes/libjacobi_smt.so, loaded with JACOBI_LIB).  For sweeps 21-24 of
a fixed-count solve, each CTA's start of work (after the grid barrier and stop test) and end of work
(before its barrier arrival), via %globaltimer.

python probes/grid_timeline.py [c2|n]  -> one JSON line per sweep + a summary line:
  work_us   per-CTA work time (min / median / max)
  go_spread spread of the CTAs' start times (barrier release skew)
  wait_us   per CTA, end of its work -> start of the next sweep (barrier wait incl. the slowest CTA)
  cycle_us  median start-to-start time
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = g.CONFIGS[arg] if arg in g.CONFIGS else g.GenConfig(int(arg), diag_mode=g.DIAG_SCALE, diag_scale=1.2)
n = cfg.n
dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
lib = ctypes.CDLL(jb.LIB_PATH)
os.environ["JACOBI_PERSIST"] = "1"
with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
    G = p.info.persistent_ctas
    assert G > 0
    bh = db.cpu().numpy()
    for rep in range(2):
        r = p.solve(bh, None, 40, 0.0)
        assert r.iters == 40
        buf = (ctypes.c_ulonglong * (3 * 4096))()
        assert lib.jacobi_debug_sm_times(buf, 4096) == 0
        a = np.array(buf[:], dtype=np.int64).reshape(4, 1024, 3)[:, :G, :]
        t0 = a[:, :, 1].min()
        go = (a[:, :, 1] - t0) / 1e3
        end = (a[:, :, 2] - t0) / 1e3
        work = end - go
        for s in range(4):
            line = {"n": n, "rep": rep, "sweep": 21 + s, "go_spread_us": float(go[s].max() - go[s].min()),
                    "work_us": [float(work[s].min()), float(np.median(work[s])), float(work[s].max())],
                    "end_spread_us": float(end[s].max() - end[s].min())}
            if s < 3:
                wait = go[s + 1] - end[s]
                line["wait_us"] = [float(wait.min()), float(np.median(wait)), float(wait.max())]
                line["release_after_last_end_us"] = float(go[s + 1].min() - end[s].max())
                line["cycle_us"] = float(np.median(go[s + 1] - go[s]))
            print(json.dumps(line), flush=True)
        rows = [(b + 1) * n // G - b * n // G for b in range(G)]
        print(json.dumps({"n": n, "rep": rep, "cta_rows": rows, "cta_smid": a[0, :, 0].tolist(),
                          "cta_work_us": [round(float(v), 3) for v in work.mean(0)],
                          "slowest_ctas": np.argsort(-work.mean(0))[:8].tolist(),
                          "slowest_sms": [int(a[0, i, 0]) for i in np.argsort(-work.mean(0))[:8]]}), flush=True)
