"""Tuning probe: time every sweep-kernel variant (JACOBI_SWEEP_VARIANT) on a workload and check that
all variants produce bitwise-identical iterates (the summation order does not depend on R/U/grid).

python probes/sweep_variants.py [c4|c5|c2|c3] [sweeps]   -> one JSON line per variant
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
variants = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else list(range(11))
cfg = g.CONFIGS[name]
n = cfg.n
dt = torch.float32 if cfg.a_dtype == g.F32 else torch.float64
pad = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # row pitch padding (elements) experiment
dA_full = torch.empty((n, n + pad), dtype=dt, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA_full.data_ptr(), n + pad, db.data_ptr(), 0)
dA = dA_full[:, :n]
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
xo = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
ref = None
for v in variants:
    os.environ["JACOBI_SWEEP_VARIANT"] = str(v)
    with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
        inf = p.info
        ms = p.time_sweeps(db, dx0, sweeps)
        p.solve_device(db, dx0, xo, 3, 0.0)
        x3 = xo.cpu().numpy()
        # sustained: a 100-sweep graph solve (5 batches of 20) timed with events, after a warm-up solve
        p.set_batch(20)
        p.solve_device(db, dx0, xo, 100, 0.0)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        p.solve_device(db, dx0, xo, 100, 0.0)
        e1.record(st)
        e1.synchronize()
        sus_ms = e0.elapsed_time(e1) / 100
        xo.copy_(torch.from_numpy(x3))
        x = x3
        same = True if ref is None else bool(np.array_equal(x, ref))
        if ref is None:
            ref = x
        med = float(np.median(ms[1:]))
        print(json.dumps({"workload": name, "variant": inf.variant, "requested": v, "R": inf.rows_per_warp, "threads": inf.threads_per_cta,
                          "grid": inf.grid_ctas, "chunk": inf.chunk_cols, "lda": inf.lda, "median_ms": med, "min_ms": float(ms[1:].min()),
                          "gbs": inf.bytes_per_sweep / (med * 1e-3) / 1e9, "sustained_ms": sus_ms,
                          "sustained_gbs": inf.bytes_per_sweep / (sus_ms * 1e-3) / 1e9, "bitwise_equal_v0": same}), flush=True)
