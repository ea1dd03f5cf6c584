"""Throughput of every BASELINE.json config on one GPU (device-resident inputs, CUDA-graph solves).

python probes/config_rates.py [c1,c2,c3,c4,c5]  -> one JSON line per run:
  c1: fixed 200 and tol 1e-12;  c2: fixed 500;  c3: tol 1e-10 (or 5000) + fixed 1000 companion;
  c4: fixed 100;  c5: tol 1e-6 (or 2000) + fixed 100 companion.
it/s = sweeps / time (CUDA events around plan_solve_device, best of 3 after a warm-up);
GB/s = algorithmic bytes per sweep (rows*n*s_A + 8n + 16 rows) * it/s.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

RUNS = {"c1": [(200, 0.0), (200, 1e-12)], "c2": [(500, 0.0)], "c3": [(5000, 1e-10), (1000, 0.0)],
        "c4": [(100, 0.0)], "c5": [(2000, 1e-6), (100, 0.0)]}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(RUNS)
stream = torch.cuda.current_stream()
for name in names:
    cfg = g.CONFIGS[name]
    n = cfg.n
    dt = torch.float32 if cfg.a_dtype == g.F32 else torch.float64
    dA = torch.empty((n, n), dtype=dt, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    xo = torch.empty(n, dtype=torch.float64, device="cuda")
    with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
        inf = p.info
        for max_iter, tol in RUNS[name]:
            p.set_batch(8 if tol > 0 else (20 if max_iter % 20 == 0 else 32))
            r = p.solve_device(db, dx0, xo, max_iter, tol)  # warm-up (graph capture)
            best = None
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = p.solve_device(db, dx0, xo, max_iter, tol)
                e1.record(stream)
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
            its = r.iters / (best * 1e-3)
            xs = g.host_xstar(cfg)
            err = float((xo.cpu() - torch.from_numpy(xs)).abs().max())
            print(json.dumps({"config": name, "n": n, "max_iter": max_iter, "tol": tol,
                              "status": jb.STATUS_NAMES[r.status], "iters": r.iters, "ms": best,
                              "it_per_s": its, "gbs": inf.bytes_per_sweep * its / 1e9,
                              "us_per_sweep": 1e3 * best / r.iters, "err_vs_xstar": err,
                              "variant": inf.variant, "chunk": inf.chunk_cols}), flush=True)
    del dA
    torch.cuda.empty_cache()
