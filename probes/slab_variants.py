"""Column-slab (NEXT-4) emulation on one GPU: c3 as P slabs of n/P columns (slab GEMVs writing row sums
+ the column-sum epilogue) — per-sweep time by sweep-kernel variant (JACOBI_SWEEP_VARIANT, all variants
give the same bits).

python probes/slab_variants.py [P] [variants, comma-separated; '' = default]  -> one JSON line each
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else [""]
cfg = g.CONFIGS["c3"]
n = cfg.n
stream = torch.cuda.current_stream()
dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
xo = torch.empty(n, dtype=torch.float64, device="cuda")
for v in variants:
    if v:
        os.environ["JACOBI_SWEEP_VARIANT"] = v
    else:
        os.environ.pop("JACOBI_SWEEP_VARIANT", None)
    with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
        p.set_batch(20)
        p.set_col_blocks(P)
        inf = p.info
        p.solve_device(db, dx0, xo, 200, 0.0)
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            p.solve_device(db, dx0, xo, 200, 0.0)
            e1.record(stream)
            e1.synchronize()
            best = e0.elapsed_time(e1) if best is None else min(best, e0.elapsed_time(e1))
        print(json.dumps({"P": P, "variant": jb.variant_name(inf.variant), "us_per_sweep": 1e3 * best / 200,
                          "gbs": inf.bytes_per_sweep * 200 / (best * 1e-3) / 1e9}), flush=True)
