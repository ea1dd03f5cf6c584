"""Per-sweep time of chosen sweep-kernel variants over a list of n (fp64, graph path):
python probes/variant_sizes.py n1,n2,... v1,v2,..."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g
os.environ["JACOBI_PERSIST"] = "0"
import paper_1403_5805_b200 as jb
stream = torch.cuda.Stream()
for n in [int(v) for v in sys.argv[1].split(",")]:
    cfg = g.GenConfig(n, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
    dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda"); xo = torch.empty_like(dx0)
    torch.cuda.synchronize()
    for v in sys.argv[2].split(","):
        os.environ["JACOBI_SWEEP_VARIANT"] = v
        with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
            p.set_batch(20)
            p.solve_device(db, dx0, xo, 40, 0.0)
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream); p.solve_device(db, dx0, xo, 40, 0.0); e1.record(stream); e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            inf = p.info
            print(json.dumps({"n": n, "chunks": (n + inf.chunk_cols - 1) // inf.chunk_cols, "variant": jb.variant_name(inf.variant),
                              "us": 1e3 * best / 40, "gbs": inf.bytes_per_sweep * 40 / best / 1e6}), flush=True)
    del dA; torch.cuda.empty_cache()
