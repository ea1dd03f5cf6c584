import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import jacobi_gen as g
import paper_1403_5805_b200 as jb
cfg = g.CONFIGS["c5"]; n = cfg.n
dA = torch.empty((n, n), dtype=torch.float32, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda"); dxo = torch.empty_like(dx0)
torch.cuda.synchronize()
for v in sys.argv[1].split(","):
    os.environ["JACOBI_SWEEP_VARIANT"] = v
    with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
        ms = p.time_sweeps(db, dx0, 30)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p.solve_device(db, dx0, dxo, 20, 0.0)
        e0.record(); r = p.solve_device(db, dx0, dxo, 100, 0.0); e1.record(); torch.cuda.synchronize()
        print(json.dumps({"v": v, "name": jb.variant_name(p.info.variant), "ts_ms": [round(x, 3) for x in ms],
                          "solve100_ms_per_sweep": e0.elapsed_time(e1) / 100}), flush=True)
