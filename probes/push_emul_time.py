import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import jacobi_gen as g
import paper_1403_5805_b200 as jb
for n in (4096, 8192):
    cfg = g.GenConfig(n, a_dtype=g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
    dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), s.cuda_stream)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda"); xo = torch.empty_like(dx0)
    with jb.Plan(dA, n=n, stream=s.cuda_stream) as p:
        p.set_p2p_emulation(2)
        p.solve_device(db, dx0, xo, 200, 0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); p.solve_device(db, dx0, xo, 200, 0.0); e1.record(s); e1.synchronize()
        print(json.dumps({"n": n, "persist": os.environ.get("JACOBI_PERSIST"), "us_per_sweep": 1e3 * e0.elapsed_time(e1) / 200, "persistent": p.info.persistent_ctas}))
