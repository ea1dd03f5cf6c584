"""Wall time of one device solve (solve_device) of c1 for a few run lengths: the fixed per-solve
overhead (prepare, launch, finalize, one synchronisation) beside the per-sweep cost."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g
import paper_1403_5805_b200 as jb
for name, runs in (("c1", ((1, 0.0), (12, 0.0), (200, 0.0), (200, 1e-12))),):
    cfg = g.CONFIGS[name]
    A, b, xs = g.host_system(cfg)
    dA = torch.from_numpy(A).cuda(); db = torch.from_numpy(b).cuda()
    dx0 = torch.zeros(cfg.n, dtype=torch.float64, device="cuda"); xo = torch.empty_like(dx0)
    s = torch.cuda.Stream()
    with jb.Plan(dA, n=cfg.n, stream=s.cuda_stream) as p:
        for mi, tol in runs:
            p.solve_device(db, dx0, xo, mi, tol)
            t0 = time.perf_counter()
            for _ in range(50):
                r = p.solve_device(db, dx0, xo, mi, tol)
            el = (time.perf_counter() - t0) / 50
            print(json.dumps({"config": name, "max_iter": mi, "tol": tol, "iters": r.iters, "solve_us": el * 1e6}))
