import os, sys
import torch
sys.path.insert(0, os.getcwd())
import jacobi_gen as g
import paper_1403_5805_b200 as jb
cfg = g.CONFIGS["c1"]
A, b, xs = g.host_system(cfg)
dA = torch.from_numpy(A).cuda(); db = torch.from_numpy(b).cuda()
dx0 = torch.zeros(cfg.n, dtype=torch.float64, device="cuda"); xo = torch.empty_like(dx0)
s = torch.cuda.Stream()
with jb.Plan(dA, n=cfg.n, stream=s.cuda_stream) as p:
    for mi in (1, 1, 12, 12, 200):
        r = p.solve_device(db, dx0, xo, mi, 0.0)
