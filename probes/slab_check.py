import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1403_5805_b200 as jb
n = 8192
A = np.random.default_rng(1).uniform(-1, 1, (n, n)); np.fill_diagonal(A, np.abs(A).sum(1) * 1.05)
dA = torch.from_numpy(A).cuda(); db = torch.ones(n, dtype=torch.float64, device="cuda"); dx0 = torch.zeros_like(db)
jb.bounds_violations(True)
with jb.Plan(dA, n=n) as p:
    for P in (1, 2, 8, 16):
        for r in (0, P - 1):
            p.time_shard(db, dx0, P, r, 4, "colslab")
print("checked build:", jb.bounds_violations(True))
