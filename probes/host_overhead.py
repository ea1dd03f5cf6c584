"""Host-side cost of a small device solve (c1): ctypes call, launch, state read-back, synchronisation.

python probes/host_overhead.py -> one JSON line per measurement (µs per call, mean of 200)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

cfg = g.CONFIGS["c1"]
A, b, xs = g.host_system(cfg)
dA = torch.from_numpy(A).cuda()
db = torch.from_numpy(b).cuda()
dx0 = torch.zeros(cfg.n, dtype=torch.float64, device="cuda")
xo = torch.empty_like(dx0)
s = torch.cuda.Stream()


def t(name, fn, reps=200):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    print(json.dumps({"what": name, "us": round((time.perf_counter() - t0) / reps * 1e6, 2)}), flush=True)


with jb.Plan(dA, n=cfg.n, stream=s.cuda_stream) as p:
    t("jacobi_version (bare ctypes call)", jb.version)
    t("plan.info (ctypes + struct)", lambda: p.info)
    t("stream synchronize (idle)", s.synchronize)
    t("solve_device max_iter=0 (prepare + read-back + sync)", lambda: p.solve_device(db, dx0, xo, 0, 0.0))
    t("solve_device max_iter=1 (cluster, one launch)", lambda: p.solve_device(db, dx0, xo, 1, 0.0))
    t("solve_device max_iter=12", lambda: p.solve_device(db, dx0, xo, 12, 0.0))
