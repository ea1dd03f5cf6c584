"""Parity at sizes where the dynamic-tile kernel is the default (fp64 rows >= 32 x 4 x SMs), ragged n.

python probes/parity_dyn_sizes.py -> one JSON line per case (GPU vs oracle: status, iters, rel L-inf).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

for n, seed, max_iter, tol in ((18950, 1, 6, 0.0), (20001, 2, 40, 1e-9), (24575, 3, 5, 0.0)):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05 * rng.choice([-1.0, 1.0], n))
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-1, 1, n)
    st_o, x_o, it_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=os.cpu_count())
    with jb.Plan(A) as p:
        v = jb.variant_name(p.info.variant)
        r = p.solve(b, x0, max_iter, tol)
    err = float(np.max(np.abs(r.x - x_o)) / np.max(np.abs(x_o)))
    print(json.dumps({"n": n, "variant": v, "status": [r.status, st_o], "iters": [r.iters, it_o], "rel_linf": err,
                      "ok": (r.status, r.iters) == (st_o, it_o) and err <= 1e-10}), flush=True)
