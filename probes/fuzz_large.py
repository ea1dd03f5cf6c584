"""Randomized parity sweep at larger, ragged sizes (graph path with the L2-resident share, static and
dynamic tiles, partial tiles, row-block splits), against the CPU oracle.

python probes/fuzz_large.py first_seed count -> one JSON line per failure, then a summary line.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([4353, 6000, 8191, 12289, 16385, 20001, 24577]))
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * float(rng.uniform(1.02, 1.3)) * rng.choice([-1.0, 1.0], n))
    b = rng.uniform(-1, 1, n)
    x0 = None if rng.random() < 0.5 else rng.uniform(-1, 1, n)
    max_iter = int(rng.choice([1, 2, 7, 20]))
    tol = float(rng.choice([0.0, 1e-9]))
    blocks = int(rng.choice([b_ for b_ in (1, 2, 3) if n % b_ == 0]))
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=16, history=True)
    with jb.Plan(A) as p:
        if blocks > 1:
            p.set_row_blocks(blocks)
        inf = p.info
        r = p.solve(b, x0, max_iter, tol, history=True)
    den = max(np.max(np.abs(x_o)), 1e-300)
    err = float(np.max(np.abs(r.x - x_o)) / den)
    ok = (r.status, r.iters) == (st_o, it_o) and err <= 1e-10 and np.allclose(r.hist, h_o, rtol=1e-8, atol=1e-14)
    print(json.dumps({"seed": seed, "n": n, "blocks": blocks, "max_iter": max_iter, "tol": tol, "ok": bool(ok),
                      "variant": jb.variant_name(inf.variant), "keep_pm": inf.l2_keep_permille,
                      "iters": [r.iters, it_o], "err": err}), flush=True)
    fails += 0 if ok else 1
print(json.dumps({"first": first, "count": count, "fails": fails}), flush=True)
