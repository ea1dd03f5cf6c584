"""Extended randomized parity sweep (tests/test_fuzz_gpu.py's case generator, more seeds).

python probes/fuzz_more.py first_seed count -> one JSON line per failure, then a summary line.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402
from test_fuzz_gpu import case  # noqa: E402

first, count = int(sys.argv[1]), int(sys.argv[2])
fails = ties = 0
for seed in range(first, first + count):
    n, f32, A, b, x0, max_iter, tol, norm, persist, small, blocks = case(seed)
    for var, val in (("JACOBI_PERSIST", persist), ("JACOBI_SMALL_N", small)):
        if val == "default":
            os.environ.pop(var, None)
        else:
            os.environ[var] = val
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=16, history=True, norm=norm)
    with jb.Plan(A) as p:
        p.set_norm(norm)
        if blocks > 1:
            p.set_row_blocks(blocks)
        r = p.solve(b, x0, max_iter, tol, history=True)
    if tol > 0 and it_o >= 1 and abs(h_o[it_o - 1] - tol) <= 1e-6 * tol:
        ties += 1
        continue
    den = max(np.max(np.abs(x_o)), 1e-300)
    err = float(np.max(np.abs(r.x - x_o)) / den)
    ok = (r.status, r.iters) == (st_o, it_o) and err <= 1e-10 and np.allclose(r.hist, h_o, rtol=1e-8, atol=1e-14)
    if not ok:
        fails += 1
        print(json.dumps({"seed": seed, "n": n, "f32": f32, "max_iter": max_iter, "tol": tol, "norm": norm,
                          "persist": persist, "small": small, "blocks": blocks, "status": [r.status, st_o],
                          "iters": [r.iters, it_o], "err": err}), flush=True)
print(json.dumps({"first": first, "count": count, "fails": fails, "ties": ties}), flush=True)
