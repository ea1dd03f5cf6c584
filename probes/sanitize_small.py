"""Small solves touching every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck).

Run ONE tool per gpurun call, e.g.
  compute-sanitizer --tool memcheck --error-exitcode 9 python probes/sanitize_small.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_5805_b200 as jb  # noqa: E402


def dominant(n, seed, f32=False):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * 1.05 + (n == 1))
    return (A.astype(np.float32) if f32 else A), rng.uniform(-1, 1, n)


for n, f32, variants in ((1, False, [None]), (37, False, [None]), (300, True, [None]),
                         (8190, False, [None, "1", "6", "9", "10"]), (8190, True, [None])):
    A, b = dominant(n, n, f32)
    for v in variants:
        if v is None:
            os.environ.pop("JACOBI_SWEEP_VARIANT", None)
        else:
            os.environ["JACOBI_SWEEP_VARIANT"] = v
        with jb.Plan(A) as p:
            r = p.solve(b, None, 6, 0.0, history=True)
            r2 = p.solve(b, None, 50, 1e-9)
            if n % 2 == 0:
                p.set_row_blocks(2)
                p.solve(b, None, 5, 0.0)
        print(n, f32, v, r.iters, r2.status, r2.iters, flush=True)
print("sanitize_small ok")
