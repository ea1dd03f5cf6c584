"""Randomized parity of the group kernel (variant 12, forced with JACOBI_SWEEP_VARIANT) at ragged sizes,
fp32 and fp64 A, random x0 / tol / iteration counts / row-block splits, against the CPU oracle; also
bitwise against the row-panel kernel (variant 6) on the same plan inputs.

python probes/fuzz_group.py first_seed count -> one JSON line per case, then a summary line.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

os.environ["JACOBI_SMALL_N"] = "0"
os.environ["JACOBI_PERSIST"] = "0"
first, count = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(seed)
    f32 = bool(rng.random() < 0.6)
    n = int(rng.choice([150, 511, 1025, 3001, 4353, 8191, 12289, 16385, 20001]))
    A = rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(1) * float(rng.uniform(1.02, 1.3)) * rng.choice([-1.0, 1.0], n))
    if f32:
        A = A.astype(np.float32)
    b = rng.uniform(-1, 1, n)
    x0 = None if rng.random() < 0.5 else rng.uniform(-1, 1, n)
    max_iter = int(rng.choice([1, 2, 7, 20]))
    tol = float(rng.choice([0.0, 1e-9]))
    blocks = int(rng.choice([b_ for b_ in (1, 2, 3, 5) if n % b_ == 0]))
    st_o, x_o, it_o, h_o = oracle.jacobi(A, b, x0, max_iter, tol, nthreads=16, history=True)
    res = {}
    for v in ("12", "6"):
        os.environ["JACOBI_SWEEP_VARIANT"] = v
        with jb.Plan(A) as p:
            if blocks > 1:
                p.set_row_blocks(blocks)
            ran = jb.variant_name(p.info.variant)
            res[v] = (ran, p.solve(b, x0, max_iter, tol, history=True))
    r = res["12"][1]
    den = max(np.max(np.abs(x_o)), 1e-300)
    err = float(np.max(np.abs(r.x - x_o)) / den)
    same = np.array_equal(r.x, res["6"][1].x) and np.array_equal(r.hist, res["6"][1].hist)
    ok = ((r.status, r.iters) == (st_o, it_o) and err <= 1e-10 and np.allclose(r.hist, h_o, rtol=1e-8, atol=1e-14)
          and same and res["12"][0].startswith("k_sweep_group"))
    print(json.dumps({"seed": seed, "n": n, "f32": f32, "blocks": blocks, "max_iter": max_iter, "tol": tol,
                      "ok": bool(ok), "ran": res["12"][0], "bitwise_vs_panel": bool(same), "rel_err": err}),
          flush=True)
    fails += not ok
print(json.dumps({"cases": count, "failures": fails}))
sys.exit(1 if fails else 0)
