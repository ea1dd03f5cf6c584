"""Small solves touching every kernel path.  compute-sanitizer is closed on this GPU pool, so the
driver for it is the bounds-checked build instead:
  JACOBI_LIB=check python probes/sanitize_small.py   (exit 3 and the mask if a check fired)
(tests/test_bounds_gpu.py runs it, plus a self-test of the checker.)
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


# (n, fp32 A, variants, persistent modes): the cluster path (small n), the persistent grid solver
# (mid n, JACOBI_PERSIST=1), and the graph path with the item / CTA / row-panel / x-smem / L2-keep
# kernels, including ragged rows and columns.
QUICK = "--quick" in sys.argv  # one graph-path case (checker self-test)
# Variant indices are the round-2 table's; a variant that cannot tile a case's chunking
# falls back to the default, and the line printed says which ran.
CASES = ((1, False, [None], ["0"]), (37, False, [None], ["0"]), (300, True, [None], ["0"]),
         (700, False, [None], ["1", "0"]), (3001, False, [None, "0", "3", "5", "6"], ["1", "0"]),
         (2049, True, [None, "5", "6", "12"], ["1", "0"]),
         (8190, False, [None, "0", "1", "2", "3", "5", "6", "7", "8", "9", "10", "12"], ["0"]),
         (8190, True, [None, "0", "5", "6", "12"], ["0"]), (20000, True, ["12"], ["0"]),
         (300, True, ["12"], ["0"]), (149, False, ["12"], ["0"]))
for n, f32, variants, modes in (((3001, False, [None], ["0"]),) if QUICK else CASES):
    A, b = dominant(n, n, f32)
    for v, mode in [(v, m) for v in variants for m in modes]:
        os.environ["JACOBI_PERSIST"] = mode
        if v is None:
            os.environ.pop("JACOBI_SWEEP_VARIANT", None)
        else:
            os.environ["JACOBI_SWEEP_VARIANT"] = v
        if v is not None and n < 1000:  # a forced sweep variant on a small n: graph path, not the cluster solver
            os.environ["JACOBI_SMALL_N"] = "0"
        else:
            os.environ.pop("JACOBI_SMALL_N", None)
        with jb.Plan(A) as p:
            ran = jb.variant_name(p.info.variant)
            r = p.solve(b, None, 6, 0.0, history=True)
            r2 = p.solve(b, None, 50, 1e-9)
            if n % 2 == 0:
                p.set_row_blocks(2)
                p.solve(b, None, 5, 0.0)
        print(n, f32, v, mode, ran, r.iters, r2.status, r2.iters, flush=True)
# fused exchange with emulated ranks: graph path and persistent solver
if not QUICK:
    A, b = dominant(4096, 4096, False)
    for mode in ("0", "1"):
        os.environ["JACOBI_PERSIST"] = mode
        os.environ.pop("JACOBI_SWEEP_VARIANT", None)
        with jb.Plan(A) as p:
            p.set_p2p_emulation(4)
            r = p.solve(b, None, 8, 0.0)
        print("p2p-emulation", mode, r.iters, flush=True)

checked, mask = jb.bounds_violations()
if checked:
    print(f"bounds check: violations mask = {mask:#x}", flush=True)
    sys.exit(3 if mask else 0)
print("sanitize_small ok")
