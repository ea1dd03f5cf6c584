"""Where the e2e time of the one-shot jacobi_solve goes (c4: 34 GB A from pinned host memory).

Times, on one GPU: cudaMalloc + cudaFree of the A block, the pinned H2D copy of A (one call, and in
1 GiB pieces on two streams), plan creation from host A, a 100-sweep solve, plan destroy.
"""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

cfg = g.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = cfg.n
nbytes = n * n * 8
cudart = ctypes.CDLL("libcudart.so.12")
hA = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
g.host_rows(cfg, 0, n, out=hA.numpy())
hb = torch.from_numpy(g.host_diag_b(cfg, 0, n)[1].copy())
out = {}

p = ctypes.c_void_p()
t0 = time.perf_counter()
assert cudart.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(nbytes)) == 0
cudart.cudaDeviceSynchronize()
out["cudaMalloc_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
assert cudart.cudaMemcpy(p, ctypes.c_void_p(hA.data_ptr()), ctypes.c_size_t(nbytes), 1) == 0
out["h2d_one_call_s"] = time.perf_counter() - t0
out["h2d_one_call_gbs"] = nbytes / out["h2d_one_call_s"] / 1e9
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
piece = 1 << 30
torch.cuda.synchronize()
t0 = time.perf_counter()
for i, off in enumerate(range(0, nbytes, piece)):
    sz = min(piece, nbytes - off)
    st = (s1 if i % 2 == 0 else s2).cuda_stream
    cudart.cudaMemcpyAsync(ctypes.c_void_p(p.value + off), ctypes.c_void_p(hA.data_ptr() + off), ctypes.c_size_t(sz), 1,
                           ctypes.c_void_p(st))
torch.cuda.synchronize()
out["h2d_two_streams_s"] = time.perf_counter() - t0
out["h2d_two_streams_gbs"] = nbytes / out["h2d_two_streams_s"] / 1e9
t0 = time.perf_counter()
cudart.cudaFree(p)
cudart.cudaDeviceSynchronize()
out["cudaFree_s"] = time.perf_counter() - t0

for rep in range(2):
    t0 = time.perf_counter()
    plan = jb.Plan(hA.numpy(), n=n)
    t1 = time.perf_counter()
    r = plan.solve(hb.numpy(), None, 100, 0.0)
    t2 = time.perf_counter()
    plan.close()
    t3 = time.perf_counter()
    out[f"plan_create_s_{rep}"] = t1 - t0
    out[f"solve100_s_{rep}"] = t2 - t1
    out[f"destroy_s_{rep}"] = t3 - t2
print(json.dumps(out))
