"""Per-sweep time across problem sizes (fp64 or fp32 A), default kernel choice, graph-batched solves.

python probes/size_sweep.py f64|f32 n1,n2,... [sweeps]   -> one JSON line per n
System: seeded generator (off-diagonals U[-1,1], diag = 1.2 x row abs-sum), written on the device.
Shows the regimes: cluster (A in shared memory), L2-resident, L2-keep, HBM streaming.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

f32 = sys.argv[1] == "f32"
sizes = [int(v) for v in sys.argv[2].split(",")]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 400
stream = torch.cuda.Stream()
if os.environ.get("SETASIDE_MB"):  # experiment: persisting-L2 set-aside (cudaLimitPersistingL2CacheSize)
    import ctypes
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    mx = ctypes.c_int(0)
    rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    want = min(mx.value, int(float(os.environ["SETASIDE_MB"]) * 1e6))
    err = rt.cudaDeviceSetLimit(0x06, ctypes.c_size_t(want))  # cudaLimitPersistingL2CacheSize
    got = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(got), 0x06)
    print(json.dumps({"setaside_max": mx.value, "want": want, "err": err, "got": got.value}), flush=True)
for n in sizes:
    cfg = g.GenConfig(n, a_dtype=g.F32 if f32 else g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
    dA = torch.empty((n, n), dtype=torch.float32 if f32 else torch.float64, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    xo = torch.empty(n, dtype=torch.float64, device="cuda")
    with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
        inf = p.info
        p.set_batch(20)
        p.solve_device(db, dx0, xo, sweeps, 0.0)
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = p.solve_device(db, dx0, xo, sweeps, 0.0)
            e1.record(stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        us = 1e3 * best / sweeps
        print(json.dumps({"n": n, "f32": f32, "a_mb": n * n * (4 if f32 else 8) / 1e6, "us_per_sweep": us,
                          "it_per_s": 1e6 / us, "effective_gbs": inf.bytes_per_sweep / us / 1e3,
                          "path": (f"cluster x{inf.cluster_ctas}" if inf.cluster_ctas else
                                   f"persistent x{inf.persistent_ctas}" if inf.persistent_ctas else
                                   f"graph: {jb.variant_name(inf.variant)}")}),
              flush=True)
    del dA
    torch.cuda.empty_cache()
