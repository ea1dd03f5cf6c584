"""Per-CTA finish times of one sweep-kernel launch (probe build: make lib NVFLAGS+=-DJACOBI_SM_TIMING,
copied over libjacobi.so).  python probes/sm_times.py n f64|f32 -> one JSON line: per CTA (smid,
start, end) in ns relative to the earliest start, plus a summary."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

n = int(sys.argv[1])
f32 = sys.argv[2] == "f32"
cfg = g.GenConfig(n, a_dtype=g.F32 if f32 else g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
dA = torch.empty((n, n), dtype=torch.float32 if f32 else torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
lib = ctypes.CDLL(jb.LIB_PATH)
with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
    inf = p.info
    for rep in range(3):
        ms = p.time_sweeps(db, dx0, 2)
        buf = (ctypes.c_ulonglong * (3 * inf.grid_ctas))()
        assert lib.jacobi_debug_sm_times(buf, inf.grid_ctas) == 0
        a = np.array(buf[:], dtype=np.int64).reshape(-1, 3)
        t0 = a[:, 1].min()
        end = (a[:, 2] - t0) / 1e3
        print(json.dumps({"n": n, "dtype": "f32" if f32 else "f64", "variant": jb.variant_name(inf.variant),
                          "ms": list(ms), "end_us_min": end.min(), "end_us_med": float(np.median(end)),
                          "end_us_max": end.max(), "idle_frac_avg": float(1 - end.mean() / end.max()),
                          "smid": a[:, 0].tolist(), "end_us": [round(v, 2) for v in end.tolist()]}), flush=True)
