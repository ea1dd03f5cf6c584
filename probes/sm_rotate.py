"""Is the sweep's tail a property of the SMs or of the rows?  Probe build (-DJACOBI_SM_TIMING, loaded
with JACOBI_LIB=probes/libjacobi_smt.so): the row-panel kernel of c5 with the CTA -> row-block map
rotated by r (CTA b takes block (b + r) mod G); per CTA its %smid, row block and finish time.

python probes/sm_rotate.py [n] [f32|f64] -> one JSON line per rotation
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
f32 = (sys.argv[2] if len(sys.argv) > 2 else "f32") == "f32"
cfg = g.GenConfig(n, a_dtype=g.F32 if f32 else g.F64, diag_mode=g.DIAG_SCALE, diag_scale=1.2)
dA = torch.empty((n, n), dtype=torch.float32 if f32 else torch.float64, device="cuda")
db = torch.empty(n, dtype=torch.float64, device="cuda")
g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), torch.cuda.current_stream().cuda_stream)
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
lib = ctypes.CDLL(jb.LIB_PATH)
with jb.Plan(dA, n=n, stream=torch.cuda.current_stream().cuda_stream) as p:
    G = p.info.grid_ctas
    for rot in (0, 37, 74, 111):
        assert lib.jacobi_debug_set_rotation(rot) == 0
        for rep in range(2):
            ms = p.time_sweeps(db, dx0, 2)
            buf = (ctypes.c_ulonglong * (3 * G))()
            assert lib.jacobi_debug_sm_times(buf, G) == 0
            a = np.array(buf[:], dtype=np.int64).reshape(-1, 3)
            end = (a[:, 2] - a[:, 1].min()) / 1e3
            print(json.dumps({"n": n, "rot": rot, "rep": rep, "variant": jb.variant_name(p.info.variant),
                              "ms": list(ms), "smid": a[:, 0].tolist(),
                              "block": [(b + rot) % G for b in range(G)],
                              "end_us": [round(v, 1) for v in end.tolist()]}), flush=True)
    lib.jacobi_debug_set_rotation(0)
