"""Experiment: c2 (n = 4096, A = 134 MB ~ L2 size) with an L2 persisting access-policy window on A.

Sets cudaLimitPersistingL2CacheSize to the device maximum and a stream access-policy window over A
(hitRatio = persisting bytes / A bytes), captures the plan's graphs under it, and times solves.
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

cudart = ctypes.CDLL("libcudart.so.12")


class AccessPolicyWindow(ctypes.Structure):
    _fields_ = [("base_ptr", ctypes.c_void_p), ("num_bytes", ctypes.c_size_t), ("hitRatio", ctypes.c_float),
                ("hitProp", ctypes.c_int), ("missProp", ctypes.c_int)]


class StreamAttrValue(ctypes.Union):
    _fields_ = [("accessPolicyWindow", AccessPolicyWindow), ("pad", ctypes.c_char * 64)]


def attr(a):
    v = ctypes.c_int()
    cudart.cudaDeviceGetAttribute(ctypes.byref(v), a, 0)
    return v.value


L2 = attr(38)            # cudaDevAttrL2CacheSize
MAXP = attr(108)         # cudaDevAttrMaxPersistingL2CacheSize
MAXW = attr(109)         # cudaDevAttrMaxAccessPolicyWindowSize
print(json.dumps({"l2": L2, "max_persisting": MAXP, "max_window": MAXW}), flush=True)

cfg = g.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
n = cfg.n
A, b, xs = g.host_system(cfg)
dA = torch.from_numpy(A).cuda()
db = torch.from_numpy(b).cuda()
dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
xo = torch.empty_like(dx0)
stream = torch.cuda.Stream()


def run(label):
    with torch.cuda.stream(stream):
        with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
            p.set_batch(20)
            p.solve_device(db, dx0, xo, 500, 0.0)
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                r = p.solve_device(db, dx0, xo, 500, 0.0)
                e1.record(stream)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1))
            print(json.dumps({"mode": label, "us_per_sweep": 1e3 * best / r.iters,
                              "err": float((xo.cpu() - torch.from_numpy(xs)).abs().max())}), flush=True)
            return xo.cpu().clone()


x_plain = run("plain")
rc1 = cudart.cudaDeviceSetLimit(0x06, ctypes.c_size_t(MAXP))  # cudaLimitPersistingL2CacheSize
nbytes = min(A.nbytes, MAXW)
v = StreamAttrValue()
v.accessPolicyWindow = AccessPolicyWindow(dA.data_ptr(), nbytes, min(1.0, MAXP / nbytes), 2, 1)  # persisting/streaming
rc2 = cudart.cudaStreamSetAttribute(ctypes.c_void_p(stream.cuda_stream), 1, ctypes.byref(v))
print(json.dumps({"set_limit_rc": rc1, "set_attr_rc": rc2, "window_bytes": nbytes,
                  "hit_ratio": min(1.0, MAXP / nbytes)}), flush=True)
x_p = run("persisting")
print(json.dumps({"bitwise_equal": bool(torch.equal(x_plain, x_p))}))
