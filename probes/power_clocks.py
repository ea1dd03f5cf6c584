"""SM clock, board power and throttle reasons while a config's fixed-count solve streams (NVML sampled
every ~10 ms in a thread), to test whether a config's plateau is a power limit (c5 at
P = 1 sits at ~7.03 TB/s sustained for every kernel design).

python probes/power_clocks.py c4,c5 [solves] [env-variant-list]  -> one JSON line per (config, variant)
  variant list: comma-separated JACOBI_SWEEP_VARIANT values ('' = default), applied per plan.
Each line: GB/s of back-to-back 100-sweep solves (device-resident inputs) and the median / min SM
clock, median / max power and the throttle reasons seen while they ran.
"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import jacobi_gen as g  # noqa: E402
import paper_1403_5805_b200 as jb  # noqa: E402

import pynvml  # noqa: E402

REASONS = {0x1: "gpu_idle", 0x2: "app_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal",
           0x40: "hw_thermal", 0x80: "hw_power_brake"}

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c4", "c5"]
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 6
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else [""]
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
stream = torch.cuda.current_stream()


def sampler(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.01)


for name in names:
    cfg = g.CONFIGS[name]
    n = cfg.n
    dt = torch.float32 if cfg.a_dtype == g.F32 else torch.float64
    dA = torch.empty((n, n), dtype=dt, device="cuda")
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), stream.cuda_stream)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    xo = torch.empty(n, dtype=torch.float64, device="cuda")
    for v in variants:
        if v:
            os.environ["JACOBI_SWEEP_VARIANT"] = v
        else:
            os.environ.pop("JACOBI_SWEEP_VARIANT", None)
        with jb.Plan(dA, n=n, stream=stream.cuda_stream) as p:
            inf = p.info
            p.set_batch(20)
            p.solve_device(db, dx0, xo, 100, 0.0)  # warm-up (graph capture)
            time.sleep(1.0)
            samples, stop = [], threading.Event()
            th = threading.Thread(target=sampler, args=(stop, samples))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            th.start()
            e0.record(stream)
            for _ in range(solves):
                p.solve_device(db, dx0, xo, 100, 0.0)
            e1.record(stream)
            e1.synchronize()
            stop.set()
            th.join()
            ms = e0.elapsed_time(e1)
            busy = samples[len(samples) // 10:]  # drop the ramp
            clk = sorted(s[0] for s in busy)
            pw = sorted(s[1] for s in busy)
            reasons = 0
            for s in busy:
                reasons |= s[2]
            print(json.dumps({"config": name, "variant": jb.variant_name(inf.variant) if hasattr(jb, "variant_name")
                              else inf.variant, "solves": solves, "sweeps": 100 * solves,
                              "gbs": inf.bytes_per_sweep * 100 * solves / (ms * 1e-3) / 1e9,
                              "us_per_sweep": 1e3 * ms / (100 * solves),
                              "sm_mhz_median": clk[len(clk) // 2], "sm_mhz_min": clk[0],
                              "power_w_median": pw[len(pw) // 2], "power_w_max": pw[-1],
                              "reasons": [nm for bit, nm in REASONS.items() if reasons & bit],
                              "samples": len(busy)}), flush=True)
    del dA
    torch.cuda.empty_cache()
