#!/usr/bin/env python
"""Benchmark of the dense Jacobi sweep (BASELINE.json metric: Jacobi iterations/s and effective HBM
GB/s, % of peak) on the headline workload c4: n = 65536 dense fp64 (34.4 GB), fixed 100 sweeps.

One STEP = one jacobi_plan_solve of the workload (100 sweeps, tol = 0, the whole hot path:
sweep + fused update + max|dx| + device stop test; + allgather/allreduce when N > 1).
  value : iterations/s with A, b, x0 resident in HBM (device-pointer solve), CUDA events on the
          plan's stream, max over ranks.  A (34 GB) >> L2 (126 MB): every sweep streams A from HBM,
          so no L2 flush is needed between steps.
  e2e   : the same metric through the C-ABI one-shot call jacobi_solve() with HOST (pinned) buffers:
          the H2D copy of A, b, x0, plan setup, 100 sweeps and the D2H copy of x are inside the
          timed region every step (N = 1; under torchrun the distributed plan is created per step
          from host rows).
  --impl reference : the CPU oracle (oracle/), as it stands, on the box's host cores, on a bounded
          row sample of the same workload per step; it/s extrapolated to whole sweeps.

Launch: python bench.py [--gpus N --steps K --warmup W]; N > 1 under torchrun (one rank per GPU).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (gen config key, sweeps per step, tol, description)
    "c4": ("c4", 100, 0.0, "c4: n=65536 dense fp64 (34.4 GB), off-diag U[-1,1], diag=rowabs+U[1,2], "
                           "b=A x*, x0=0, fixed 100 iterations, row-block sharded"),
    "c2": ("c2", 500, 0.0, "c2: n=4096 dense fp64 (134 MB), fixed 500 iterations"),
    "c5": ("c5", 100, 0.0, "c5 companion: n=131072, A fp32 (68.7 GB), fp64 accumulate, fixed 100 iterations"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c4")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU oracle sample budget per run")
    ap.add_argument("--exchange", choices=["auto", "nccl", "p2p", "cols"], default="auto",
                    help="N > 1: fused NVLink push (NEXT-1, 'p2p'), NCCL row-wise, or column-wise (NEXT-4); "
                         "auto = p2p when every GPU pair has peer access (agreed by all ranks), else nccl")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config rates of the other BASELINE.json configs (N = 1 only)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks sampling
class Clocks:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(name):
    """dram bytes per sweep launch from the committed ncu --set full summary (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(name, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ----------------------------------------------------------------------------- CPU oracle timing
def cpu_oracle_rate(wname, seconds, steps=None):
    """Oracle (oracle.sweep_rows) on a bounded row sample of the workload, on all host
    cores (rows split over threads; ctypes releases the GIL).  Returns (it/s, cores, sample)."""
    import jacobi_gen as g
    import oracle
    cfg = g.CONFIGS[WORKLOADS[wname][0]]
    n = cfg.n
    cores = len(os.sched_getaffinity(0))
    rows = min(n, max(cores * 64, 4096 if n >= 65536 else n))
    A, b = g.host_rows(cfg, 0, rows)
    x = g.host_xstar(cfg) * 0.5  # any x^(k-1); the work per row is data independent
    chunks = np.array_split(np.arange(rows), cores)

    def one_pass():
        out = [None] * len(chunks)

        def run(t):
            idx = chunks[t]
            if len(idx):
                out[t] = oracle.sweep_rows(A[idx[0]: idx[-1] + 1], int(idx[0]), b[idx[0]: idx[-1] + 1], x)

        th = [threading.Thread(target=run, args=(t,)) for t in range(len(chunks))]
        for t in th:
            t.start()
        for t in th:
            t.join()

    one_pass()  # warm
    t0 = time.perf_counter()
    passes = 0
    while True:
        one_pass()
        passes += 1
        el = time.perf_counter() - t0
        if (steps is not None and passes >= steps) or (steps is None and el >= seconds):
            break
    rate = passes * rows / n / el
    sample = f"oracle.sweep_rows over rows [0,{rows}) of {n} x {passes} passes in {el:.2f}s; it/s = passes*rows/n/t"
    return rate, cores, sample, el


# ----------------------------------------------------------------------------- other configs (N = 1)
OTHER_RUNS = (("c1", 200, 0.0), ("c1", 200, 1e-12), ("c2", 500, 0.0), ("c3", 5000, 1e-10), ("c3", 1000, 0.0),
              ("c5", 2000, 1e-6), ("c5", 100, 0.0))


def other_configs(jb, g, torch, stream):
    """Rates of the other BASELINE.json configs on this GPU (informational; the headline is c4):
    device-resident inputs, best of 3 solves after a warm-up, CUDA events on the plan's stream.
    it/s = sweeps / time; GB/s = algorithmic bytes per sweep x it/s (c1/c2 sit in or near L2)."""
    out = []
    sh = stream.cuda_stream
    for name in dict.fromkeys(r[0] for r in OTHER_RUNS):
        cfg = g.CONFIGS[name]
        n = cfg.n
        dA = torch.empty((n, n), dtype=torch.float32 if cfg.a_dtype == g.F32 else torch.float64, device="cuda")
        db = torch.empty(n, dtype=torch.float64, device="cuda")
        g.device_rows(cfg, 0, n, dA.data_ptr(), n, db.data_ptr(), sh)
        dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
        dxo = torch.empty(n, dtype=torch.float64, device="cuda")
        with jb.Plan(dA, n=n, stream=sh) as p:
            inf = p.info
            for _, max_iter, tol in (r for r in OTHER_RUNS if r[0] == name):
                p.set_batch(20 if max_iter % 20 == 0 else 32)
                r = p.solve_device(db, dx0, dxo, max_iter, tol)
                best = None
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    r = p.solve_device(db, dx0, dxo, max_iter, tol)
                    e1.record(stream)
                    e1.synchronize()
                    ms = e0.elapsed_time(e1)
                    best = ms if best is None else min(best, ms)
                its = r.iters / (best * 1e-3)
                out.append({"config": name, "n": n, "max_iter": max_iter, "tol": tol,
                            "status": jb.STATUS_NAMES[r.status], "iters": r.iters, "it_per_s": round(its, 1),
                            "us_per_sweep": round(1e3 * best / r.iters, 2),
                            "effective_gbs": round(inf.bytes_per_sweep * its / 1e9, 1),
                            "path": (f"cluster x{inf.cluster_ctas}" if inf.cluster_ctas else
                                     f"persistent x{inf.persistent_ctas}: cta_sweep" if inf.persistent_ctas else
                                     f"graph: {jb.variant_name(inf.variant)}")})
        del dA, db
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- main (GPU arm)
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    gname, sweeps, tol, desc = WORKLOADS[args.workload]

    if args.impl == "reference":
        if rank != 0:
            return 0
        per_step = []
        rate, cores, sample, el = cpu_oracle_rate(args.workload, None, steps=1)  # warm-up + sizing
        for _ in range(args.warmup):
            cpu_oracle_rate(args.workload, None, steps=1)
        t0 = time.perf_counter()
        rate, cores, sample, el = cpu_oracle_rate(args.workload, None, steps=args.steps)
        line = {"impl": "reference", "metric": "Jacobi iterations/s", "value": rate, "unit": "it/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": desc, "n": 65536 if gname == "c4" else None, "sweeps_per_step": sweeps},
                "cpu_baseline": {"value": rate, "unit": "it/s", "cores": cores, "kind": "oracle", "sample": sample},
                "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    import jacobi_gen as g
    import paper_1403_5805_b200 as jb

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = g.CONFIGS[gname]
    n = cfg.n
    dt = torch.float32 if cfg.a_dtype == g.F32 else torch.float64
    # A dedicated stream: the plan issues every kernel and collective on it and the CUDA events that
    # time the step are recorded on it.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream
    row0, m = jb.partition(n, world, rank)

    # ---- resident inputs (device twin of the generator; identical bits to the host generator)
    if world > 1 and args.exchange == "auto":
        ok = all(torch.cuda.can_device_access_peer(local, q) for q in range(world) if q != local)
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)  # every rank takes the same decision
        args.exchange = "p2p" if int(flag.item()) else "nccl"
    cols = world > 1 and args.exchange == "cols"
    db = torch.empty(m, dtype=torch.float64, device="cuda")
    if cols:  # column slab [row0, row0 + m) of all n rows: generate all rows, keep the slab
        dA = torch.empty((n, m), dtype=dt, device="cuda")
        tmp = torch.empty((4096, n), dtype=dt, device="cuda")
        tb = torch.empty(4096, dtype=torch.float64, device="cuda")
        for r in range(0, n, 4096):
            g.device_rows(cfg, r, min(n, r + 4096), tmp.data_ptr(), n, tb.data_ptr(), sh)
            dA[r:r + 4096].copy_(tmp[: min(4096, n - r), row0:row0 + m])
            if row0 <= r < row0 + m or r <= row0 < r + 4096:
                lo, hi = max(r, row0), min(r + 4096, row0 + m)
                if lo < hi:
                    db[lo - row0:hi - row0].copy_(tb[lo - r:hi - r])
        del tmp, tb
    else:
        dA = torch.empty((m, n), dtype=dt, device="cuda")
        g.device_rows(cfg, row0, row0 + m, dA.data_ptr(), n, db.data_ptr(), sh)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    dxo = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    K = 20 if sweeps % 20 == 0 else 4  # 100 sweeps = 5 graph batches exactly: no no-op overshoot launches
    plan = None

    def step():
        return plan.solve_device(db, dx0, dxo, sweeps, tol)

    def local_planted_error():
        """max |x - x*| on this rank after the warm-up solves (BASELINE.json: b = A x*, so the
        fixed-iteration configs end at x* to ~1e-16): a cheap end-to-end check of the exchange."""
        xs = torch.empty(n, dtype=torch.float64, device="cuda")
        g.device_xstar(cfg, xs.data_ptr(), sh)
        return float((dxo - xs).abs().max().item())

    def planted_error():  # max over ranks
        e = torch.tensor([local_planted_error()], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        return float(e.item())

    if world > 1 and args.exchange == "p2p":
        # The fused exchange is validated with emulated ranks only: any error on any rank (IPC attach,
        # a bounded peer wait that faulted) or a wrong result (planted-solution check) makes every rank
        # fall back to the NCCL exchange together.  No collective runs between here and the vote.
        from paper_1403_5805_b200.dist import dist_plan
        ok = 1
        try:
            plan = dist_plan(dA, n, stream=sh, p2p=True)
            plan.set_batch(K)
            for _ in range(max(3, args.warmup)):
                r = step()
            ok = int(r.iters == sweeps and r.status == jb.MAX_ITER and (tol != 0.0 or local_planted_error() <= 1e-10))
        except Exception as ex:  # noqa: BLE001 - any failure of the opt-in path means "fall back"
            print(f"bench: rank {rank}: fused exchange failed ({ex})", file=sys.stderr)
            ok = 0
        flag = torch.tensor([ok], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            print("bench: fused exchange unusable on some rank; using the NCCL exchange", file=sys.stderr)
            if plan is not None:
                try:
                    plan.close()
                except Exception:  # noqa: BLE001
                    pass
            plan = None
            args.exchange = "nccl"
    if plan is None:
        if world > 1:
            from paper_1403_5805_b200.dist import dist_plan
            plan = dist_plan(dA, n, stream=sh, layout="cols" if cols else "rows")
        else:
            plan = jb.Plan(dA, n=n, stream=sh)
        plan.set_batch(K)
        for _ in range(max(3, args.warmup)):
            r = step()
    assert r.iters == sweeps and r.status == jb.MAX_ITER
    planted = planted_error() if tol == 0.0 else None  # reported: the solve reached x*
    info = plan.info
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        launches = 0
        for _ in range(args.steps):
            step()
            li = plan.info
            launches += li.sweeps_launched + li.sweeps_launched // K + 1  # sweeps + k_advance + k_prepare
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    its = args.steps * sweeps / (ms * 1e-3)
    sweep_ms = ms / (args.steps * sweeps)  # average sweep (kernel + exchange) duration on the stream
    bytes_sweep = info.bytes_per_sweep  # per GPU
    achieved = bytes_sweep / (sweep_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak_hbm()

    # per-kernel timing (untimed cross-check: events around each sweep kernel alone)
    kms = plan.time_sweeps(db, dx0, min(sweeps, 20))
    kernel_ms = float(np.median(kms[1:])) if len(kms) > 1 else float(kms[0])

    ceiling = None
    if rank == 0:
        try:
            ceiling = jb.bwprobe(min(32 << 30, int(bytes_sweep)), 5)
        except Exception:
            ceiling = None

    plan.close()
    del dA, db
    torch.cuda.empty_cache()

    # ---- e2e through the public C-ABI with host buffers (pinned), copies inside the timed region.
    # N = 1: the one-shot jacobi_solve (north-star signature).  N > 1: per step every rank creates a
    # distributed plan from its host row block (H2D inside), solves from host b / x0 and reads x back.
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        import ctypes
        hA = torch.empty((m, n), dtype=dt, pin_memory=True)
        g.host_rows(cfg, row0, row0 + m, out=hA.numpy())
        hb = torch.empty(m, dtype=torch.float64, pin_memory=True)
        hb.numpy()[:] = g.host_diag_b(cfg, row0, row0 + m)[1]
        hx0 = torch.zeros(n, dtype=torch.float64, pin_memory=True)
        hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
        solve_fn = jb._lib.jacobi_solve_f32a if cfg.a_dtype == g.F32 else jb._lib.jacobi_solve
        it = ctypes.c_int64()

        def e2e_step():
            if world == 1:
                st = solve_fn(n, hA.data_ptr(), hb.data_ptr(), hx0.data_ptr(), sweeps, tol, hx.data_ptr(),
                              ctypes.byref(it))
                assert st == jb.MAX_ITER and it.value == sweeps, (st, jb.last_error())
            else:
                from paper_1403_5805_b200.dist import dist_plan
                with dist_plan(hA.numpy(), n) as p:
                    r = p.solve(hb.numpy(), hx0.numpy(), sweeps, tol)
                    assert r.status == jb.MAX_ITER and r.iters == sweeps

        e2e_step()  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        e2e = {"value": args.e2e_steps * sweeps / el, "unit": "it/s",
               "h2d_bytes_per_step": int(world * (hA.numel() * hA.element_size() + 8 * m + 8 * n)),
               "d2h_bytes_per_step": int(world * (8 * n + 48)), "steps": args.e2e_steps,
               "api": ("jacobi_solve (C-ABI one-shot, host pinned buffers: plan setup + H2D + sweeps + D2H per step)"
                       if world == 1 else
                       "jacobi_dist_plan_create + jacobi_plan_solve per step on every rank (host row block, H2D, "
                       "NCCL comm init, sweeps, D2H); wall time, max over ranks")}
        del hA

    configs = None
    if world == 1 and not args.no_configs:
        configs = other_configs(jb, g, torch, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, _ = cpu_oracle_rate(args.workload, args.cpu_seconds)
        cpu = {"value": rate, "unit": "it/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": "Jacobi iterations/s", "value": its, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based generator, BASELINE.json recipe; device twin)",
            "config": {"workload": desc, "n": n, "sweeps_per_step": sweeps, "tol": tol,
                       "parallelism": (f"row-block x{world}" if not cols else f"column-slab x{world}") + (
                           {"nccl": " + NCCL allgather/allreduce", "p2p": " + fused NVLink push exchange (NEXT-1)",
                            "cols": " + NCCL reduce-scatter/allreduce (NEXT-4)"}[args.exchange] if world > 1 else ""),
                       "l2": "A per GPU >> 126 MB L2; each sweep streams A from HBM (no flush needed)",
                       "graph_batch": K, "chunk_cols": info.chunk_cols, "rows_per_warp": info.rows_per_warp,
                       "grid": f"{info.grid_ctas}x{info.threads_per_cta}"},
            "effective_gbs_per_gpu": achieved, "effective_gbs_aggregate": achieved * world,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(args.workload),
                         "peak_source": peak_src, "kernel": f"{jb.variant_name(info.variant)} ({'fp64' if dt == torch.float64 else 'fp32'} A)",
                         "bytes_per_launch": bytes_sweep, "avg_launch_ms": sweep_ms,
                         "kernel_only_ms": kernel_ms, "kernel_only_gbs": bytes_sweep / (kernel_ms * 1e-3) / 1e9,
                         "read_ceiling_gbs": ceiling,
                         "frac_of_read_ceiling": (achieved / ceiling) if ceiling else None,
                         "frac_of_8tbs": achieved / 8000.0},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "other_configs": configs,
            "check": {"planted_max_abs_err": planted,
                      "what": "max_i |x_i - x*_i| after the warm-up solves (b = A x*), max over ranks"},
        }
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
