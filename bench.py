#!/usr/bin/env python
"""Benchmark of the dense Jacobi sweep (BASELINE.json metric: Jacobi iterations/s and effective HBM
GB/s, % of peak) on the headline workload c4: n = 65536 dense fp64 (34.4 GB), fixed 100 sweeps.

One STEP = one jacobi_plan_solve of the workload (100 sweeps, tol = 0, the whole hot path:
sweep + fused update + max|dx| + device stop test; + allgather/allreduce when N > 1).
  value : iterations/s with A, b, x0 resident in HBM (device-pointer solve), CUDA events on the
          plan's stream, max over ranks.  A (34 GB, or 34/N GB per GPU) >> L2 (126 MB): every sweep
          streams A from HBM, so no L2 flush is needed between steps.
  e2e   : the same metric through the C-ABI with HOST (pinned) buffers: N = 1 the one-shot
          jacobi_solve() (H2D of A, b, x0, plan setup, 100 sweeps, D2H of x inside the timed region
          every step); N > 1 every rank creates its distributed plan from its host row block per step.
  cpu_baseline : the CPU oracle (oracle/), as it stands, on the host cores of rank 0: its sweep
          (oracle.sweep_rows on all cores + oracle.maxnorm_dist) over the WHOLE c4 system for a bounded
          number of its 100 sweeps, the once-per-solve validation pass of oracle.jacobi timed beside it,
          plus one-thread oracle.jacobi per-sweep times of c1-c3.
  --impl reference : the same oracle sweeps as the reference arm; each step = --ref-sweeps consecutive
          sweeps of the whole system (rank 0 only under torchrun).

Multi-GPU: ``python bench.py --gpus N`` re-launches itself with N ranks (torch.distributed.run,
127.0.0.1) when WORLD_SIZE is unset; under torchrun (the driver's form) it runs as one rank per GPU.
Row blocks (§3) with the NCCL allgather of x + one-scalar max allreduce per sweep
(the north star's exchange) is the headline; the fused NVLink push exchange (NEXT-1)
is timed after it as a separate field (``fused_exchange``), bounded by a watchdog so a failure there
can never cost the headline line.
"""
import argparse
import json
import os
import socket
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
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU oracle budget: sweeps of the full system timed for about this long")
    ap.add_argument("--ref-sweeps", type=int, default=3,
                    help="--impl reference: oracle sweeps of the full system per step")
    ap.add_argument("--exchange", choices=["nccl", "p2p", "cols"], default="nccl",
                    help="N > 1 headline exchange: NCCL row-wise (north star, default), fused NVLink push "
                         "(NEXT-1) or column-wise reduce-scatter (NEXT-4)")
    ap.add_argument("--no-fused", action="store_true", help="N > 1: skip the fused-exchange side measurement")
    ap.add_argument("--fused-timeout", type=float, default=180.0,
                    help="watchdog (s) of the fused-exchange side measurement")
    ap.add_argument("--force-dist", action="store_true",
                    help="test hook: take the N > 1 code path (distributed plans, fused-exchange leg) even at N = 1")
    ap.add_argument("--launcher-dry-run", action="store_true",
                    help="spawn the ranks (gloo, no GPU work) and report what was spawned: tests the launcher")
    ap.add_argument("--out", default=None, help="also append the JSON line to this file")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config rates of the other BASELINE.json configs (N = 1 only)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- self-launch (N > 1)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args):
    """`bench.py --gpus N` without WORLD_SIZE: re-run this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1.  Fails loudly if fewer than N GPUs are visible."""
    if not args.launcher_dry_run:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launcher_dry_run(world, rank):
    """Each spawned rank joins a gloo group and reports itself; rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    got = [None] * world
    dist.all_gather_object(got, {"rank": rank, "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
                                 "pid": os.getpid()})
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "world_size": dist.get_world_size(),
                          "ranks": [g["rank"] for g in got], "local_ranks": [g["local_rank"] for g in got],
                          "distinct_pids": len({g["pid"] for g in got}), "torch": torch.__version__}), flush=True)
    dist.destroy_process_group()
    return 0


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
def oracle_sweeps(A, b, x, sweeps, cores):
    """`sweeps` sweeps of the oracle over the whole system: oracle.sweep_rows on row ranges
    in `cores` host threads (ctypes releases the GIL; per-row arithmetic unchanged, so the bits equal
    oracle.jacobi's at any thread count: pins P11/P13) and oracle.maxnorm_dist for d_k.  Returns
    (x, hist, seconds)."""
    import oracle
    n = A.shape[0]
    bounds = [n * t // cores for t in range(cores + 1)]
    hist = []
    t0 = time.perf_counter()
    for _ in range(sweeps):
        xn = np.empty(n)

        def run(t):
            r0, r1 = bounds[t], bounds[t + 1]
            if r1 > r0:
                xn[r0:r1] = oracle.sweep_rows(A[r0:r1], r0, b[r0:r1], x)

        th = [threading.Thread(target=run, args=(t,)) for t in range(cores)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        hist.append(oracle.maxnorm_dist(xn, x))
        x = xn
    return x, hist, time.perf_counter() - t0


def cpu_oracle_full(wname, seconds, A=None, b=None, sweeps=None):
    """The oracle as it stands on all host cores of this process, over the WHOLE system of the workload:
    its sweeps (oracle_sweeps: oracle.sweep_rows + oracle.maxnorm_dist) for `sweeps`
    sweeps, or as many of the workload's sweeps as fit in about `seconds` (sized by a first sweep).
    The once-per-solve validation pass of oracle.jacobi (max_iter = 0: the EZERODIAG/ENONFINITE scan,
    single-threaded) is timed separately.  A, b: the host system if the caller already holds it (the
    e2e leg does); else it is generated here."""
    import jacobi_gen as g
    import oracle
    cfg = g.CONFIGS[WORKLOADS[wname][0]]
    total_sweeps = WORKLOADS[wname][1]
    cores = len(os.sched_getaffinity(0))
    t_gen = None
    if A is None:
        t0 = time.perf_counter()
        A, b = g.host_rows(cfg, 0, cfg.n)
        t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.jacobi(A, b, None, 0, 0.0, nthreads=cores)  # validation pass alone
    t_val = time.perf_counter() - t0
    x = np.zeros(cfg.n)
    if sweeps is None:
        x, _, t1 = oracle_sweeps(A, b, x, 1, cores)
        sweeps = int(max(1, min(total_sweeps - 1, seconds // max(t1, 1e-6))))
    x, hist, el = oracle_sweeps(A, b, x, sweeps, cores)
    per_sweep = el / sweeps
    solve_s = t_val + total_sweeps * per_sweep
    return {"value": 1.0 / per_sweep, "unit": "it/s", "cores": cores, "kind": "oracle",
            "sample": (f"{sweeps} of the {total_sweeps} sweeps of the whole {wname} system (n={cfg.n}) with the "
                       f"oracle's sweep (oracle.sweep_rows on {cores} threads + oracle.maxnorm_dist) in {el:.2f} s; "
                       f"it/s = sweeps / time.  oracle.jacobi's once-per-solve validation pass took {t_val:.2f} s "
                       f"(single thread): a whole {total_sweeps}-sweep oracle solve ~ {solve_s:.1f} s"),
            "per_sweep_s": per_sweep, "sweeps": sweeps, "seconds": el, "validation_s": t_val,
            "solve_it_per_s": total_sweeps / solve_s, "gen_s": t_gen}


def cpu_oracle_t1(configs=("c1", "c2", "c3"), seconds=2.0):
    """One-thread oracle per-sweep time of the small configs (T = 1 for c1-c3)."""
    import jacobi_gen as g
    import oracle
    out = {}
    for name in configs:
        cfg = g.CONFIGS[name]
        A, b = g.host_rows(cfg, 0, cfg.n)
        t0 = time.perf_counter()
        oracle.jacobi(A, b, None, 1, 0.0, nthreads=1)
        t1 = time.perf_counter() - t0
        k = int(max(1, min(200, seconds // max(t1, 1e-6))))
        t0 = time.perf_counter()
        oracle.jacobi(A, b, None, k, 0.0, nthreads=1)
        el = time.perf_counter() - t0
        out[name] = {"n": cfg.n, "sweeps": k, "seconds": el, "per_sweep_s": el / k, "it_per_s": k / el,
                     "threads": 1}
        del A
    return out


def reference_arm(args, rank):
    """--impl reference: the CPU oracle as it stands on the host cores (rank 0 only under torchrun);
    each step = args.ref_sweeps sweeps of oracle.jacobi over the WHOLE workload system."""
    if rank != 0:
        return 0
    import jacobi_gen as g
    gname, sweeps, tol, desc = WORKLOADS[args.workload]
    cfg = g.CONFIGS[gname]
    t0 = time.perf_counter()
    A, b = g.host_rows(cfg, 0, cfg.n)
    t_gen = time.perf_counter() - t0
    import oracle
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    oracle.jacobi(A, b, None, 0, 0.0, nthreads=cores)  # the oracle's validation pass, once per solve
    t_val = time.perf_counter() - t0
    x = np.zeros(cfg.n)
    for _ in range(args.warmup):
        x, _, _ = oracle_sweeps(A, b, x, args.ref_sweeps, cores)
    x = np.zeros(cfg.n)
    el = 0.0
    for _ in range(args.steps):  # consecutive sweeps of one solve from x0 = 0
        x, _, t = oracle_sweeps(A, b, x, args.ref_sweeps, cores)
        el += t
    rate = args.steps * args.ref_sweeps / el
    cb = {"value": rate, "unit": "it/s", "cores": cores, "kind": "oracle", "seconds": el, "validation_s": t_val,
          "gen_s": t_gen,
          "sample": (f"{args.steps} steps x {args.ref_sweeps} consecutive sweeps of the whole {gname} system "
                     f"(n={cfg.n}) with the oracle's sweep (oracle.sweep_rows on {cores} threads + "
                     f"oracle.maxnorm_dist); the once-per-solve validation pass ({t_val:.2f} s) is not in a step")}
    line = {"impl": "reference", "metric": "Jacobi iterations/s", "value": rate, "unit": "it/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter-based generator, host)",
            "config": {"workload": desc, "n": cfg.n, "sweeps_per_step": args.ref_sweeps,
                       "note": "reference step = a bounded sample of the workload's sweeps (the GPU arm's step is "
                               "all of them); it/s is the comparable quantity"},
            "cpu_baseline": cb,
            "e2e": {"value": rate, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- other configs (N = 1)
OTHER_RUNS = (("c1", 200, 0.0), ("c1", 200, 1e-12), ("c2", 500, 0.0), ("c3", 5000, 1e-10), ("c3", 1000, 0.0),
              ("c5", 2000, 1e-6), ("c5", 100, 0.0))
# The NEXT rows measured on c3 (informational): the paper's Euclidean stop rule (NEXT-2: per-sweep dx^2
# block tree + final sum) and the column-wise scheme's slab kernels as 8 slabs on one GPU (NEXT-4: 8
# slab GEMVs writing row sums + the column-sum epilogue), each over 1000 fixed sweeps.
NEXT_RUNS = (("c3", 1000, 0.0, "l2", 1), ("c3", 1000, 0.0, "max", 8))


def other_configs(jb, g, torch, stream):
    """Rates of the other BASELINE.json configs on this GPU (informational; the headline is c4):
    device-resident inputs, best of 3 solves (10 for c1/c2) after a warm-up, CUDA events on the plan's
    stream; a 1 s pause first lets the SM clock recover from the headline's power-capped run.
    it/s = sweeps / time; GB/s = algorithmic bytes per sweep x it/s (c1/c2 sit in or near L2); for the
    footprint above 32 GiB (c5) the read-only ceiling over min(A, 64 GiB) is measured beside it."""
    out = []
    sh = stream.cuda_stream
    time.sleep(1.0)
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
            runs = [(mi, tol, "max", 1) for nm, mi, tol in OTHER_RUNS if nm == name]
            runs += [(mi, tol, norm, cb) for nm, mi, tol, norm, cb in NEXT_RUNS if nm == name]
            for max_iter, tol, norm, colblocks in runs:
                # fixed runs: batches that divide the sweep count; tol runs: short loop bodies (a stop
                # inside a batch leaves its remaining sweeps as no-ops)
                p.set_batch(8 if tol > 0 else (20 if max_iter % 20 == 0 else 32))
                p.set_norm(norm)
                p.set_col_blocks(colblocks)
                r = p.solve_device(db, dx0, dxo, max_iter, tol)
                best = None
                # latency-bound small configs (c1, c2: µs per solve, clock-sensitive): best of 10
                for _ in range(10 if n <= 4096 else 3):
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
                                     f"graph: {jb.variant_name(inf.variant)}")
                            + ("" if norm == "max" else " + Euclidean rule (NEXT-2)")
                            + ("" if colblocks == 1 else f"; as {colblocks} column slabs of {n // colblocks} columns on "
                                                          "one GPU (NEXT-4 emulation: slab GEMVs + column-sum epilogue)")})
            p.set_norm("max")
            p.set_col_blocks(1)
            if name == "c3":  # NEXT-4 per rank: rank 0's compact 16384 x 2048 slab at P = 8 (+ its epilogue)
                try:  # informational: a failure must not cost the line
                    slab_ms, slab_v = p.time_shard(db, dx0, 8, 0, 40, "colslab")
                except jb.JacobiError as ex:
                    slab_ms, slab_v = None, str(ex)
            if name == "c3" and slab_ms is None:
                out.append({"config": "c3", "path": "one rank's column slab at P = 8 (NEXT-4)", "error": slab_v})
            elif name == "c3":
                slab_bytes = n * (n // 8) * 8 + 8 * n + 16 * (n // 8)
                out.append({"config": "c3", "n": n, "max_iter": 40, "tol": 0.0, "status": "n/a", "iters": 40,
                            "it_per_s": round(1e3 / slab_ms, 1), "us_per_sweep": round(1e3 * slab_ms, 2),
                            "effective_gbs": round(slab_bytes / (slab_ms * 1e-3) / 1e9, 1),
                            "path": f"graph: {jb.variant_name(slab_v)}; one rank's column slab at P = 8 (NEXT-4, "
                                    "jacobi_plan_time_shard mode 3: 16384 x 2048 compact slab + own-row epilogue, "
                                    "reduce-scatter excluded)"})
            if inf.bytes_per_sweep > (32 << 30):  # c5: the read ceiling over its own footprint (capped at
                # 64 GiB), measured here beside its rates (the headline's ceiling covers 32 GiB; a probe
                # over c3's 2.1 GB is one 0.3 ms launch per pass, ramp-bound, so it is not reported)
                try:  # informational: a failed probe (e.g. no room beside A) must not cost the line
                    ceil = jb.bwprobe(int(min(inf.bytes_per_sweep, 64 << 30)), 3)
                except jb.JacobiError as ex:
                    ceil, err = None, str(ex)
                for e in out:
                    if e["config"] == name:
                        if ceil:
                            e["read_ceiling_gbs"] = round(ceil, 1)
                            e["frac_of_read_ceiling"] = round(e["effective_gbs"] / ceil, 3)
                        else:
                            e["read_ceiling_error"] = err
        del dA, db
        torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- fused exchange (N > 1 side leg)
def fused_exchange_leg(jb, torch, dist, dA, db, dx0, dxo, n, sh, stream, sweeps, steps, K, rank, world,
                       planted_ok):
    """Times the fused NVLink push exchange (NEXT-1) on the same row blocks.
    Every stage that can fail on one rank alone ends in a vote (MIN all-reduce of an ok flag) that every
    rank reaches, so a failure becomes a reported error, not a hang; hangs inside NCCL are covered by
    the caller's watchdog.  Returns a dict for the JSON line."""
    from paper_1403_5805_b200.dist import bootstrap

    def vote(ok):
        f = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
        return bool(int(f.item()))

    plan = None
    try:
        uid, _, _, _, _ = bootstrap(n)  # torch.distributed broadcast: every rank enters
        err = None
        try:
            plan = jb.Plan(dA, n=n, stream=sh, dist=(uid, rank, world))
        except Exception as ex:  # noqa: BLE001
            err = f"plan: {ex}"
        if not vote(err is None):
            return {"error": err or "plan creation failed on another rank"}
        mine = None
        try:
            mine = plan.ipc_export()
        except Exception as ex:  # noqa: BLE001
            err = f"ipc_export: {ex}"
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        if err is None and any(h is None for h in allh):
            err = "ipc_export failed on another rank"
        if err is None:
            try:
                plan.ipc_attach(b"".join(allh))
                plan.set_batch(K)
            except Exception as ex:  # noqa: BLE001
                err = f"ipc_attach: {ex}"
        if not vote(err is None):
            return {"error": err or "ipc attach failed on another rank"}
        for i in range(3):  # warm-up solves, one vote after each (every rank enters every solve)
            ok = True
            try:
                r = plan.solve_device(db, dx0, dxo, sweeps, 0.0)
                ok = r.iters == sweeps and r.status == jb.MAX_ITER and planted_ok()
            except Exception as ex:  # noqa: BLE001
                err, ok = f"warm-up solve: {ex}", False
            if not vote(ok):
                return {"error": err or "warm-up solve failed or wrong on some rank"}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        ok = True
        try:
            for _ in range(steps):
                plan.solve_device(db, dx0, dxo, sweeps, 0.0)
        except Exception as ex:  # noqa: BLE001
            err, ok = f"timed solve: {ex}", False
        e1.record(stream)
        torch.cuda.synchronize()
        if not vote(ok):
            return {"error": err or "timed solve failed on some rank"}
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        inf = plan.info
        its = steps * sweeps / (ms * 1e-3)
        return {"value": its, "unit": "it/s", "ms_per_step": ms / steps, "steps": steps,
                "effective_gbs_per_gpu": inf.bytes_per_sweep * its / 1e9,
                "kernel": jb.variant_name(inf.variant),
                "what": "row blocks, the sweep kernel pushes x_i^(k) into every rank's buffer over NVLink and "
                        "signals arrival counters (no NCCL per sweep); planted-solution check passed"}
    finally:
        if plan is not None:
            try:
                plan.close()
            except Exception:  # noqa: BLE001
                pass


# ----------------------------------------------------------------------------- main (GPU arm)
def main():
    args = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1 and args.impl == "cuda":
        return launch_ranks(args)
    world = int(world_env or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.launcher_dry_run:
        return launcher_dry_run(world, rank)
    if args.impl == "reference":
        return reference_arm(args, rank)
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    gname, sweeps, tol, desc = WORKLOADS[args.workload]

    import torch
    import torch.distributed as dist

    import jacobi_gen as g
    import paper_1403_5805_b200 as jb

    if torch.cuda.device_count() <= local:
        print(f"bench.py: rank {rank} needs CUDA device {local}; {torch.cuda.device_count()} visible", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dist_on = world > 1 or args.force_dist
    if dist_on:
        if world == 1 and "MASTER_PORT" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
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
    cols = dist_on and args.exchange == "cols"
    db = torch.empty(m, dtype=torch.float64, device="cuda")
    if cols:  # column slab [row0, row0 + m) of all n rows: generate all rows, keep the slab
        dA = torch.empty((n, m), dtype=dt, device="cuda")
        tmp = torch.empty((4096, n), dtype=dt, device="cuda")
        tb = torch.empty(4096, dtype=torch.float64, device="cuda")
        for r in range(0, n, 4096):
            g.device_rows(cfg, r, min(n, r + 4096), tmp.data_ptr(), n, tb.data_ptr(), sh)
            dA[r:r + 4096].copy_(tmp[: min(4096, n - r), row0:row0 + m])
            lo, hi = max(r, row0), min(r + 4096, row0 + m)
            if lo < hi:
                db[lo - row0:hi - row0].copy_(tb[lo - r:hi - r])
        del tmp, tb
    else:
        dA = torch.empty((m, n), dtype=dt, device="cuda")
        g.device_rows(cfg, row0, row0 + m, dA.data_ptr(), n, db.data_ptr(), sh)
    dx0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    dxo = torch.empty(n, dtype=torch.float64, device="cuda")
    xs_dev = torch.empty(n, dtype=torch.float64, device="cuda")
    g.device_xstar(cfg, xs_dev.data_ptr(), sh)
    torch.cuda.synchronize()
    K = 20 if sweeps % 20 == 0 else 4  # 100 sweeps = 5 graph batches exactly: no no-op overshoot launches

    def local_planted_error():
        """max |x - x*| on this rank after a solve (BASELINE.json: b = A x*, so the fixed-iteration
        configs end at x* to ~1e-16): a cheap end-to-end check of the exchange."""
        return float((dxo - xs_dev).abs().max().item())

    def planted_error():  # max over ranks
        e = torch.tensor([local_planted_error()], dtype=torch.float64, device="cuda")
        if dist_on:
            dist.all_reduce(e, op=dist.ReduceOp.MAX)
        return float(e.item())

    if dist_on:
        from paper_1403_5805_b200.dist import dist_plan
        plan = dist_plan(dA, n, stream=sh, layout="cols" if cols else "rows", p2p=args.exchange == "p2p")
    else:
        plan = jb.Plan(dA, n=n, stream=sh)
    plan.set_batch(K)

    def step():
        return plan.solve_device(db, dx0, dxo, sweeps, tol)

    for _ in range(max(3, args.warmup)):
        r = step()
    assert r.iters == sweeps and r.status == jb.MAX_ITER
    planted = planted_error() if tol == 0.0 else None  # reported: the solve reached x*
    info = plan.info
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        if dist_on:
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
        if dist_on:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if dist_on:
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
    if dist_on:
        t = torch.tensor([kernel_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kernel_ms = float(t.item())

    ceiling = None
    if rank == 0:
        try:
            ceiling = jb.bwprobe(min(32 << 30, int(bytes_sweep)), 5)
        except Exception:  # noqa: BLE001
            ceiling = None
    plan.close()

    line = {
        "metric": "Jacobi iterations/s", "value": its, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter-based generator, BASELINE.json recipe; device twin)",
        "config": {"workload": desc, "n": n, "sweeps_per_step": sweeps, "tol": tol,
                   "parallelism": (f"row-block x{world}" if not cols else f"column-slab x{world}") + (
                       {"nccl": " + NCCL allgather/allreduce", "p2p": " + fused NVLink push exchange (NEXT-1)",
                        "cols": " + NCCL reduce-scatter/allreduce (NEXT-4)"}[args.exchange] if dist_on else ""),
                   "l2": "A per GPU >> 126 MB L2; each sweep streams A from HBM (no flush needed)",
                   "graph_batch": K, "chunk_cols": info.chunk_cols, "rows_per_warp": info.rows_per_warp,
                   "grid": f"{info.grid_ctas}x{info.threads_per_cta}"},
        "effective_gbs_per_gpu": achieved, "effective_gbs_aggregate": achieved * world,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(args.workload),
                     "peak_source": peak_src,
                     "kernel": f"{jb.variant_name(info.variant)} ({'fp64' if dt == torch.float64 else 'fp32'} A)",
                     "bytes_per_launch": bytes_sweep, "avg_launch_ms": sweep_ms,
                     "kernel_only_ms": kernel_ms, "kernel_only_gbs": bytes_sweep / (kernel_ms * 1e-3) / 1e9,
                     "read_ceiling_gbs": ceiling,
                     "frac_of_read_ceiling": (achieved / ceiling) if ceiling else None,
                     "frac_of_8tbs": achieved / 8000.0},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": None,
        "e2e": None,
        "other_configs": None,
        "check": {"planted_max_abs_err": planted,
                  "what": "max_i |x_i - x*_i| after the warm-up solves (b = A x*), max over ranks"},
    }

    # ---- N > 1: the fused NVLink exchange as a side measurement, under a watchdog
    if dist_on and args.exchange == "nccl" and not args.no_fused and not cols:
        done = threading.Event()

        def watchdog():
            if not done.wait(args.fused_timeout):
                if rank == 0:
                    line["fused_exchange"] = {"error": f"watchdog: no result within {args.fused_timeout:.0f} s"}
                    print(json.dumps(line), flush=True)
                os._exit(0)

        threading.Thread(target=watchdog, daemon=True).start()
        try:
            line["fused_exchange"] = fused_exchange_leg(
                jb, torch, dist, dA, db, dx0, dxo, n, sh, stream, sweeps, args.steps, K, rank, world,
                lambda: local_planted_error() <= 1e-10)
        except Exception as ex:  # noqa: BLE001
            line["fused_exchange"] = {"error": str(ex)}
        done.set()
    del dA, db
    torch.cuda.empty_cache()

    # ---- e2e through the public C-ABI with host buffers (pinned), copies inside the timed region.
    # N = 1: the one-shot jacobi_solve (north-star signature).  N > 1: per step every rank creates a
    # distributed plan from its host row block (H2D inside), solves from host b / x0 and reads x back.
    hA = None
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
            if not dist_on:
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
        if dist_on:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if dist_on:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        line["e2e"] = {"value": args.e2e_steps * sweeps / el, "unit": "it/s",
                       "h2d_bytes_per_step": int(world * (hA.numel() * hA.element_size() + 8 * m + 8 * n)),
                       "d2h_bytes_per_step": int(world * (8 * n + 48)), "steps": args.e2e_steps,
                       "api": ("jacobi_solve (C-ABI one-shot, host pinned buffers: plan setup + H2D + sweeps + D2H "
                               "per step)" if not dist_on else
                               "jacobi_dist_plan_create + jacobi_plan_solve per step on every rank (host row block, "
                               "H2D, NCCL comm init, sweeps, D2H); wall time, max over ranks")}

    if not dist_on and not args.no_configs:
        line["other_configs"] = other_configs(jb, g, torch, stream)

    # ---- CPU oracle on rank 0's host cores (every N); reuses the e2e host A when it is the whole system
    if rank == 0 and not args.no_cpu_baseline:
        whole = hA is not None and m == n
        cb = cpu_oracle_full(args.workload, args.cpu_seconds, hA.numpy() if whole else None,
                             g.host_diag_b(cfg, 0, n)[1] if whole else None)
        hA = None
        cb["t1"] = cpu_oracle_t1()
        line["cpu_baseline"] = cb
    hA = None

    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
