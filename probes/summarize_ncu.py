"""Summarise an ncu --set full report of the sweep kernel and an ncu launch list into profiles/.

python probes/summarize_ncu.py <report.ncu-rep> <launches.csv> <tag> <command description>
-> profiles/ncu_sweep_summary.json (per workload key 'c4'), profiles/launches_<tag>_summary.txt
"""
import collections
import csv
import json
import subprocess
import sys

rep, launches, tag, cmd = sys.argv[1:5]
key = sys.argv[5] if len(sys.argv) > 5 else "c4"             # workload key in ncu_sweep_summary.json
alg = float(sys.argv[6]) if len(sys.argv) > 6 else 34361311232  # algorithmic bytes per launch
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, u, v = r[0], r[1], r[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def num(k):
    val, unit = d[k]
    return float(val.replace(",", "")) * scale.get(unit, 1)


summ = {key: {
    "kernel": d["Kernel Name"][0] if "Kernel Name" in d else "k_sweep",
    "source": f"{rep} (ncu --set full --clock-control none, {cmd})",
    "duration_ms": num("gpu__time_duration.sum") * 1e3,
    "dram_bytes_read": num("dram__bytes_read.sum"), "dram_bytes_write": num("dram__bytes_write.sum"),
    "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
    "algorithmic_bytes_per_launch": alg,
    "dram_gbs": (num("dram__bytes_read.sum") + num("dram__bytes_write.sum")) / num("gpu__time_duration.sum") / 1e9,
    "dram_throughput_pct_of_ncu_peak": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]),
    "dram_slice_active_min_pct": float(d["dram__cycles_active.min.pct_of_peak_sustained_elapsed"][0]),
    "dram_slice_active_max_pct": float(d["dram__cycles_active.max.pct_of_peak_sustained_elapsed"][0]),
    "l2_hit_rate_pct": float(d["lts__t_sector_hit_rate.pct"][0]),
    "l1_hit_rate_pct": float(d["l1tex__t_sector_hit_rate.pct"][0]),
    "registers": int(float(d["launch__registers_per_thread"][0])),
    "achieved_warps_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
    "sm_clock_ghz": num("sm__cycles_elapsed.avg.per_second") / 1e9 if d["sm__cycles_elapsed.avg.per_second"][1] == "hz" else float(d["sm__cycles_elapsed.avg.per_second"][0]),
    "stall_samples": {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(d[k][0])) for k in d
                      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                      and float(d[k][0]) > 100},
}}
try:
    allsum = json.load(open("profiles/ncu_sweep_summary.json"))
except (OSError, ValueError):
    allsum = {}
allsum.update(summ)
json.dump(allsum, open("profiles/ncu_sweep_summary.json", "w"), indent=1)
print(json.dumps(summ, indent=1))

if launches == "-":
    sys.exit(0)
rows = [x for x in csv.reader(open(launches)) if len(x) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for x in rows[1:]:
    nm = x[ki].split("(")[0]
    agg[nm][0] += 1
    agg[nm][1] += float(x[vi].replace(",", ""))
tot = sum(a[1] for a in agg.values())
with open(f"profiles/launches_{tag}_summary.txt", "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of\n# {cmd}\n"
            "# launches  total_ms  share  kernel\n")
    for k, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        f.write(f"{a[0]:5d} {a[1] / 1e6:10.3f} {100 * a[1] / tot:6.2f}%  {k}\n")
print(open(f"profiles/launches_{tag}_summary.txt").read())
