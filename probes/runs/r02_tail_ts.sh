# c5: per-sweep launch times (time_sweeps) and a 100-sweep device solve, static (6) vs dynamic-tail (12) panels
python probes/tail_ts.py 6,12,6,12 > gpurun_out/tail_ts.jsonl 2>&1
echo done
