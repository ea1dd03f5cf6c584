for rep in 1 2; do for v in 6 13 15; do JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 2,4,8 graph 100; done; done > gpurun_out/group3_c5.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/group3_c5.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['P'], d['variant'], round(d['shard_us'],1), round(d['gbs_per_gpu'],1))
"
