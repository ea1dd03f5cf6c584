# partial-tile row count as a compile-time constant: rates + parity
python probes/config_rates.py c2,c3 > gpurun_out/cfg_r02_nv.jsonl 2>&1
python probes/shard_rates.py c3 1,2,4,8 graph,persistent,persistent-push 40 > gpurun_out/shard_r02_nv_c3.jsonl 2>&1
python probes/shard_rates.py c4 1,8 graph 10 > gpurun_out/shard_r02_nv_c4.jsonl 2>&1
python -m pytest tests -m gpu -q -x > gpurun_out/gt_r02_nv.log 2>&1
echo done
