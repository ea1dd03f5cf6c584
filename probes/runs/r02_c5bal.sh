# c5 shards: balanced panel tiling (variant 6) and the R8 panel (12), P = 1, 2, 4, 8
python -m pytest tests/test_parity_gpu.py -q -k "variant" > gpurun_out/c5bal_tests.log 2>&1; tail -2 gpurun_out/c5bal_tests.log
python probes/shard_rates.py c5 1,2,4,8 graph 10 > gpurun_out/c5bal_v6.jsonl 2>&1
JACOBI_SWEEP_VARIANT=12 python probes/shard_rates.py c5 1,2,4,8 graph 10 > gpurun_out/c5bal_v12.jsonl 2>&1
python probes/shard_rates.py c5 1,2,4,8 graph 10 >> gpurun_out/c5bal_v6.jsonl 2>&1
JACOBI_SWEEP_VARIANT=12 python probes/shard_rates.py c5 1,2,4,8 graph 10 >> gpurun_out/c5bal_v12.jsonl 2>&1
cat gpurun_out/c5bal_v6.jsonl gpurun_out/c5bal_v12.jsonl | cut -c1-250
