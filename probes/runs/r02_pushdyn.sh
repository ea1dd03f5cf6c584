python -m pytest tests/test_parity_gpu.py -m gpu -q -k "fused or time_shard or c5_full or variants" > gpurun_out/gt_pushdyn.log 2>&1
python bench.py --force-dist --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_forcedist2.jsonl 2> gpurun_out/bench_forcedist2.err
echo done
