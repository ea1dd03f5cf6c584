# Round-2 evidence (v7: group kernel for fp32 shards, bench small-config timing): GPU suite, smoke, bench, launch list
python -m pytest tests -m gpu -q > gpurun_out/gt_r02_v7.log 2>&1; tail -2 gpurun_out/gt_r02_v7.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v7.log 2>&1; cat gpurun_out/smoke_v7.log
python bench.py --out gpurun_out/bench_r02_v7.jsonl > gpurun_out/bench_r02_v7.out 2> gpurun_out/bench_r02_v7.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs"
$B > gpurun_out/plain_launch7.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v7.csv $B > gpurun_out/ncu_launch7.log 2>&1; echo "ncu rc=$?"
