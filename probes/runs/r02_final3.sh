# after the fixed-count distance-read skip in the persistent solvers: suite, smoke, launch list, bench
python -m pytest tests -m gpu -q > gpurun_out/gt_r02_v6.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v6.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs"
$B > gpurun_out/plain_launch6.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v6.csv $B > gpurun_out/ncu_launch6.log 2>&1
python bench.py --out gpurun_out/bench_r02_v6.jsonl > gpurun_out/bench_r02_v6.out 2> gpurun_out/bench_r02_v6.err
echo done
