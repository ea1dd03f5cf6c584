# Round-2 evidence run (final code): bench line, shard rates, launch list, ncu --set full of the c4
# kernel, the c3 P = 8 shard kernel and the c2 persistent solver, GPU test suite.
python bench.py --out gpurun_out/bench_r02_v4.jsonl > gpurun_out/bench_r02_v4.out 2> gpurun_out/bench_r02_v4.err
python probes/shard_rates.py c3 1,2,4,8 graph,persistent,persistent-push 40 > gpurun_out/shard_r02_v4_c3.jsonl 2>&1
python probes/shard_rates.py c4 1,2,4,8 graph,persistent-push 10 > gpurun_out/shard_r02_v4_c4.jsonl 2>&1
python probes/shard_rates.py c5 2,4,8 graph 10 > gpurun_out/shard_r02_v4_c5.jsonl 2>&1
python probes/config_rates.py > gpurun_out/cfg_r02_v4.jsonl 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gt_r02_v4.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs"
$B > gpurun_out/plain_launch4.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v4.csv $B > gpurun_out/ncu_launch4.log 2>&1
python probes/one_plan.py 65536 f64 3 > gpurun_out/plain_c4d.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_cta -s 1 -c 1 -o gpurun_out/prof_c4_r02v4 -f python probes/one_plan.py 65536 f64 3 > gpurun_out/ncu_c4d.log 2>&1
python probes/shard_rates.py c3 8 graph 4 > gpurun_out/plain_c3p8d.log 2>&1 && ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_sweep_cta -s 6 -c 1 -o gpurun_out/prof_c3p8_r02v4 -f python probes/shard_rates.py c3 8 graph 4 > gpurun_out/ncu_c3p8d.log 2>&1
python probes/size_sweep.py f64 4096 50 > gpurun_out/plain_c2d.log 2>&1 && ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_solve_gridsync -s 2 -c 1 -o gpurun_out/prof_c2_r02v4 -f python probes/size_sweep.py f64 4096 50 > gpurun_out/ncu_c2d.log 2>&1
echo done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v4.log 2>&1
