# Round-2 final-session evidence (v9: kernels as v7/v8; slow-companion parity tests added): GPU suite,
# smoke, bench, launch list of the bench command, ncu --set full of the c4 default kernel.
python -m pytest tests -m gpu -q > gpurun_out/gt_r02_v9.log 2>&1; tail -2 gpurun_out/gt_r02_v9.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v9.log 2>&1; cat gpurun_out/smoke_v9.log
python bench.py --out gpurun_out/bench_r02_v9.jsonl > gpurun_out/bench_r02_v9.out 2> gpurun_out/bench_r02_v9.err; echo "bench rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-configs"
$B > gpurun_out/plain_launch9.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_v9.csv $B > gpurun_out/ncu_launch9.log 2>&1; echo "ncu launches rc=$?"
python probes/one_plan.py 65536 f64 3 > gpurun_out/plain_c4_v9.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_cta -s 1 -c 1 -o gpurun_out/prof_c4_r02_v9 -f python probes/one_plan.py 65536 f64 3 > gpurun_out/ncu_c4_v9.log 2>&1; echo "ncu full rc=$?"
