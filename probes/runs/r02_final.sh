# final validation of the round: GPU suite, smoke, default bench line
python -m pytest tests -m gpu -q > gpurun_out/gt_r02_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
python bench.py --out gpurun_out/bench_r02_v3.jsonl > gpurun_out/bench_r02_v3.out 2> gpurun_out/bench_r02_v3.err
echo done
