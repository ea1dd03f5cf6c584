set -x
for b in 0.5 0.6; do echo "budget $b"; JACOBI_L2_BUDGET=$b python probes/config_rates.py c2; JACOBI_L2_BUDGET=$b python probes/shard_rates.py c3 8 graph,persistent 40; done > gpurun_out/keep_budget3_r02.txt 2>&1
for pf in 0 1 2 4; do echo "prefetch $pf"; JACOBI_PREFETCH=$pf python probes/shard_rates.py c3 1,8 graph 40; JACOBI_PREFETCH=$pf python probes/shard_rates.py c4 8 graph 10; done > gpurun_out/prefetch_r02.txt 2>&1
python probes/shard_rates.py c3 1,2,4,8 graph,persistent,persistent-push 40 > gpurun_out/shard_r02e_c3.jsonl 2>&1
python -m pytest tests -m gpu -q > gpurun_out/gt_r02e.log 2>&1
echo done
