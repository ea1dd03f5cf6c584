# persistent solver: L2 prefetch of the next sweep's first unit during the grid barrier; keep budget
for pf in 0 1; do echo "grid_prefetch $pf"; JACOBI_GRID_PREFETCH=$pf python probes/config_rates.py c2; JACOBI_GRID_PREFETCH=$pf python probes/shard_rates.py c3 8 persistent 40; JACOBI_GRID_PREFETCH=$pf python probes/size_sweep.py f64 1024,2048,3072 400; done > gpurun_out/gridpf_r02.txt 2>&1
for b in 0.45 0.55 0.6 0.65; do echo "budget $b"; JACOBI_L2_BUDGET=$b python probes/config_rates.py c2; JACOBI_L2_BUDGET=$b python probes/shard_rates.py c3 1,4,8 graph,persistent 40; done > gpurun_out/keep_budget5_r02.txt 2>&1
echo done
