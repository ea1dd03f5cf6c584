# persistent solver: L1 prefetch of the next sweep's first unit during the grid barrier
for pf in 0 1 2 8; do echo "grid_prefetch $pf"; JACOBI_GRID_PREFETCH=$pf python probes/config_rates.py c2; JACOBI_GRID_PREFETCH=$pf python probes/shard_rates.py c3 8 persistent 40; JACOBI_GRID_PREFETCH=$pf python probes/size_sweep.py f64 1024,2048,3072 400; done > gpurun_out/l1pf_r02.txt 2>&1
echo done
