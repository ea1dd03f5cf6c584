# persistent solver with 2 column steps in flight (JACOBI_GRID_U) and persistent vs graph across sizes
for u in 1 2; do echo "grid_u $u"; JACOBI_GRID_U=$u python probes/config_rates.py c2; JACOBI_GRID_U=$u python probes/shard_rates.py c3 1,8 persistent 40; JACOBI_GRID_U=$u python probes/size_sweep.py f64 2048,3072 400; done > gpurun_out/gridu_r02.txt 2>&1
for p in 0 1; do echo "persist $p"; JACOBI_PERSIST=$p python probes/size_sweep.py f64 4608,6144,8192,12288,16384,24576 100; done > gpurun_out/persist_sizes_r02.txt 2>&1
echo done
