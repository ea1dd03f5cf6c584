# persistent solver: L2 bulk prefetch of the next tile's HBM-streamed units (JACOBI_GRID_PF)
JACOBI_GRID_PF=1 timeout 600 python -m pytest tests/test_gridsync_gpu.py -x -q > gpurun_out/gridpf2_tests.txt 2>&1
for a in 0 1 0 1; do echo "pf $a"; JACOBI_GRID_PF=$a python probes/config_rates.py c2; JACOBI_GRID_PF=$a JACOBI_PERSIST=1 python probes/size_sweep.py f64 3072,6144,8192 200; done > gpurun_out/gridpf2_rates.txt 2>&1
echo done
