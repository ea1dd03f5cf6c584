# persistent solver: hybrid units (register step 0 + bulk-copied step 1) at c2
JACOBI_GRID_HY=1 timeout 600 python -m pytest tests/test_gridsync_gpu.py -x -q > gpurun_out/hy_tests.txt 2>&1
make lib-check > /dev/null 2>&1 && JACOBI_LIB=check JACOBI_GRID_HY=1 timeout 600 python -m pytest tests/test_bounds_gpu.py -x -q >> gpurun_out/hy_tests.txt 2>&1
for a in 0 1 0 1; do echo "hy $a"; JACOBI_GRID_HY=$a python probes/config_rates.py c2; JACOBI_GRID_HY=$a JACOBI_PERSIST=1 python probes/size_sweep.py f64 3900 200; done > gpurun_out/hy_rates.txt 2>&1
echo done
