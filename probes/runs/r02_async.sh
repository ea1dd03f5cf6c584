# persistent solver: register-loaded vs asynchronous-copy sweep (cta_sweep_async)
JACOBI_GRID_ASYNC=1 timeout 600 python -m pytest tests/test_gridsync_gpu.py -x -q -k "async" > gpurun_out/async_tests.txt 2>&1
for a in 0 1 0 1; do echo "async $a"; JACOBI_GRID_ASYNC=$a python probes/config_rates.py c2; JACOBI_GRID_ASYNC=$a JACOBI_PERSIST=1 python probes/size_sweep.py f64 3900,8192 200; done > gpurun_out/async_rates.txt 2>&1
export JACOBI_PERSIST=1
JACOBI_GRID_ASYNC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_gridsync -c 1 \
  -o gpurun_out/grid_async1 python probes/size_sweep.py f64 4096 100 > gpurun_out/grid_async_ncu1.log 2>&1
echo done
