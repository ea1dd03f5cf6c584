# persistent solver: step 0 of each warp's first unit bulk-copied into shared memory during the grid barrier
timeout 900 python -m pytest tests/test_gridsync_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/pre_tests.txt 2>&1
JACOBI_LIB=check timeout 600 python -m pytest tests/test_bounds_gpu.py -x -q >> gpurun_out/pre_tests.txt 2>&1
for i in 1 2; do python probes/config_rates.py c2; python probes/size_sweep.py f64 1024,2048,3072 400; JACOBI_PERSIST=1 python probes/size_sweep.py f64 6144,8192 100; python probes/size_sweep.py f32 4096,8192 400; python probes/shard_rates.py c3 8 persistent,persistent-push 40; done > gpurun_out/pre_rates.txt 2>&1
JACOBI_LIB=$PWD/probes/libjacobi_smt.so python probes/grid_timeline.py c2 > gpurun_out/grid_timeline_pre.jsonl 2>&1
echo done
