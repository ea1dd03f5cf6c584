# fixed-count runs skip the distance read between sweeps of the persistent solvers
timeout 900 python -m pytest tests/test_gridsync_gpu.py tests/test_parity_gpu.py -x -q > gpurun_out/needd_tests.txt 2>&1
for i in 1 2; do python probes/config_rates.py c2,c1; python probes/size_sweep.py f64 1024,2048,3072 400; python probes/shard_rates.py c3 8 persistent,persistent-push 40; done > gpurun_out/needd_rates.txt 2>&1
JACOBI_LIB=$PWD/probes/libjacobi_smt.so python probes/grid_timeline.py c2 > gpurun_out/grid_timeline_needd.jsonl 2>&1
echo done
