# persistent solver with shared-memory-resident rows of A (JACOBI_GRID_RES=0 disables)
python -m pytest tests/test_gridsync_gpu.py -q -x > gpurun_out/res_tests.log 2>&1; tail -2 gpurun_out/res_tests.log
JACOBI_LIB=check timeout 600 python probes/sanitize_small.py > gpurun_out/res_sanitize.log 2>&1; echo "sanitize rc=$?"; tail -1 gpurun_out/res_sanitize.log
for rep in 1 2; do
JACOBI_GRID_RES=0 python probes/size_sweep.py f64 1024,2048,3072,4096 400 | sed 's/^/{"res": 0, /; s/^{"res": 0, {/{"res": 0, /'
python probes/size_sweep.py f64 1024,2048,3072,4096 400 | sed 's/^{/{"res": 1, /'
done > gpurun_out/res_sizes.jsonl 2>&1
for rep in 1 2; do
JACOBI_GRID_RES=0 python probes/size_sweep.py f32 1024,2048,4096,6000 400 | sed 's/^{/{"res": 0, /'
python probes/size_sweep.py f32 1024,2048,4096,6000 400 | sed 's/^{/{"res": 1, /'
done > gpurun_out/res_sizes_f32.jsonl 2>&1
cut -c1-200 gpurun_out/res_sizes.jsonl gpurun_out/res_sizes_f32.jsonl
