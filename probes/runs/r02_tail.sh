# row-panel kernel with a dynamic tail (variant 12) vs the static x-smem panel (6): parity, bounds, c5 rates
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "all_sweep_variants" > gpurun_out/tail_tests.txt 2>&1
timeout 900 python -m pytest tests/test_bounds_gpu.py -x -q >> gpurun_out/tail_tests.txt 2>&1
JACOBI_LIB=check python probes/sanitize_small.py > gpurun_out/tail_sanitize.txt 2>&1
for i in 1 2; do for v in 6 12; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c5; JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 2,4,8 graph 10; done; done > gpurun_out/tail_rates.txt 2>&1
echo done
