# dynamic-tail panel (variant 12), chunk-group-major units, vs the static x-smem panel (6)
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "all_sweep_variants" > gpurun_out/tail2_tests.txt 2>&1
JACOBI_LIB=check python probes/sanitize_small.py > gpurun_out/tail2_sanitize.txt 2>&1
for i in 1 2; do for v in 6 12; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c5; JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 2,8 graph 10; done; done > gpurun_out/tail2_rates.txt 2>&1
echo done
