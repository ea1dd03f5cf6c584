python -m pytest tests/test_parity_gpu.py -q -x -k "variant" > gpurun_out/group2_tests.log 2>&1; tail -2 gpurun_out/group2_tests.log
JACOBI_LIB=check timeout 600 python probes/sanitize_small.py > gpurun_out/group2_sanitize.log 2>&1; echo "sanitize rc=$?"; tail -1 gpurun_out/group2_sanitize.log
for v in 6 13 14 15; do JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 1,2,4,8 graph 10; done > gpurun_out/group2_c5.jsonl 2>&1
python probes/sweep_variants.py c5 10 6,13,14,15,6,13 > gpurun_out/group2_c5_sust.jsonl 2>&1
python probes/sweep_variants.py c3 40 7,13,14,7,13,14 > gpurun_out/group2_c3.jsonl 2>&1
cut -c1-200 gpurun_out/group2_c5.jsonl; cut -c1-330 gpurun_out/group2_c5_sust.jsonl gpurun_out/group2_c3.jsonl
