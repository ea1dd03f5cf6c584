python -m pytest tests/test_parity_gpu.py -q -x -k "group or variant or c5_full" > gpurun_out/group4_tests.log 2>&1; tail -3 gpurun_out/group4_tests.log
JACOBI_LIB=check timeout 600 python probes/sanitize_small.py > gpurun_out/group4_sanitize.log 2>&1; echo "sanitize rc=$?"; tail -1 gpurun_out/group4_sanitize.log
python probes/shard_rates.py c5 1,2,4,8 graph 100 > gpurun_out/shard_rates_r02_v5_c5.jsonl 2>&1
cut -c1-220 gpurun_out/shard_rates_r02_v5_c5.jsonl
