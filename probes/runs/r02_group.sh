# group kernel (variants 12: G2, 13: G4) vs the panel default (6) on c5 shards; parity + bounds first
python -m pytest tests/test_parity_gpu.py -q -x -k "variant" > gpurun_out/group_tests.log 2>&1; tail -2 gpurun_out/group_tests.log
JACOBI_LIB=check timeout 600 python probes/sanitize_small.py > gpurun_out/group_sanitize.log 2>&1; echo "sanitize rc=$?"; tail -3 gpurun_out/group_sanitize.log
for v in 6 12 13 6 12 13; do JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 1,2,4,8 graph 10; done > gpurun_out/group_c5.jsonl 2>&1
cut -c1-230 gpurun_out/group_c5.jsonl
