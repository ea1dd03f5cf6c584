python -m pytest tests/test_parity_gpu.py -q -x -k "group" > gpurun_out/fewrows_tests.log 2>&1; tail -2 gpurun_out/fewrows_tests.log
JACOBI_LIB=check timeout 900 python probes/sanitize_small.py > gpurun_out/fewrows_sanitize.log 2>&1; echo "sanitize rc=$?"; grep -E "^(300|149) " gpurun_out/fewrows_sanitize.log; tail -1 gpurun_out/fewrows_sanitize.log
