# bounds-checked build over every round-2 sweep variant (sanitize cases with round-2 variant indices)
timeout 900 python -m pytest tests/test_bounds_gpu.py -x -q > gpurun_out/bounds_tests.txt 2>&1
JACOBI_LIB=check python probes/sanitize_small.py > gpurun_out/bounds_sanitize.txt 2>&1
echo done
