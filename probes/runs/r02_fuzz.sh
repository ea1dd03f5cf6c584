# extended randomized parity: the test generator's cases (more seeds) and larger ragged sizes
python probes/fuzz_more.py 7000 400 > gpurun_out/fuzz_more_r02.txt 2>&1
python probes/fuzz_large.py 100 30 > gpurun_out/fuzz_large_r02.txt 2>&1
echo done
