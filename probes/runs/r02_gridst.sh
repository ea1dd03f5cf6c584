# persistent solver: stop-test parameters in registers, one CTA barrier less per sweep (max norm)
python probes/config_rates.py c2 > gpurun_out/gridst_r02.txt 2>&1
python probes/size_sweep.py f64 640,1024,2048,3072,4096 400 >> gpurun_out/gridst_r02.txt 2>&1
python probes/shard_rates.py c3 8 persistent,persistent-push 40 >> gpurun_out/gridst_r02.txt 2>&1
timeout 600 python -m pytest tests/test_gridsync_gpu.py tests/test_fuzz_gpu.py -m gpu -q > gpurun_out/gt_gridst.log 2>&1
echo done
