# release fences (fence.acq_rel) instead of fence.sc in the grid barrier and the fused exchange signal
python probes/config_rates.py c2 > gpurun_out/fence_r02.txt 2>&1
python probes/size_sweep.py f64 1024,2048,3072 400 >> gpurun_out/fence_r02.txt 2>&1
python probes/shard_rates.py c3 8 persistent,persistent-push 40 >> gpurun_out/fence_r02.txt 2>&1
timeout 900 python -m pytest tests/test_gridsync_gpu.py tests/test_fuzz_gpu.py -m gpu -q > gpurun_out/gt_fence.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "fused or persistent_fused or silent_peer" >> gpurun_out/gt_fence.log 2>&1
echo done
