# keep pattern walked per unit position (per warp) instead of per tile
python probes/config_rates.py c2 > gpurun_out/keepwarp_r02.txt 2>&1
python probes/shard_rates.py c3 1,4,8 graph,persistent 40 >> gpurun_out/keepwarp_r02.txt 2>&1
python probes/size_sweep.py f64 2048,3072,4608,6144 200 >> gpurun_out/keepwarp_r02.txt 2>&1
echo done
