# system-scope reductions in the fused exchange's signal: parity of every fused path + shard timing
timeout 900 python -m pytest tests -m gpu -q -k "fused or persistent_fused or silent_peer or multi_gpu or bench_distributed" > gpurun_out/gt_sysred.log 2>&1
python probes/shard_rates.py c3 1,8 persistent-push 40 > gpurun_out/sysred_shard.jsonl 2>&1
echo done
