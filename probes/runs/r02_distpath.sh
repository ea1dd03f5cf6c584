# N > 1 code paths on one GPU: multi-process parity harness at P = 1, bench.py's distributed path + fused leg
python -m pytest tests/test_multigpu_gpu.py -m gpu -q -rs > gpurun_out/multigpu_p1.log 2>&1
python bench.py --force-dist --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_forcedist.jsonl 2> gpurun_out/bench_forcedist.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --exchange p2p --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_forcedist_p2p.jsonl 2> gpurun_out/bench_forcedist_p2p.err
echo done
