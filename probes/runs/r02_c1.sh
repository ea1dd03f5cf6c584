timeout 300 python probes/solve_latency.py > gpurun_out/c1_lat.jsonl 2>&1
cat gpurun_out/c1_lat.jsonl
timeout 300 python probes/size_sweep.py f64 256 400 2>&1 | cut -c1-200
timeout 300 python probes/size_sweep.py f64 256 2000 2>&1 | cut -c1-200
