for rep in 1 2; do
JACOBI_GRID_RES=0 timeout 120 python probes/size_sweep.py f64 3072,4096 400 | sed 's/^{/{"exp": "off", /'
timeout 120 python probes/size_sweep.py f64 3072,4096 400 | sed 's/^{/{"exp": "on", /'
JACOBI_GRID_RES_EXP=0 timeout 120 python probes/size_sweep.py f64 3072,4096 400 | sed 's/^{/{"exp": "smem-only", /'
JACOBI_GRID_RES_NOKEEP=1 timeout 120 python probes/size_sweep.py f64 3072,4096 400 | sed 's/^{/{"exp": "on-nokeepscale", /'
done > gpurun_out/res2.jsonl 2>&1
cut -c1-140 gpurun_out/res2.jsonl
