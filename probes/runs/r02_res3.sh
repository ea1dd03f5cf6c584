for rep in 1 2; do
JACOBI_GRID_RES=0 timeout 120 python probes/size_sweep.py f64 4096 400 | sed 's/^{/{"exp": "off", /'
JACOBI_GRID_RES=0 JACOBI_GRID_SMEM_PAD=65536 timeout 120 python probes/size_sweep.py f64 4096 400 | sed 's/^{/{"exp": "pad64k", /'
JACOBI_GRID_RES=0 JACOBI_GRID_SMEM_PAD=131072 timeout 120 python probes/size_sweep.py f64 4096 400 | sed 's/^{/{"exp": "pad128k", /'
JACOBI_GRID_RES=0 JACOBI_GRID_SMEM_PAD=196608 timeout 120 python probes/size_sweep.py f64 4096 400 | sed 's/^{/{"exp": "pad192k", /'
done > gpurun_out/res3.jsonl 2>&1
cut -c1-140 gpurun_out/res3.jsonl
