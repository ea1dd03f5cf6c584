# per-CTA timeline of sweeps inside the persistent solver (probe build with -DJACOBI_SM_TIMING)
for n in c2 3072 2048; do JACOBI_LIB=$PWD/probes/libjacobi_smt.so python probes/grid_timeline.py $n; done > gpurun_out/grid_timeline_r02.jsonl 2>&1
echo done
