# per-CTA work of the persistent solver vs rows and SM (probe build with -DJACOBI_SM_TIMING)
for n in c2 4000 3700; do JACOBI_LIB=$PWD/probes/libjacobi_smt.so python probes/grid_timeline.py $n; done > gpurun_out/grid_timeline2_r02.jsonl 2>&1
echo done
