# per-CTA finish times of the static (6) and dynamic-tail (12) panel kernels at c5 size
for v in 6 12; do JACOBI_SWEEP_VARIANT=$v JACOBI_LIB=$PWD/probes/libjacobi_smt.so python probes/sm_times.py 131072 f32; done > gpurun_out/tail_smt.jsonl 2>&1
echo done
