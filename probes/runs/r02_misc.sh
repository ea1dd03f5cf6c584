# fp64 x staged in shared memory (panel x-smem, variant 6) vs the fp64 defaults; fresh ncu of the c5 kernel
for v in default 6; do echo "variant $v"; if [ "$v" = default ]; then unset JACOBI_SWEEP_VARIANT; else export JACOBI_SWEEP_VARIANT=$v; fi; python probes/config_rates.py c3,c4; done > gpurun_out/xsmem_fp64_r02.txt 2>&1
unset JACOBI_SWEEP_VARIANT
python probes/one_plan.py 131072 f32 3 > gpurun_out/plain_c5.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_sweep_panel -s 1 -c 1 -o gpurun_out/prof_c5_r02 -f python probes/one_plan.py 131072 f32 3 > gpurun_out/ncu_c5.log 2>&1
echo done
