# c5 (fp32 A): CTA-kernel dynamic-tile instances vs the panel x-smem default
for v in 6 9 10 7; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c5; done > gpurun_out/c5var_r02.txt 2>&1
echo done
