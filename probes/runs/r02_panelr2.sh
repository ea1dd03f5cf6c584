for v in 6 12 13; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c5; done > gpurun_out/panel_r2_r02.txt 2>&1
echo done
