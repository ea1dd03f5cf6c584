# panel kernel, one row per warp with 8 column steps in flight (variant 11) vs the fp32 default (6)
for v in 6 11; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c5; JACOBI_SWEEP_VARIANT=$v python probes/shard_rates.py c5 2,8 graph 10; done > gpurun_out/panel_r1_r02.txt 2>&1
for v in 10 11; do echo "variant $v"; JACOBI_SWEEP_VARIANT=$v python probes/config_rates.py c4; done >> gpurun_out/panel_r1_r02.txt 2>&1
echo done
