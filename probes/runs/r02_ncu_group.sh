# ncu --set full of the c5 P = 8 shard kernel: the group kernel (default) and the panel kernel (6)
timeout 300 python probes/shard_rates.py c5 8 graph 4 > gpurun_out/plain_c5p8.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_group -s 2 -c 1 -o gpurun_out/prof_c5p8_group_r02 -f python probes/shard_rates.py c5 8 graph 4 > gpurun_out/ncu_c5p8g.log 2>&1
JACOBI_SWEEP_VARIANT=6 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_panel -s 2 -c 1 -o gpurun_out/prof_c5p8_panel_r02 -f python probes/shard_rates.py c5 8 graph 4 > gpurun_out/ncu_c5p8p.log 2>&1
tail -3 gpurun_out/ncu_c5p8g.log gpurun_out/ncu_c5p8p.log; ls -la gpurun_out/*.ncu-rep
