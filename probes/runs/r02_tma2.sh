# TMA-fed persistent solver: rows per tile (bulk copy size) R = 1 / 2 vs the LDG solver
for r in 1 2; do echo "tma R<=$r"; JACOBI_GRID_TMA=1 JACOBI_TMA_R=$r timeout 120 python probes/config_rates.py c2; JACOBI_GRID_TMA=1 JACOBI_TMA_R=$r timeout 120 python probes/size_sweep.py f64 2048,3072 200; done > gpurun_out/tma_rates2.txt 2>&1
JACOBI_GRID_TMA=1 JACOBI_TMA_R=1 timeout 300 python -m pytest tests/test_gridsync_gpu.py -q -x -k "bitwise_vs_graph" > gpurun_out/tma_tests2.log 2>&1
python probes/size_sweep.py f64 4096 50 > /dev/null 2>&1 && JACOBI_GRID_TMA=1 ncu --set full --clock-control none --cache-control none -k regex:k_solve_gridsync_tma -s 2 -c 1 -o gpurun_out/prof_c2_tma -f python probes/size_sweep.py f64 4096 50 > gpurun_out/ncu_tma.log 2>&1
echo done
