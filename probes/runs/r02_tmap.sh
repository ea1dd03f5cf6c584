# 2D-TMA-fed persistent solver (JACOBI_GRID_TMA=1): parity vs the graph path and the oracle, then rates
export JACOBI_GRID_TMA=1
timeout 300 python -m pytest tests/test_gridsync_gpu.py -q -x -k "bitwise_vs_graph or from_device" > gpurun_out/tmap_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/tmap_tests.log
for t in 0 1; do echo "tma $t"; JACOBI_GRID_TMA=$t timeout 120 python probes/config_rates.py c2; JACOBI_GRID_TMA=$t timeout 120 python probes/size_sweep.py f64 1024,2048,3072,4096 200; done > gpurun_out/tmap_rates.txt 2>&1
echo done
