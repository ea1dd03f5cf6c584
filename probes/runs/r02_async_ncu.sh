# one --set full capture of the asynchronous-copy persistent solver (c2 shape) and of the register one
export JACOBI_PERSIST=1
for a in 1 0; do
JACOBI_GRID_ASYNC=$a timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve_gridsync -c 1 \
  -o gpurun_out/grid_async$a python probes/size_sweep.py f64 4096 100 > gpurun_out/grid_async_ncu$a.log 2>&1
done
echo done
