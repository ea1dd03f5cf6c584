# cp.async variants of the asynchronous-copy persistent sweep: cache hint / none / .ca / L2::128B
export JACOBI_PERSIST=1 JACOBI_GRID_ASYNC=1
for m in 0 1 2 3; do
  if [ $m = 0 ]; then L=""; else L=$PWD/probes/libjacobi_cpa$m.so; fi
  echo "mode $m"; JACOBI_LIB=$L python probes/size_sweep.py f64 4096,8192 200
  JACOBI_LIB=$L timeout 600 ncu --metrics lts__t_sectors_srcunit_tex.sum,l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum,gpu__time_duration.sum --clock-control none -k regex:k_solve_gridsync -c 1 python probes/size_sweep.py f64 4096 100 2>&1 | grep -E "sectors|duration"
done > gpurun_out/cpa_modes.txt 2>&1
echo done
