# speed-weighted static split (JACOBI_SM_WEIGHTS): rates off/on, then the GPU suite with the default
for rep in 1 2; do for w in 0 1; do echo "sm_weights $w rep $rep"; JACOBI_SM_WEIGHTS=$w timeout 300 python probes/config_rates.py c3,c5; JACOBI_SM_WEIGHTS=$w timeout 120 python probes/config_rates.py c2; done; done > gpurun_out/smw_r02.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gt_smw.log 2>&1
echo done
