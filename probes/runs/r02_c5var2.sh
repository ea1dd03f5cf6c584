# c5: every fp32-capable sweep variant on the final code (burst launches + a sustained 100-sweep solve)
python probes/sweep_variants.py c5 10 6,5,10,9,7,3,2,0,6 > gpurun_out/c5_variants_r02b.jsonl 2>&1
echo done
