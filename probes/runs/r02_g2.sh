timeout 600 python probes/sweep_variants.py c5 10 6,12,13,14,6,12,13,14 > gpurun_out/g2_c5.jsonl 2>&1
cut -c1-330 gpurun_out/g2_c5.jsonl
