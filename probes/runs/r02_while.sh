# device-side while loop of graph batches (conditional graph node) vs host-polled batches
for w in 0 1; do echo "graph_while $w"; JACOBI_GRAPH_WHILE=$w timeout 300 python probes/config_rates.py c3,c4; done > gpurun_out/while_r02.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gt_while.log 2>&1
echo done
