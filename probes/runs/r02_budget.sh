# L2 keep budget sweep (fraction of the L2 kept with evict_last): c2 persistent solve, c3 shards, c3 whole
for b in 0.55 0.6 0.7 0.8; do echo "budget $b"; JACOBI_L2_BUDGET=$b python probes/config_rates.py c2; JACOBI_L2_BUDGET=$b python probes/shard_rates.py c3 1,4,8 graph,persistent 40; done
