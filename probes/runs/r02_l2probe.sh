# L2-hit streaming rate of the sweep's load flavours (16-96 MiB buffers stay L2-resident, 20 passes per
# launch) vs HBM (8 GiB)
for s in "16 mib" "48 mib" "64 mib" "96 mib" "8"; do echo "size $s"; probes/bwprobe $s; done > gpurun_out/l2probe_r02.txt 2>&1
echo done
