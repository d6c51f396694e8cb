#!/bin/bash
# ncu --set full of the halo4 launches of one forward (source counters for the stall analysis)
mkdir -p gpurun_out
B=${B:-1024}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"halo4" -c 4 -o gpurun_out/halo_b$B -f python tools/prof_net.py $B > gpurun_out/halo_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/halo_ncu.log
tail -3 gpurun_out/halo_ncu.log
