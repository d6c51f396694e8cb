#!/bin/bash
# ncu --set full of fused launch $LAUNCH (default 3 = conv3, BN=256) at B=4096.
mkdir -p gpurun_out
L=${LAUNCH:-3}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s $L -c 1 -o gpurun_out/prof_fused_l$L -f python tools/prof_net.py 4096 > gpurun_out/prof.log 2>&1
echo rc=$? >> gpurun_out/prof.log
