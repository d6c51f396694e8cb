#!/bin/bash
mkdir -p gpurun_out
L=${LAUNCH:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_layer -s $L -c 1 -o gpurun_out/prof_l$L -f python tools/prof_net.py 256 > gpurun_out/prof.log 2>&1
echo rc=$? >> gpurun_out/prof.log
