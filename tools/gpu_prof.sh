#!/bin/bash
# ncu --set full of the first two fused launches (conv0 float-input, conv1 pooled) at B=4096.
set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -c 2 -o gpurun_out/prof_fused -f python tools/prof_net.py 4096 > gpurun_out/prof.log 2>&1
echo rc=$? >> gpurun_out/prof.log
