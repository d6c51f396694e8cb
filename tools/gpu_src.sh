#!/bin/bash
# ncu --set full with source of the FP4 conv1 launch (swap4 cg=1) and conv0 at batch 256.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"swap" -c 3 -o gpurun_out/src256 -f python tools/prof_net.py 256 > gpurun_out/src.log 2>&1
echo "rc=$?" >> gpurun_out/src.log; tail -3 gpurun_out/src.log
