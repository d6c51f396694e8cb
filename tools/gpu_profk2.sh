#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:im2col -s 1 -c 1 -o gpurun_out/prof_im2col -f python tools/prof_kernel.py im2col > gpurun_out/prof.log 2>&1
echo rc=$? >> gpurun_out/prof.log
