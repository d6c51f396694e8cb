#!/bin/bash
# halo-conv design probe (tools/halo_probe.cu), compiled on the box
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_04477_b200/csrc tools/halo_probe.cu -o /tmp/halo_probe -lcuda && timeout 120 /tmp/halo_probe > gpurun_out/halo_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/halo_probe.log
cat gpurun_out/halo_probe.log
