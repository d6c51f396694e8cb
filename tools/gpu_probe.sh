#!/bin/bash
# tcgen05 dispatch-rate microbenchmark (tools/mma_probe.cu), compiled on the box
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_04477_b200/csrc tools/mma_probe.cu -o /tmp/mma_probe -lcuda && timeout 120 /tmp/mma_probe > gpurun_out/mma_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/mma_probe.log
