#!/bin/bash
# ncu --set full of the standalone operator kernels (K2 im2col, K3 popc / xnor4, the batch-1 conv)
mkdir -p gpurun_out
for w in im2col gemm_popc gemm_xnor4 conv_b1; do
  timeout 600 ncu --set full --clock-control none --import-source on -c 4 -o gpurun_out/ops_$w -f python tools/prof_kernel.py $w > gpurun_out/ops_ncu_$w.log 2>&1
  echo "$w rc=$?"
done
