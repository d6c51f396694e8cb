#!/bin/bash
mkdir -p gpurun_out
for P in 1 3; do
  for F in 0 2; do
    echo "== PROFILE=$P fp4=$F swap=2" >> gpurun_out/roles.log
    BNN_FUSED_SWAP=2 BNN_FUSED_FP4=$F BNN_FUSED_PROFILE=$P timeout 120 python tools/prof_net.py 4096 2>&1 | grep "swap" >> gpurun_out/roles.log
  done
done
