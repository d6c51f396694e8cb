#!/bin/bash
mkdir -p gpurun_out
for P in 1 3 17 5; do
  for B in 256 4096; do
    echo "== B=$B PROFILE=$P" >> gpurun_out/roles.log
    BNN_FUSED_SWAP=2 BNN_FUSED_PROFILE=$P timeout 120 python tools/prof_net.py $B 2>&1 | grep -v "^ok" | head -6 >> gpurun_out/roles.log
  done
done
