#!/bin/bash
# Per-role wait cycles of every fused launch at the bench batch (and 4096), stores on / off.
mkdir -p gpurun_out
for B in 256 4096; do for m in 1 3; do
  echo "== B=$B profile=$m"; BNN_FUSED_PROFILE=$m timeout 120 python tools/prof_net.py $B 2>&1 | grep "per-CTA"
done; done > gpurun_out/roles256.log 2>&1
timeout 120 python tools/timeline.py 256 0 > gpurun_out/timeline256.log 2>&1
cat gpurun_out/roles256.log; cat gpurun_out/timeline256.log | tail -12
