#!/bin/bash
# Per-role barrier wait cycles of every fused launch (BNN_FUSED_PROFILE), B=4096:
# 1 = normal, 3 = producer skips A stores, 5 = epilogue skips math, 7 = both (results invalid).
mkdir -p gpurun_out
for m in 1 3 5 7; do
  echo "== BNN_FUSED_PROFILE=$m" >> gpurun_out/dbg.log
  BNN_FUSED_PROFILE=$m timeout 120 python tools/prof_net.py 4096 >> gpurun_out/dbg.log 2>&1
done
