#!/bin/bash
# Per-role barrier wait cycles of every fused launch (BNN_FUSED_PROFILE), B=4096:
# 1 = normal, 3 = producer skips A stores, 5 = epilogue skips math, 7 = both (results invalid).
mkdir -p gpurun_out
rm -f gpurun_out/dbg.log
for cg in ${CGS:-1 2}; do for m in 1 3 7; do
  echo "== CG=$cg BNN_FUSED_PROFILE=$m" >> gpurun_out/dbg.log
  BNN_FUSED_CG=$cg BNN_FUSED_PROFILE=$m timeout 120 python tools/prof_net.py 4096 2>&1 | grep "KB=9\|KB=18\|KB=1 " >> gpurun_out/dbg.log
done; done
