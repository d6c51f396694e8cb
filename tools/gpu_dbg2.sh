#!/bin/bash
mkdir -p gpurun_out
for bn in 64 128 256; do for m in 1 7; do
  echo "== BN=$bn PROFILE=$m" >> gpurun_out/dbg2.log
  BNN_FUSED_BN=$bn BNN_FUSED_PROFILE=$m timeout 120 python tools/prof_net.py 4096 2>&1 | grep "KB=18\|KB=9 " >> gpurun_out/dbg2.log
done; done
