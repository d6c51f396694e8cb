#!/bin/bash
# Per-role barrier waits (BNN_FUSED_PROFILE=1/3/5) at B=256 and B=4096, plus an ncu --set full
# source-level capture of fused launch $LAUNCH (default 0) at B=256.
mkdir -p gpurun_out
for B in 256 4096; do
  for P in 1 3 5; do
    echo "== B=$B PROFILE=$P" >> gpurun_out/roles.log
    BNN_FUSED_PROFILE=$P timeout 120 python tools/prof_net.py $B >> gpurun_out/roles.log 2>&1
  done
done
L=${LAUNCH:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s $L -c 1 -o gpurun_out/prof_l$L -f python tools/prof_net.py 256 > gpurun_out/prof.log 2>&1
echo rc=$? >> gpurun_out/prof.log
