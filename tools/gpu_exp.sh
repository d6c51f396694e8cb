#!/bin/bash
# Experiments: timeline with split-K on/off; producer store / wait::st knock-outs (role clocks).
mkdir -p gpurun_out
echo "== default" >> gpurun_out/tl.log; timeout 120 python tools/timeline.py 256 0 >> gpurun_out/tl.log 2>&1
echo "== nosplit" >> gpurun_out/tl.log; BNN_FUSED_SPLIT=1 timeout 120 python tools/timeline.py 256 0 >> gpurun_out/tl.log 2>&1
for P in 1 3 17 5; do
  for B in 256 4096; do
    echo "== B=$B PROFILE=$P" >> gpurun_out/roles.log
    BNN_FUSED_PROFILE=$P timeout 120 python tools/prof_net.py $B >> gpurun_out/roles.log 2>&1
  done
done
