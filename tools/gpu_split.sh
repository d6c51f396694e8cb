#!/bin/bash
mkdir -p gpurun_out
for S in 2 4 8 16; do
  echo "== split=$S" >> gpurun_out/tl.log; BNN_FUSED_SPLIT=$S BNN_FUSED_CHAIN_TAIL=0 timeout 120 python tools/timeline.py 256 0 2>&1 | grep -E "timeline  [5678]" >> gpurun_out/tl.log
  echo "== split=$S chain-tail" >> gpurun_out/tl.log; BNN_FUSED_SPLIT=$S timeout 120 python tools/timeline.py 256 0 2>&1 | grep -E "timeline  [5678]" >> gpurun_out/tl.log
done
