#!/bin/bash
mkdir -p gpurun_out
BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 256 2>&1 | grep "per-CTA" > gpurun_out/tl.log
timeout 120 python tools/timeline.py 256 0 >> gpurun_out/tl.log 2>&1
cat gpurun_out/tl.log
