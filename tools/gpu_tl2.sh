#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/timeline.py 256 0 > gpurun_out/tl.log 2>&1
BNN_FUSED_SPLIT=1 timeout 120 python tools/timeline.py 256 0 >> gpurun_out/tl.log 2>&1
