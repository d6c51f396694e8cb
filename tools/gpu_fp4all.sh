#!/bin/bash
mkdir -p gpurun_out
BNN_FUSED_FP4=2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_fp4all.log 2>&1
echo "== fp4all" >> gpurun_out/roles.log
BNN_FUSED_FP4=2 BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 2>&1 | grep -v "^ok" >> gpurun_out/roles.log
