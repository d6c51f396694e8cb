#!/bin/bash
# bench line (default) + a second e2e sample
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-sweep --no-configs > gpurun_out/bench2.log 2>&1
