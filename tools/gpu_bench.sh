#!/bin/bash
# fused tests + bench line (default) + B=4096 line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --batch 4096 --steps 20 --no-cpu-baseline --no-sweep > gpurun_out/bench_4k.log 2>&1
