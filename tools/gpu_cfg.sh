#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.log 2>&1
