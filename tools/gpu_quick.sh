#!/bin/bash
# Fused parity tests + bench B=256/4096 + per-role waits (dev loop).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1
timeout 200 python bench.py --steps 10 --warmup 5 --batch 4096 --no-cpu-baseline --no-e2e > gpurun_out/bench_fused_4k.log 2>&1
BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 > gpurun_out/dbg.log 2>&1
