#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x -k "fp4" --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fp4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fp4.log
for F in 1 2; do
BNN_FUSED_FP4=$F timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_fp4_$F.log 2>&1
done
for F in 1 2; do
  echo "== fp4=$F" >> gpurun_out/roles.log
  BNN_FUSED_FP4=$F BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 >> gpurun_out/roles.log 2>&1
done
