#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
for T in 1 0; do
  echo "== tail=$T" >> gpurun_out/tl.log; BNN_FUSED_CHAIN_TAIL=$T timeout 120 python tools/timeline.py 256 0 >> gpurun_out/tl.log 2>&1
  BNN_FUSED_CHAIN_TAIL=$T timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_tail$T.log 2>&1
done
echo "== full chain" >> gpurun_out/tl.log; timeout 120 python tools/timeline.py 256 1 >> gpurun_out/tl.log 2>&1
BNN_FUSED_CHAIN=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/bench_chain.log 2>&1
