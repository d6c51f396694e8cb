#!/bin/bash
mkdir -p gpurun_out
timeout 120 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
for S in 1 0; do
BNN_FUSED_SWAP=$S timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_swap$S.log 2>&1
done
