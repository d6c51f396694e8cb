#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x -k "auto or fp4all or nofp4" --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
for N in 240 192; do
BNN_FP4_NP=$N timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_np$N.log 2>&1
echo "== NP=$N" >> gpurun_out/roles.log
BNN_FP4_NP=$N BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 2>&1 | grep swap4 >> gpurun_out/roles.log
done
