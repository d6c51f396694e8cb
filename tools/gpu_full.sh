#!/bin/bash
# Full GPU pass: all GPU tests, smoke, bench (default + B=4096), per-role waits.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1
timeout 200 python bench.py --steps 10 --warmup 5 --batch 4096 --no-cpu-baseline --no-e2e > gpurun_out/bench_fused_4k.log 2>&1
BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 > gpurun_out/dbg.log 2>&1
