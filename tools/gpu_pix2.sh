#!/bin/bash
# full GPU suite + bench + launch list (pix_popc with PDL)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_pix.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs --no-sweep > gpurun_out/bench_pix_b.log 2>&1
tail -c 300 gpurun_out/bench_pix.log
