#!/bin/bash
# One GPU-box pass: parity tests, smoke, GEMM kernel timings, bench line, ncu launch list.
# Usage (from this container): gpurun --timeout 1500 -- bash tools/gpu_check.sh
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_bench.log
timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/*.log
