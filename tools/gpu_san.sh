#!/bin/bash
# compute-sanitizer over the fused engine: memcheck on every engine setting (tools/sanitize.py),
# racecheck and synccheck on the default setting (quick), then the GPU test-suite
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize.py quick > gpurun_out/san_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py quick > gpurun_out/san_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck.log
tail -n 3 gpurun_out/san_memcheck.log gpurun_out/san_racecheck.log gpurun_out/san_synccheck.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
