#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cpp_api.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-sweep --no-cpu-baseline > gpurun_out/bench.log 2>&1
