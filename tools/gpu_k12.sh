#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cpp_api.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 300 python tools/gemm_bench.py --shapes 1024,1024,1024 2048,2048,2048 4096,1024,4096 1000,1024,4096 4096,1024,9216 64,1024,576 128,4096,1152 > gpurun_out/gemm.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-sweep > gpurun_out/bench.log 2>&1
