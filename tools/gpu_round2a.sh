#!/bin/bash
# New-tests pass + bench on one B200
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_harness_gpu.py tests/test_bench_parity_gpu.py tests/test_cpp_api.py tests/test_control_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_new.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_new.log
./paper_1911_04477_b200/bin/test_cpp_api . > gpurun_out/cpp_api.log 2>&1; echo "rc=$?" >> gpurun_out/cpp_api.log
timeout 600 python bench.py > gpurun_out/bench_r2a.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2a.log 2>&1
tail -2 gpurun_out/pytest_new.log
