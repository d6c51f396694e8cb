#!/bin/bash
# TMA-fed FP4 GEMM (xnor4t_kernel): parity subset + kernel times vs the in-CTA-expansion kernel.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "gemm or conv_large" --timeout 300 -p no:cacheprovider > gpurun_out/tma_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/tma_pytest.log
timeout 300 python tools/gemm_bench.py --kernels umma,tma --shapes 1024,1024,1024 4096,1024,9216 1000,1024,4096 4096,4096,4096 128,262144,1152 8192,8192,8192 16384,16384,16384 2048,2048,2048 > gpurun_out/tma_bench.jsonl 2>&1
tail -n 3 gpurun_out/tma_pytest.log; cat gpurun_out/tma_bench.jsonl
