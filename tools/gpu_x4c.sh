#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "gemm or conv_large" > gpurun_out/x4c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/x4c_pytest.log
tail -n 2 gpurun_out/x4c_pytest.log
for c in 1 2; do echo "cluster=$c"; BNN_XNOR4T_CLUSTER=$c timeout 300 python tools/gemm_bench.py --kernels tma --shapes 8192,8192,8192 4096,1024,9216 16384,16384,16384 4096,4096,4096 1000,1024,4096 2>&1; done
