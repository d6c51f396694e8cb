#!/bin/bash
# iteration: parity subset of the touched kernels, their timings, and an ncu capture of K2 im2col
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_halo_lin4_gpu.py tests/test_fused_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "gemm or conv_large or lin4 or default_network_fused" > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
tail -n 2 gpurun_out/it_pytest.log
timeout 300 python tools/gemm_bench.py --kernels tma --shapes 8192,8192,8192 4096,1024,9216 16384,16384,16384 2>&1
for i in 1 2; do timeout 120 python tools/fc4_layers.py 1024; done 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -c 2 -o gpurun_out/ops_im2col -f python tools/prof_kernel.py im2col > gpurun_out/ops_ncu_im2col.log 2>&1; echo "ncu rc=$?"
