#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_halo_lin4_gpu.py tests/test_fused_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "gemm or conv_large or lin4 or default_network_fused" > gpurun_out/l4c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l4c_pytest.log
tail -n 2 gpurun_out/l4c_pytest.log
for c in 1 2; do echo "cluster=$c"; BNN_LIN4_CLUSTER=$c timeout 120 python tools/fc4_layers.py 1024; BNN_LIN4_CLUSTER=$c timeout 120 python tools/timeline.py 1024 fc4 | head -3; done 2>&1
