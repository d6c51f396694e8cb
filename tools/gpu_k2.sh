#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "im2col or conv" > gpurun_out/k2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k2_pytest.log
tail -n 2 gpurun_out/k2_pytest.log
timeout 120 python tools/k2_time.py
