#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_control_gpu.py tests/test_io.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_ctl.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ctl.log
