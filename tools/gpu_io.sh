#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_io.py tests/test_cpp_api.py tests/test_abi.py -q -x --timeout 200 -p no:cacheprovider > gpurun_out/pytest_io.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_io.log
