#!/bin/bash
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/fp4_one.py 1 > gpurun_out/san_fp4.log 2>&1; echo "rc=$?" >> gpurun_out/san_fp4.log
