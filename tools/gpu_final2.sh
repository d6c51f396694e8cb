#!/bin/bash
# memcheck over every engine setting, then the round-end evidence (tools/gpu_final.sh)
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize.py > gpurun_out/san.log 2>&1; echo "rc=$?" >> gpurun_out/san.log
tail -3 gpurun_out/san.log
bash tools/gpu_final.sh
