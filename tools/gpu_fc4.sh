#!/bin/bash
mkdir -p gpurun_out
for m in 0 1; do BNN_LIN4_TMA=$m timeout 120 python tools/fc4_layers.py 1024; done > gpurun_out/fc4.log 2>&1
BNN_LIN4_TMA=1 BNN_LIN4_PROFILE=1 timeout 120 python tools/fc4_layers.py 1024 >> gpurun_out/fc4.log 2>&1
timeout 600 python -m pytest tests/test_halo_lin4_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "lin4_tma" >> gpurun_out/fc4.log 2>&1
grep -v "^\[lin4" gpurun_out/fc4.log | tail -5; grep "^\[lin4" gpurun_out/fc4.log | sort | uniq -c | sort -rn | head -4
