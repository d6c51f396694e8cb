#!/bin/bash
# ncu --set full of the K3 pipe probes and the standalone GEMM kernels (pipe utilisation counters)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"probe" -o gpurun_out/probes -f python tools/prof_kernel.py probes > gpurun_out/probes_ncu.log 2>&1
echo "probes rc=$?"
