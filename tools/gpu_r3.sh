#!/bin/bash
# Full GPU parity suite, bench line, cfg4 per-layer, ncu --set full of the TMA-fed GEMM at 8192^3.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
for m in 1; do timeout 120 python tools/fc4_layers.py 1024; done > gpurun_out/fc4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"xnor4t|expand4" -c 3 -o gpurun_out/prof_xnor4t -f python tools/gemm_bench.py --kernels tma --iters 1 --shapes 8192,8192,8192 > gpurun_out/prof_xnor4t.log 2>&1; echo "ncu rc=$?"
