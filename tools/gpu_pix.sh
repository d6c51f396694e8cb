#!/bin/bash
# CUDA-core pixel conv (pix_popc_kernel): fused parity on the default network + pixel topologies
# (with and without it), then the bench line and the launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x --timeout 300 -p no:cacheprovider -k "auto or nopixpopc or pixf32" > gpurun_out/pytest_pix.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pix.log
tail -3 gpurun_out/pytest_pix.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_pix.log 2>&1
BNN_PIX_POPC=0 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs --no-sweep > gpurun_out/bench_nopix.log 2>&1
BNN_PIX_POPC=2 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs --no-sweep > gpurun_out/bench_pix2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_popc" -c 40 --csv --log-file gpurun_out/launches_pix.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
tail -c 600 gpurun_out/bench_pix.log; tail -c 300 gpurun_out/bench_nopix.log
