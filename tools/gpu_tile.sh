#!/bin/bash
# pix_tile_kernel (float input staged through shared memory) parity + A/B bench vs the packer path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -q -x --timeout 300 -p no:cacheprovider -k "auto or pixf32 or nopixpopc" > gpurun_out/pytest_tile.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tile.log
tail -3 gpurun_out/pytest_tile.log
BNN_PIX_POPC=1 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench_tile.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs --no-sweep > gpurun_out/bench_pack.log 2>&1
BNN_PIX_POPC=1 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --no-configs --no-sweep > gpurun_out/bench_tile2.log 2>&1
BNN_PIX_POPC=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_" -c 20 --csv --log-file gpurun_out/launches_tile.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
