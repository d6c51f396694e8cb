#!/bin/bash
# launch list of the bench's launches (pix_tile included) + ncu --set full of pix_tile_kernel
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pix_ -c 1 -o gpurun_out/prof_tile -f python tools/prof_net.py 256 > gpurun_out/prof_tile.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_tile.log
