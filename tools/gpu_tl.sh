#!/bin/bash
# Timelines (per-layer launches and the chained kernel) at B=256 and 4096 + bench of both.
mkdir -p gpurun_out
for B in 256 4096; do
  for C in 0 1; do
    echo "== B=$B chain=$C" >> gpurun_out/tl.log
    timeout 120 python tools/timeline.py $B $C >> gpurun_out/tl.log 2>&1
  done
done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_chain.log 2>&1
BNN_FUSED_CHAIN=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_perlayer.log 2>&1
