#!/bin/bash
mkdir -p gpurun_out
for P in 0 1 2; do
  echo "== pdl=$P" >> gpurun_out/tl.log; BNN_PDL=$P timeout 120 python tools/timeline.py 256 0 2>&1 >> gpurun_out/tl.log
  BNN_PDL=$P timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_pdl$P.log 2>&1
done
