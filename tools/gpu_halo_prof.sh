#!/bin/bash
# per-role cycle counters of the halo4 launches (BNN_HALO_PROFILE=1 + 2*mode: 1 no epilogue,
# 2 no halo fill, 4 no MMA; modes != 0 give invalid results)
mkdir -p gpurun_out
for B in ${BATCHES:-256 4096}; do for M in ${MODES:-0 1 3 4 6}; do
  BNN_HALO_PROFILE=$((1 + 2*M)) REPS=3 timeout 120 python tools/prof_net.py $B 2>&1 | grep halo4 | tail -n 4
done; done > gpurun_out/halo_prof.log 2>&1
cat gpurun_out/halo_prof.log | sed -e 's/per-CTA kcyc//' | cut -c1-330
