#!/bin/bash
# lin4 per-phase stamps (BNN_LIN4_PROFILE) for the default network's linear stages and cfg4
mkdir -p gpurun_out
for B in 256 1024; do BNN_LIN4_PROFILE=1 REPS=3 timeout 120 python tools/prof_net.py $B 2>&1 | grep lin4 | tail -n 2; done > gpurun_out/lin4_prof.log
cat gpurun_out/lin4_prof.log
