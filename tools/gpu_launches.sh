#!/bin/bash
# ncu launch list of one fused forward at batch ${B:-256} (cold, serialised) -> gpurun_out/launches_b$B.csv
mkdir -p gpurun_out
B=${B:-256}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels" --csv --log-file gpurun_out/launches_b$B.csv python tools/prof_net.py $B > /dev/null 2>&1
BNN_FUSED_SPLIT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels" --csv --log-file gpurun_out/launches_b${B}_nosplit.csv python tools/prof_net.py $B > /dev/null 2>&1
