#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/split_sweep.txt
for sp in 0 1 2 4 8 16; do
  BNN_FUSED_SPLIT=$sp timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused" --csv --log-file gpurun_out/l_$sp.csv python tools/prof_net.py 256 > /dev/null 2>&1
  echo "split=$sp" >> gpurun_out/split_sweep.txt
  grep -o '"[0-9,]*"$' gpurun_out/l_$sp.csv | tr -d '",' | tr '\n' ' ' >> gpurun_out/split_sweep.txt; echo >> gpurun_out/split_sweep.txt
done
