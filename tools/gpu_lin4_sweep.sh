#!/bin/bash
# lin4 (NB, split) sweep at batch 256 through the launch timeline (fc1 / fc2 rows)
for f in "" "128,8" "256,8" "128,4" "256,4" "64,2" "64,1" "32,1" "16,1" "128,2"; do
  echo "== BNN_LIN4_FORCE=$f"
  BNN_LIN4_FORCE=$f timeout 120 python tools/timeline.py 256 2>&1 | grep "lin4"
done
