#!/bin/bash
for r in 1 2 4 8; do echo "R=$r"; BNN_IM2COL_R=$r timeout 120 python tools/k2_time.py 2>&1 | head -3; done
