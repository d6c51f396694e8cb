#!/bin/bash
for pf in 0 1; do for c in 1 2; do echo "prefetch=$pf cluster=$c"; BNN_LIN4_PREFETCH=$pf BNN_LIN4_CLUSTER=$c timeout 120 python tools/timeline.py 1024 fc4 | head -3; BNN_LIN4_PREFETCH=$pf BNN_LIN4_CLUSTER=$c timeout 120 python tools/timeline.py 256 | sed -n 6,7p; done; done 2>&1
