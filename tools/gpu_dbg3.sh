#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x -k "split16" --timeout 120 -p no:cacheprovider > gpurun_out/p1.log 2>&1; echo "rc=$?" >> gpurun_out/p1.log
timeout 600 python -m pytest "tests/test_fused_gpu.py::test_default_network_fused_vs_oracle" -q -x --timeout 120 -p no:cacheprovider > gpurun_out/p2.log 2>&1; echo "rc=$?" >> gpurun_out/p2.log
cat > /tmp/one.py <<'PY'
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1911_04477_b200 as bnn
from oracle import Oracle
orc = Oracle(); lib = bnn.load()
lib.bnn_set_fused_split(16)
net = bnn.Network(seed=1); net.set_engine("fused")
x = orc.fill_random((1, 3, 32, 32), orc.mix64(1, 0x696E707574))
print(np.array_equal(net.forward(x), orc.net(seed=1).forward(x)))
PY
timeout 300 compute-sanitizer --tool memcheck python /tmp/one.py > gpurun_out/san.log 2>&1; echo "rc=$?" >> gpurun_out/san.log
