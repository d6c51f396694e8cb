"""One fused-engine forward of the default network at batch B (for ncu captures).

    python tools/prof_net.py [B] [engine]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_04477_b200 as bnn  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
net = bnn.Network(seed=1)
if len(sys.argv) > 2:
    net.set_engine(sys.argv[2])
s = torch.cuda.current_stream().cuda_stream
x = torch.empty((B, 3, 32, 32), dtype=torch.float32, device="cuda")
bnn._lib.check(bnn.load().bnn_fill_random_f32(bnn.mix64(1, 0x696E707574), 0, x.numel(), x.data_ptr(), s))
# REPS forwards (profile counters print per launch: the first forward is cold — TLB, L2)
for _ in range(int(os.environ.get("REPS", "1"))):
    out = net.forward_device(x)
torch.cuda.synchronize()
print("ok", out.shape, net.engine)
