"""Launch timeline of the fused engine (bnn_debug_timeline): per launch, the min/median/max over
CTAs of four globaltimer stamps, in us from the first stamp.

    python tools/timeline.py [B] [fc4]   (fc4: the FC stack 9216 -> 4096 -> 4096 -> 1000)
k0 entry, k1 after the TMEM dealloc (last), k2 griddepcontrol.wait returned, k3 roles done.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_04477_b200 as bnn  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
lib = bnn.load()
FC4 = len(sys.argv) > 2 and sys.argv[2] == "fc4"
if FC4:
    net = bnn.Network([{"kind": "linear", "out_features": 4096}, {"kind": "linear", "out_features": 4096},
                       {"kind": "linear", "out_features": 1000}], (9216, 1, 1), 1)
else:
    net = bnn.Network(seed=1)
s = torch.cuda.current_stream().cuda_stream  # legacy stream: eager launches (no graph)
x = torch.empty((B, 9216, 1, 1) if FC4 else (B, 3, 32, 32), dtype=torch.float32, device="cuda")
bnn._lib.check(lib.bnn_fill_random_f32(bnn.mix64(1, 0x696E707574), 0, x.numel(), x.data_ptr(), s))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    net.forward_device(x)
torch.cuda.synchronize()
flush.fill_(1.0)
torch.cuda.synchronize()
lib.bnn_debug_timeline(1)
net.forward_device(x)
lib.bnn_debug_timeline(2)
torch.cuda.synchronize()
print("ok", B, net.engine, lib.bnn_last_gemm_kernel().decode())
