"""cfg4 (FC stack 9216 -> 4096 -> 4096 -> 1000, batch 1024): per-layer event times (ms) of the
fused engine, and the lin4 phase stamps when BNN_LIN4_PROFILE is set.
    python tools/fc4_layers.py [batch]"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_04477_b200 as bnn  # noqa: E402

lib = bnn.load()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
FC = [{"kind": "linear", "out_features": 4096}, {"kind": "linear", "out_features": 4096},
      {"kind": "linear", "out_features": 1000}]
net = bnn.Network(FC, (9216, 1, 1), 1)
s = torch.cuda.current_stream().cuda_stream
x = torch.empty((B, 9216, 1, 1), dtype=torch.float32, device="cuda")
bnn._lib.check(lib.bnn_fill_random_f32(bnn.mix64(1, 0x696E707574), 0, x.numel(), x.data_ptr(), s))
out = torch.empty((1000, B), dtype=torch.float32, device="cuda")
for _ in range(3):
    net.forward_device(x, out)
n = len(net.layers)
lib.bnn_net_set_timing(net.handle, 1)
lib.bnn_net_reset_timing(net.handle)
R = 20
for _ in range(R):
    net.forward_device(x, out)
torch.cuda.synchronize()
lib.bnn_net_set_timing(net.handle, 0)
lm, gm, gn = (C.c_double * n)(), (C.c_double * n)(), (C.c_size_t * n)()
bnn._lib.check(lib.bnn_net_timing(net.handle, lm, gm, gn))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    net.forward_device(x, out)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"batch": B, "forward_ms": round(e0.elapsed_time(e1) / R, 4),
                  "layers_ms": {f"{i}": round(lm[i] / R, 4) for i in range(n)},
                  "gemm_ms": {f"{i}": round(gm[i] / R, 4) for i in range(n)},
                  "kernels": [lib.bnn_net_layer_kernel(net.handle, i).decode() for i in range(n)]}), flush=True)
