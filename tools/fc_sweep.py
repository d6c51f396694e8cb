"""fc1/fc2 per-layer event times at batch 256 under forced tile widths / split-K factors
(per-layer timing mode of bnn_net_forward; the convs run on whatever the forced tiling allows)."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_04477_b200 as bnn  # noqa: E402

lib = bnn.load()
B = 256
x = torch.empty((B, 3, 32, 32), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
bnn._lib.check(lib.bnn_fill_random_f32(bnn.mix64(1, 0x696E707574), 0, x.numel(), x.data_ptr(), s))
for bn, split in [(0, 0), (256, 16), (256, 8), (256, 4), (128, 16), (128, 8), (128, 4), (64, 8), (64, 4)]:
    lib.bnn_set_fused_tiling(1 if bn else 0, bn)
    lib.bnn_set_fused_split(split)
    net = bnn.Network(seed=1)
    n = len(net.layers)
    out = torch.empty((net.logits, B), dtype=torch.float32, device="cuda")
    for _ in range(3):
        net.forward_device(x, out)
    lib.bnn_net_set_timing(net.handle, 1)
    lib.bnn_net_reset_timing(net.handle)
    for _ in range(20):
        net.forward_device(x, out)
    torch.cuda.synchronize()
    lib.bnn_net_set_timing(net.handle, 0)
    lm, gm, gn = (C.c_double * n)(), (C.c_double * n)(), (C.c_size_t * n)()
    bnn._lib.check(lib.bnn_net_timing(net.handle, lm, gm, gn))
    print(json.dumps({"bn": bn, "split": split,
                      **{f"{i}:{net.layers[i]['kind']}": round(lm[i] / 20, 4) for i in range(n)
                         if lm[i] > 0 and net.layers[i]["kind"] == "linear"}}), flush=True)
lib.bnn_set_fused_tiling(0, 0)
lib.bnn_set_fused_split(0)
