"""K2 binary im2col at the bench shape (x [256,128,32,32] f32 -> 262144 lines x 36 words): ms per
launch (CUDA events, input > L2) and achieved GB/s of the algorithmic bytes."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_04477_b200 as bnn  # noqa: E402
from paper_1911_04477_b200 import _lib  # noqa: E402

lib = bnn.load()
S = torch.cuda.current_stream().cuda_stream
for (B, Cc, H, W) in ((256, 128, 32, 32), (256, 256, 16, 16), (256, 64, 32, 32)):
    g = _lib.ConvGeom(3, 3, 1, 1, 1, 1, Cc, Cc)
    x = torch.randn((B, Cc, H, W), device="cuda")
    wpl = (9 * Cc + 31) // 32
    out = torch.empty((B * H * W, wpl), dtype=torch.int32, device="cuda")
    f = lambda: _lib.check(lib.bnn_im2col_sign_pack_f32(x.data_ptr(), B, Cc, H, W, C.byref(g), out.data_ptr(), wpl, S))
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byt = x.numel() * 4 + out.numel() * 4
    print(json.dumps({"shape": [B, Cc, H, W], "ms": round(ms, 4), "gbs": round(byt / ms / 1e6, 1)}), flush=True)

# cfg2: conv_forward_binary x[1,64,32,32] 3x3 pad 1, D = 64 (one launch), graph-timed like bench.py
import bench  # noqa: E402

st = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
g2 = _lib.ConvGeom(3, 3, 1, 1, 1, 1, 64, 64)
xc = torch.randn((1, 64, 32, 32), device="cuda")
pw = torch.randint(-2**31, 2**31 - 1, (64, 18), dtype=torch.int32, device="cuda")
bc = torch.randn(64, device="cuda")
yc = torch.empty((1, 64, 32, 32), device="cuda")
fc = lambda: _lib.check(lib.bnn_conv_forward_binary_f32(xc.data_ptr(), 1, 64, 32, 32, pw.data_ptr(), 18, bc.data_ptr(),
                                                         C.byref(g2), yc.data_ptr(), st.cuda_stream))
print(json.dumps({"cfg2_device_ms": bench._graph_time(fc, st, flush), "cfg2_ms": bench._dev_time(fc, st, flush, 30),
                  "kernel": lib.bnn_last_gemm_kernel().decode()}), flush=True)
