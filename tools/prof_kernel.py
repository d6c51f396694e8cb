"""Run one K1/K2/K3 launch at the bench shapes (for ncu captures).

    python tools/prof_kernel.py im2col|pack_cols|pack_rows|gemm_popc|gemm_xnor4|gemm_xnor4_conv|conv_b1|probes
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_04477_b200 as bnn  # noqa: E402
from paper_1911_04477_b200 import _lib  # noqa: E402

lib = bnn.load()
S = torch.cuda.current_stream().cuda_stream
what = sys.argv[1]
if what == "im2col":
    g = _lib.ConvGeom(3, 3, 1, 1, 1, 1, 128, 128)
    x = torch.empty((256, 128, 32, 32), dtype=torch.float32, device="cuda")
    _lib.check(lib.bnn_fill_random_f32(7, 0, x.numel(), x.data_ptr(), S))
    out = torch.empty((256 * 1024, 36), dtype=torch.int32, device="cuda")
    for _ in range(2):
        _lib.check(lib.bnn_im2col_sign_pack_f32(x.data_ptr(), 256, 128, 32, 32, C.byref(g), out.data_ptr(), 36, S))
elif what.startswith("gemm"):
    # gemm_xnor4_conv: the conv-shaped product of VGG conv1 at batch 256 (M = 128, N = 262144)
    M, N, L = (128, 262144, 1152) if what.endswith("_conv") else (1024, 1024, 1024)
    w = torch.randint(-2**31, 2**31 - 1, (M, L // 32), dtype=torch.int32, device="cuda")
    x = torch.randint(-2**31, 2**31 - 1, (N, L // 32), dtype=torch.int32, device="cuda")
    out = torch.empty((M, N), dtype=torch.int32, device="cuda")
    lib.bnn_set_gemm_policy(1 if what == "gemm_popc" else 2)
    for _ in range(2):
        _lib.check(lib.bnn_xnor_gemm_s32(w.data_ptr(), L // 32, x.data_ptr(), L // 32, M, N, L, out.data_ptr(), N, S))
elif what == "probes":
    # the K3 pipe candidates: LOP3+POPC loop, emulated b1 mma.sync, tcgen05 i8 / mxf4
    a, b = C.c_double(), C.c_double()
    _lib.check(lib.bnn_probe_popc_peak(C.byref(a), C.byref(b), S))
    _lib.check(lib.bnn_probe_bmma_peak(C.byref(a), C.byref(b), S))
    _lib.check(lib.bnn_probe_umma_peak(0, 256, C.byref(a), C.byref(b), S))
    _lib.check(lib.bnn_probe_umma_peak(1, 256, C.byref(a), C.byref(b), S))
elif what == "conv_b1":
    g = _lib.ConvGeom(3, 3, 1, 1, 1, 1, 64, 64)
    x = torch.empty((1, 64, 32, 32), dtype=torch.float32, device="cuda")
    _lib.check(lib.bnn_fill_random_f32(7, 0, x.numel(), x.data_ptr(), S))
    w = torch.randint(-2**31, 2**31 - 1, (64, 18), dtype=torch.int32, device="cuda")
    b = torch.zeros(64, dtype=torch.float32, device="cuda")
    y = torch.empty((1, 64, 32, 32), dtype=torch.float32, device="cuda")
    for _ in range(2):
        _lib.check(lib.bnn_conv_forward_binary_f32(x.data_ptr(), 1, 64, 32, 32, w.data_ptr(), 18, b.data_ptr(),
                                                   C.byref(g), y.data_ptr(), S))
else:
    L = N = 16384
    x = torch.empty((L, N), dtype=torch.float32, device="cuda")
    _lib.check(lib.bnn_fill_random_f32(7, 0, x.numel(), x.data_ptr(), S))
    out = torch.empty((N, L // 32), dtype=torch.int32, device="cuda")
    fn = lib.bnn_sign_pack_cols_f32 if what == "pack_cols" else lib.bnn_sign_pack_rows_f32
    for _ in range(2):
        _lib.check(fn(x.data_ptr(), L, N, out.data_ptr(), L // 32, S))
torch.cuda.synchronize()
print("ok", what)
