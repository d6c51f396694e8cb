"""The float control group on the GPU (csrc/control.cu) against the
compiled reference's ExecKernel::Float network_forward (conv_forward_float, linear_forward
Float, network.cpp:50-63, 113-120, 350-420). The reference's float_gemm is FMA-contracted
(-O3 -march=native); the GPU keeps the same k-ascending FMA chain, so logits are compared
bit for bit when the reference build has FMA (x86-64-v3/v4), else within 1e-4 (bench.hpp:11)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, INPUT_STREAM

pytestmark = pytest.mark.gpu


def _cmp(got, want, ref):
    if ref.isa in ("v3", "v4"):
        assert np.array_equal(got, want)
    else:
        assert np.max(np.abs(got - want)) <= 1e-4


@pytest.mark.parametrize("batch", [1, 3])
def test_default_network_float_engine_vs_reference(bnn, ref, orc, batch):
    net = bnn.Network(seed=1)
    net.set_engine("float")
    assert net.engine == "float"
    x = orc.fill_random((batch, 3, 32, 32), orc.mix64(1, INPUT_STREAM))
    _cmp(net.forward(x), ref.net_default(1).forward(x, exec_kind="float"), ref)


@pytest.mark.parametrize("name", ["tiny_spec.json", "strided_spec.json"])
def test_spec_float_engine_vs_reference(bnn, ref, orc, name):
    path = os.path.join(GOLD, name)
    net = bnn.Network.from_spec_file(path)
    net.set_engine("float")
    x = orc.fill_random((4, *net.input_chw), 17)
    _cmp(net.forward(x), ref.net_file(path).forward(x, exec_kind="float"), ref)


def test_float_gemm_direct(bnn, orc):
    """bnn_float_gemm_f32 = a k-ascending fmaf chain per output, + bias."""
    torch = pytest.importorskip("torch")
    lib = bnn.load()
    M, K, N = 37, 300, 45
    w = orc.fill_random((M, K), 1)
    x = orc.fill_random((K, N), 2)
    b = orc.fill_random((M,), 3)
    dw, dx, db = (torch.from_numpy(a).cuda() for a in (w, x, b))
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.bnn_float_gemm_f32(dw.data_ptr(), M, K, dx.data_ptr(), N, db.data_ptr(), 0, out.data_ptr(), s) == 0
    got = out.cpu().numpy()
    acc = np.zeros((M, N), np.float32)
    for k in range(K):  # fp32 FMA chain emulated in float64 (exact product; rare double rounding)
        acc = (acc.astype(np.float64) + w[:, k:k + 1].astype(np.float64) * x[k:k + 1, :]).astype(np.float32)
    want = (acc + b[:, None]).astype(np.float32)
    assert np.max(np.abs(got - want)) <= 1e-5 * max(1.0, float(np.max(np.abs(want))))
