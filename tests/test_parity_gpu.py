"""CUDA (sm_100a) hot path vs the CPU oracle and the reference golden fixtures.

Bar: bit-exact for packed words and int32 GEMM outputs; float outputs after bias are also
expected bit-exact (integer + bias is one rounding on both sides), checked with array_equal.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from conftest import GOLD, INPUT_STREAM

pytestmark = pytest.mark.gpu


def torch_cuda():
    import torch

    return torch


def rng_pm1(rng, shape):
    return np.where(rng.integers(0, 2, size=shape) == 1, 1.0, -1.0).astype(np.float32)


# --------------------------------------------------------------------------- K1 encoder


def test_encoder_golden(bnn, golden):
    arrays, meta = golden
    for i, _ in enumerate(meta["cases"]["encode"]):
        x = arrays[f"enc{i}_x"]
        assert np.array_equal(bnn.sign_pack_rows(x).words, arrays[f"enc{i}_rows"]), i
        assert np.array_equal(bnn.sign_pack_cols(x).words, arrays[f"enc{i}_cols"]), i


def test_encoder_kats(bnn):
    assert bnn.pack_rows(np.ones((1, 32), np.float32)).words[0, 0] == 0xFFFFFFFF
    assert bnn.pack_rows(-np.ones((1, 32), np.float32)).words[0, 0] == 0
    alt = np.where(np.arange(32) % 2 == 0, 1.0, -1.0).astype(np.float32)[None]
    assert bnn.pack_rows(alt).words[0, 0] == 0x55555555
    col = np.ones((33, 1), np.float32)
    col[32] = -1
    assert bnn.pack_cols(col).words.tolist() == [[0xFFFFFFFF, 0]]
    m = rng_pm1(np.random.default_rng(11), (5, 37))
    assert np.array_equal(bnn.pack_cols(m.T.copy()).words, bnn.pack_rows(m).words)


def test_encoder_strict_reports_first_bad_entry(bnn):
    m = np.ones((2, 3), np.float32)
    m[1, 2] = 0.5
    for fn in (bnn.pack_rows, bnn.pack_cols):
        with pytest.raises(bnn.EncodingError, match=r"\(1,2\)"):
            fn(m)
    # the first in row-major order wins, as in the reference's loops (binarize.cpp:44,59)
    big = np.ones((300, 200), np.float32)
    big[250, 3] = 2.0
    big[17, 150] = 0.0
    big[17, 199] = np.nan
    with pytest.raises(bnn.EncodingError, match=r"\(17,150\)"):
        bnn.pack_cols(big)
    with pytest.raises(bnn.EncodingError, match=r"\(17,150\)"):
        bnn.pack_rows(big)


@pytest.mark.parametrize("shape", [(1, 1), (31, 33), (1024, 1024), (9216, 1024), (4097, 65), (3, 100000)])
def test_encoder_random_vs_oracle(bnn, orc, shape):
    x = orc.fill_random(shape, 31 + shape[0])
    x.flat[::97] = 0.0
    x.flat[1::101] = -0.0
    assert np.array_equal(bnn.sign_pack_cols(x).words, orc.pack(x, "cols", True))
    assert np.array_equal(bnn.sign_pack_rows(x).words, orc.pack(x, "rows", True))


def test_roundtrip_and_pad_hygiene(bnn):
    rng = np.random.default_rng(303)
    for _ in range(60):
        r, c = int(rng.integers(1, 9)), int(rng.integers(1, 71))
        x = rng_pm1(rng, (r, c))
        for p in (bnn.pack_rows(x), bnn.pack_cols(x)):
            assert np.array_equal(bnn.unpack(p), x)
            assert (p.words[:, -1] & np.uint32(p.pad_mask()) == 0).all()


def test_device_encoder_with_padded_leading_dimension(bnn, orc):
    torch = torch_cuda()
    lib = bnn.load()
    L, N, ld = 100, 77, 8  # wpl = 4, padded to 8 words per line
    x = orc.fill_random((L, N), 5)
    dx = torch.from_numpy(x).cuda()
    dw = torch.full((N, ld), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.bnn_sign_pack_cols_f32(dx.data_ptr(), L, N, dw.data_ptr(), ld, s) == 0
    got = dw.cpu().numpy().view(np.uint32)
    assert np.array_equal(got[:, :4], orc.pack(x, "cols", True))
    assert (got[:, 4:] == 0xFFFFFFFF).all()  # words past the line are untouched


# ----------------------------------------------------------------------- K2 im2col


GEOMS = [((2, 3, 6, 6), (3, 3, 1, 1, 1, 1, 3, 5)), ((1, 64, 32, 32), (3, 3, 1, 1, 1, 1, 64, 64)),
         ((3, 5, 9, 7), (3, 2, 2, 1, 1, 0, 5, 7)), ((2, 4, 8, 8), (5, 5, 1, 1, 2, 2, 4, 3)),
         ((1, 1, 4, 4), (1, 1, 1, 1, 0, 0, 1, 1)), ((4, 7, 5, 11), (2, 3, 1, 2, 0, 1, 7, 2)),
         ((2, 128, 16, 16), (3, 3, 1, 1, 1, 1, 128, 8)),
         # batch x output rows >= SM count: the row-bits kernel (W <= 32), incl. kW = 1 runs,
         # stride 2, 5x5 / pad 2, a partial last word and rectangular kernels
         ((6, 64, 32, 32), (3, 3, 1, 1, 1, 1, 64, 64)), ((40, 3, 8, 8), (5, 5, 1, 1, 2, 2, 3, 4)),
         ((80, 5, 9, 7), (3, 2, 2, 1, 1, 0, 5, 7)), ((160, 33, 4, 4), (1, 1, 1, 1, 0, 0, 33, 2)),
         ((150, 7, 5, 11), (2, 3, 1, 2, 0, 1, 7, 2)), ((3, 16, 64, 20), (3, 3, 1, 1, 1, 1, 16, 8)),
         # many row groups per SM (a pipelined bulk-copy variant was measured slower and removed):
         # 32 / 16 / 20 / 4 wide, stride 2, 5x5 pad 2 with a ragged last row group, a partial word
         ((160, 8, 32, 32), (3, 3, 1, 1, 1, 1, 8, 8)), ((600, 8, 16, 16), (4, 4, 2, 2, 1, 1, 8, 4)),
         ((300, 4, 20, 20), (5, 5, 1, 1, 2, 2, 4, 3)), ((650, 36, 4, 4), (1, 1, 1, 1, 0, 0, 36, 2))]


@pytest.mark.parametrize("shape,g", GEOMS)
def test_im2col_sign_pack_vs_oracle(bnn, orc, shape, g):
    x = orc.fill_random(shape, 9)
    x.flat[::13] = 0.0
    got = bnn.im2col_sign_pack(x, g)
    want = np.concatenate([orc.pack(orc.im2col(x, b, g), "cols", True) for b in range(shape[0])])
    assert np.array_equal(got.words, want)


# --------------------------------------------------------------------------- K3 GEMM


def test_gemm_golden(bnn, golden):
    arrays, meta = golden
    for i, (m, n, L) in enumerate(meta["cases"]["gemm"]):
        w = bnn.PackedBitMatrix(m, L, "rows", arrays[f"gemm{i}_w"])
        x = bnn.PackedBitMatrix(L, n, "cols", arrays[f"gemm{i}_x"])
        assert np.array_equal(bnn.xnor_gemm(w, x, L), arrays[f"gemm{i}_out"]), (m, n, L)


def test_gemm_acceptance_sweep(bnn):
    # acceptance.cpp:61-79: 200 cases, L in {1,31,32,33,40,64,96,100}, zero tolerance
    rng = np.random.default_rng(101)
    for case in range(200):
        L = int(rng.choice([1, 31, 32, 33, 40, 64, 96, 100]))
        d, n = int(rng.integers(1, 17)), int(rng.integers(1, 17))
        w, x = rng_pm1(rng, (d, L)), rng_pm1(rng, (L, n))
        got = bnn.xnor_gemm(bnn.pack_rows(w), bnn.pack_cols(x), L)
        assert np.array_equal(got, (w.astype(np.int64) @ x.astype(np.int64))), (case, L)


@pytest.mark.parametrize("m,n,L", [(1024, 1024, 1024), (64, 1024, 576), (4096, 1024, 9216),
                                   (1000, 1024, 4096), (129, 257, 1000), (7, 3000, 33),
                                   (300, 5, 70000), (1, 1, 1)])
def test_gemm_vs_oracle(bnn, orc, m, n, L):
    w = orc.pack(orc.fill_random((m, L), m + 1), "rows", True)
    x = orc.pack(orc.fill_random((L, n), n + 2), "cols", True)
    got = bnn.xnor_gemm(bnn.PackedBitMatrix(m, L, "rows", w), bnn.PackedBitMatrix(L, n, "cols", x), L)
    assert np.array_equal(got, orc.xnor_gemm(w, x, L))


@pytest.mark.parametrize("L", [1, 32, 33, 576, 9216])
def test_gemm_all_agree_all_disagree(bnn, L):
    ones = bnn.pack_rows(np.ones((3, L), np.float32))
    plus = bnn.pack_cols(np.ones((L, 5), np.float32))
    minus = bnn.pack_cols(-np.ones((L, 5), np.float32))
    assert (bnn.xnor_gemm(ones, plus, L) == L).all()
    assert (bnn.xnor_gemm(ones, minus, L) == -L).all()


@pytest.mark.parametrize("kernel", ["auto", "popc", "umma", "tma"])
@pytest.mark.parametrize("M", [70, 300])
def test_gemm_device_api_strides_and_bias(bnn, orc, policy, kernel, M):
    """Padded leading dimensions (garbage past each line), an output stride and the bias epilogue
    on every K3 kernel (tma with M = 300: a CTA pair whose second half is out of range)."""
    torch = torch_cuda()
    lib = bnn.load()
    policy(kernel)
    N, L = 90, 200
    wpl, ldw, ldx, ldo = 7, 9, 12, 100
    w = orc.pack(orc.fill_random((M, L), 1), "rows", True)
    x = orc.pack(orc.fill_random((L, N), 2), "cols", True)
    dw = torch.zeros((M, ldw), dtype=torch.int32, device="cuda")
    dx = torch.zeros((N, ldx), dtype=torch.int32, device="cuda")
    dw[:, :wpl] = torch.from_numpy(w.view(np.int32)).cuda()
    dx[:, :wpl] = torch.from_numpy(x.view(np.int32)).cuda()
    dw[:, wpl:] = -1  # garbage past the line must be ignored
    dx[:, wpl:] = 12345
    out = torch.full((M, ldo), 7, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.bnn_xnor_gemm_s32(dw.data_ptr(), ldw, dx.data_ptr(), ldx, M, N, L, out.data_ptr(), ldo, s) == 0
    want = orc.xnor_gemm(w, x, L)
    o = out.cpu().numpy()
    assert np.array_equal(o[:, :N], want) and (o[:, N:] == 7).all()
    bias = orc.fill_random((M,), 3)
    of = torch.empty((M * N,), dtype=torch.float32, device="cuda")
    assert lib.bnn_xnor_gemm_bias_f32(dw.data_ptr(), ldw, dx.data_ptr(), ldx, M, N, L,
                                      torch.from_numpy(bias).cuda().data_ptr(), N, of.data_ptr(), s) == 0
    assert np.array_equal(of.cpu().numpy().reshape(M, N), want.astype(np.float32) + bias[:, None])


def test_gemm_rejects_like_reference(bnn):
    lib = bnn.load()
    # 32*wpl > 2^26 (kernels.cpp:66-68)
    ld = (1 << 21) + 1
    assert lib.bnn_xnor_gemm_s32(None, ld, None, ld, 1, 1, (1 << 26) + 1, None, 1, None) == 1
    assert "accumulator guard" in bnn._lib.last_error()


# ------------------------------------------------------------------- layer forwards


def test_conv_forward_golden(bnn, orc, golden):
    arrays, meta = golden
    for i, c in enumerate(meta["cases"]["conv"]):
        xs, ws, bs = c["seeds"]
        g = c["geom"]
        x = orc.fill_random(tuple(c["shape"]), xs)
        pw = bnn.sign_pack_rows(orc.fill_random((g[7], g[0] * g[1] * g[6]), ws))
        y = bnn.conv_forward_binary(x, pw, orc.fill_random((g[7],), bs), g)
        assert orc.fnv1a(y) == c["fnv1a"], c
        if f"conv{i}_out" in arrays:
            assert np.array_equal(y, arrays[f"conv{i}_out"])


@pytest.mark.parametrize("shape,g", GEOMS)
def test_conv_forward_vs_oracle(bnn, orc, shape, g):
    x = orc.fill_random(shape, 19)
    K = g[0] * g[1] * g[6]
    w = orc.fill_random((g[7], K), 20)
    b = orc.fill_random((g[7],), 21)
    y = bnn.conv_forward_binary(x, bnn.sign_pack_rows(w), b, g)
    assert np.array_equal(y, orc.conv_forward_binary(x, orc.pack(w, "rows", True), b, list(g)))


def test_conv_kats(bnn, orc):
    g = (3, 3, 1, 1, 1, 1, 3, 2)
    y = bnn.conv_forward_binary(np.ones((1, 3, 6, 6), np.float32), bnn.pack_rows(np.ones((2, 27), np.float32)),
                                np.zeros(2, np.float32), g)
    assert (y == 27).all()
    x = orc.fill_random((1, 1, 4, 4), 4)
    y = bnn.conv_forward_binary(x, bnn.pack_rows(np.ones((1, 1), np.float32)), np.zeros(1, np.float32),
                                (1, 1, 1, 1, 0, 0, 1, 1))
    assert np.array_equal(y, orc.sign(x))


def test_linear_forward_golden_and_cfg1(bnn, orc, golden):
    _, meta = golden
    for c in meta["cases"]["linear"]:
        xs, ws, bs = c["seeds"]
        x = orc.fill_random((c["K"], c["N"]), xs)
        pw = bnn.sign_pack_rows(orc.fill_random((c["M"], c["K"]), ws))
        y = bnn.linear_forward_packed(x, pw, orc.fill_random((c["M"],), bs))
        assert orc.fnv1a(y) == c["fnv1a"], c


def test_linear_binary_equals_float_on_pm1(bnn):
    # test_network.cpp:90-100
    rng = np.random.default_rng(5)
    for features in (8, 33):
        x = rng_pm1(rng, (features, 6))
        w = rng_pm1(rng, (4, features))
        bias = np.array([0.5, -0.5, 1.0, 0.0], np.float32)
        want = (w @ x).astype(np.float32) + bias[:, None]
        assert np.array_equal(bnn.linear_forward(x, w, bias), want)


# ------------------------------------------------------------------------ glue ops


def test_glue_ops_vs_oracle(bnn, orc):
    x = orc.fill_random((3, 5, 6, 8), 77)
    x.flat[::11] = 0.0
    x.flat[3] = -0.0
    s, t = orc.fill_random((5,), 78), orc.fill_random((5,), 79)
    assert np.array_equal(bnn.affine_norm(x, s, t), orc.affine_tensor(x, s, t))
    m = orc.fill_random((7, 9), 80)
    s7, t7 = orc.fill_random((7,), 81), orc.fill_random((7,), 82)
    assert np.array_equal(bnn.affine_norm(m, s7, t7), orc.affine_matrix(m, s7, t7))
    assert np.array_equal(bnn.maxpool2(x), orc.maxpool2(x))
    assert np.array_equal(bnn.sign(x), orc.sign(x))
    y = x * 3
    assert np.array_equal(bnn.htanh(y), orc.htanh(y))
    assert np.array_equal(bnn.flatten_to_columns(x), x.reshape(3, -1).T)


def test_fill_random_matches_reference(bnn, golden):
    arrays, _ = golden
    assert np.array_equal(bnn.fill_random((257,), 42), arrays["fill_random_s42"])
    a = bnn.fill_random((1000,), 9)
    b = bnn.fill_random((400,), 9, offset=600)
    assert np.array_equal(a[600:], b)  # shard-local generation == slice of the global tensor


# ------------------------------------------------------------------------- networks


def _spec_net(bnn, orc, name):
    js = json.load(open(os.path.join(GOLD, name + ".json")))
    net = bnn.Network.from_spec(js)
    x = orc.fill_random(tuple(js["input_shape"]), orc.mix64(js["seed"], INPUT_STREAM))
    return net, x


def test_network_golden(bnn, orc, golden):
    arrays, meta = golden
    for c in meta["cases"]["network"]:
        if c["name"] == "default":
            net = bnn.Network(seed=c["seed"])
            x = orc.fill_random((c["batch"], 3, 32, 32), orc.mix64(c["seed"], INPUT_STREAM))
            key = f"net_default_b{c['batch']}"
        else:
            net, x = _spec_net(bnn, orc, c["name"])
            key = f"net_{c['name']}"
        lg = net.forward(x)
        assert np.array_equal(lg, arrays[key]), c["name"]
        assert bnn.fnv1a_hash(lg) == c["fnv1a"]


def test_network_parameters_match_reference_build(bnn, orc):
    net = bnn.Network(seed=3)
    onet = orc.net(seed=3)
    for i, l in enumerate(net.layers):
        pk, b, sc, sh = net.layer_params(i)
        words = np.zeros_like(pk)
        bo, sco, sho = np.zeros_like(b), np.zeros_like(sc), np.zeros_like(sh)
        orc.lib.orc_net_layer_params(onet.h, i, words.ctypes.data if pk.size else None,
                                     bo.ctypes.data if b.size else None,
                                     sco.ctypes.data if sc.size else None,
                                     sho.ctypes.data if sh.size else None)
        assert np.array_equal(words, pk) and np.array_equal(bo, b), (i, l)
        assert np.array_equal(sco, sc) and np.array_equal(sho, sh), (i, l)


@pytest.mark.parametrize("batch", [1, 3, 64])
def test_default_network_vs_oracle(bnn, orc, batch):
    net = bnn.Network(seed=1)
    x = orc.fill_random((batch, 3, 32, 32), orc.mix64(5, INPUT_STREAM))
    assert np.array_equal(net.forward(x), orc.net(seed=1).forward(x))


def test_network_device_path_and_deterministic(bnn, orc):
    torch = torch_cuda()
    net = bnn.Network(seed=2)
    x = orc.fill_random((16, 3, 32, 32), 99)
    dx = torch.from_numpy(x).cuda()
    a = net.forward_device(dx).cpu().numpy()
    b = net.forward_device(dx).cpu().numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(a, net.forward(x))
    assert net.last_launches() > 0


# ------------------------------------------------------- both K3 kernels, forced


@pytest.fixture
def policy(bnn):
    lib = bnn.load()
    yield lambda p: lib.bnn_set_gemm_policy({"auto": 0, "popc": 1, "umma": 2, "tma": 3}[p])
    lib.bnn_set_gemm_policy(0)


GEMM_KERNEL = {"popc": "popc", "umma": "xnor4_kernel", "tma": "xnor4t_kernel"}


@pytest.mark.parametrize("kernel", ["popc", "umma", "tma"])
@pytest.mark.parametrize("m,n,L", [(1, 1, 1), (3, 4, 31), (16, 16, 33), (128, 256, 128), (130, 70, 9216),
                                   (257, 513, 1000), (1024, 1024, 1024), (64, 1024, 576),
                                   (1000, 300, 4096), (5, 3000, 200), (300, 481, 257), (129, 241, 2050)])
def test_gemm_kernels_vs_oracle(bnn, orc, policy, kernel, m, n, L):
    policy(kernel)
    w = orc.pack(orc.fill_random((m, L), m + 7), "rows", True)
    x = orc.pack(orc.fill_random((L, n), n + 9), "cols", True)
    got = bnn.xnor_gemm(bnn.PackedBitMatrix(m, L, "rows", w), bnn.PackedBitMatrix(L, n, "cols", x), L)
    assert bnn.load().bnn_last_gemm_kernel().decode() == GEMM_KERNEL[kernel]
    assert np.array_equal(got, orc.xnor_gemm(w, x, L))


@pytest.mark.parametrize("kernel", ["popc", "umma", "tma"])
def test_gemm_kernels_golden_and_layers(bnn, orc, golden, policy, kernel):
    policy(kernel)
    arrays, meta = golden
    for i, (m, n, L) in enumerate(meta["cases"]["gemm"]):
        w = bnn.PackedBitMatrix(m, L, "rows", arrays[f"gemm{i}_w"])
        x = bnn.PackedBitMatrix(L, n, "cols", arrays[f"gemm{i}_x"])
        assert np.array_equal(bnn.xnor_gemm(w, x, L), arrays[f"gemm{i}_out"]), (m, n, L)
    for i, c in enumerate(meta["cases"]["conv"]):
        xs, ws, bs = c["seeds"]
        g = c["geom"]
        x = orc.fill_random(tuple(c["shape"]), xs)
        pw = bnn.sign_pack_rows(orc.fill_random((g[7], g[0] * g[1] * g[6]), ws))
        y = bnn.conv_forward_binary(x, pw, orc.fill_random((g[7],), bs), g)
        assert orc.fnv1a(y) == c["fnv1a"], (kernel, c)
    for c in meta["cases"]["linear"]:
        xs, ws, bs = c["seeds"]
        x = orc.fill_random((c["K"], c["N"]), xs)
        pw = bnn.sign_pack_rows(orc.fill_random((c["M"], c["K"]), ws))
        y = bnn.linear_forward_packed(x, pw, orc.fill_random((c["M"],), bs))
        assert orc.fnv1a(y) == c["fnv1a"], (kernel, c)


@pytest.mark.parametrize("kernel", ["popc", "umma"])
def test_network_both_kernels(bnn, orc, policy, kernel):
    policy(kernel)
    net = bnn.Network(seed=1)
    x = orc.fill_random((8, 3, 32, 32), orc.mix64(1, INPUT_STREAM))
    assert np.array_equal(net.forward(x), orc.net(seed=1).forward(x))


@pytest.mark.parametrize("m,n,L", [(2048, 2100, 1030), (4096, 1024, 9216)])
def test_gemm_auto_large_takes_tma_kernel(bnn, orc, policy, m, n, L):
    """Above 2^32 bit-MACs AUTO runs the TMA-fed FP4 kernel (operands expanded once in HBM)."""
    policy("auto")
    w = orc.pack(orc.fill_random((m, L), m + 3), "rows", True)
    x = orc.pack(orc.fill_random((L, n), n + 5), "cols", True)
    got = bnn.xnor_gemm(bnn.PackedBitMatrix(m, L, "rows", w), bnn.PackedBitMatrix(L, n, "cols", x), L)
    assert bnn.load().bnn_last_gemm_kernel().decode() == "xnor4t_kernel"
    assert np.array_equal(got, orc.xnor_gemm(w, x, L))


def test_conv_large_takes_tma_kernel(bnn, orc, policy):
    """conv_forward_binary whose GEMM is above 2^32 bit-MACs: the TMA kernel's f32 epilogue
    (to_float + bias_add + reshape_output scatter) against the oracle (forced: with 136 output
    channels AUTO keeps the in-CTA expansion kernel)."""
    policy("tma")
    g = bnn.ConvGeometry(3, 3, 1, 1, 1, 1, 128, 136)
    x = orc.fill_random((33, 128, 32, 32), 5)
    w = orc.fill_random((136, 1152), 6)
    b = orc.fill_random((136,), 7)
    y = bnn.conv_forward_binary(x, bnn.sign_pack_rows(w), b, g)
    assert bnn.load().bnn_last_gemm_kernel().decode() == "xnor4t_kernel"
    want = orc.conv_forward_binary(x, orc.pack(w, "rows", True), b, list(g.__dict__.values()))
    assert np.array_equal(y, want)
