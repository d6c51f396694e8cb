"""Fused engine (csrc/fused.cu) parity: one tcgen05 launch per weighted layer with the glue
folded into the epilogue and packed-bit activations must reproduce the reference's
network_forward(Binary) logits bit for bit (network.cpp:330-420)."""
import numpy as np
import pytest

from conftest import INPUT_STREAM

pytestmark = pytest.mark.gpu


def _net(bnn, spec):
    return bnn.Network(spec["layers"], tuple(spec["input_shape"][1:]), spec["seed"])


def _oracle(orc, spec):
    return orc.net(spec["layers"], tuple(spec["input_shape"][1:]), spec["seed"])


def conv(d, k=3, s=1, p=1):
    return {"kind": "conv", "out_channels": d, "kernel_size": k, "stride": s, "pad": p}


def lin(f):
    return {"kind": "linear", "out_features": f}


G = [{"kind": "affine_norm"}, {"kind": "htanh"}, {"kind": "sign"}]
POOL = [{"kind": "maxpool"}]

FUSABLE = {
    # Cw = 1 and 2 (per-word producer path), stride 2, rectangular kernels, no-affine glue
    "narrow": {"input_shape": [1, 3, 16, 16], "seed": 7,
               "layers": [conv(32, 4, 2, 1)] + G + [conv(64, 3, 1, 1)] + POOL + G +
                         [conv(96, 2, 1, 0), {"kind": "sign"}, lin(64)] + G[:2] + [lin(9)]},
    # 5x5 / pad 2 first layer, odd spatial sizes, linear straight after a conv (NHWC flatten)
    "odd": {"input_shape": [1, 5, 9, 11], "seed": 11,
            "layers": [conv(128, 5, 1, 2)] + G + [conv(128, 3, 2, 0)] + [{"kind": "affine_norm"}] +
                      [lin(32), lin(10)]},
    # C = 256 / 512 fast path with pooling down to 1x1, then a single logits layer
    "wide": {"input_shape": [1, 3, 8, 8], "seed": 3,
             "layers": [conv(256)] + POOL + G + [conv(512)] + POOL + G + [conv(256)] + POOL + G + [lin(33)]},
    # 4-channel pixel input (the vectorised pixel packer's generic-C path), 8 x 8
    "pix4": {"input_shape": [1, 4, 8, 8], "seed": 17, "layers": [conv(32)] + G + [lin(10)]},
    # FP4 CTA pairs with partial channel pairs (384 = 1.5 pairs, 320: the odd CTA's channels
    # all past D), pooled and unpooled, position counts not a multiple of the 192-position tile
    "pairs": {"input_shape": [1, 3, 12, 12], "seed": 21,
              "layers": [conv(64)] + G + [conv(384)] + POOL + G + [conv(320)] + G + [lin(10)]},
    # CUDA-core pixel conv (K <= 32): pooled first layer with 3 output words, stride 2 with 2
    # words and a 2x2 kernel over 8 channels (K = 32: the full patch word), odd sizes
    "pix_pool": {"input_shape": [1, 3, 10, 14], "seed": 23,
                 "layers": [conv(96)] + POOL + G + [conv(64, 3, 2, 1)] + G + [lin(10)]},
    "pix_s2": {"input_shape": [1, 3, 9, 7], "seed": 25, "layers": [conv(64, 3, 2, 1)] + G + [lin(10)]},
    "pix_k32": {"input_shape": [1, 8, 7, 9], "seed": 27, "layers": [conv(256, 2, 1, 0)] + G + [lin(10)]},
    # linear-first stacks (BASELINE cfg1 / cfg4 shape class): K1 pack_rows of the float input,
    # linear -> linear with no glue (sign of float(a) + bias), a 4096-wide hidden layer
    "fc_stack": {"input_shape": [1, 288, 1, 1], "seed": 5, "layers": [lin(4096), lin(96), lin(10)]},
    # tensor input flattened (F = 100: a partial last word), glue between the linears
    "fc_tensor_in": {"input_shape": [1, 4, 5, 5], "seed": 9, "layers": [lin(64)] + G + [lin(10)]},
    # hidden linear layers on the CUDA-core popcount path (K % 128 == 0), affine glue between
    "fc_popc": {"input_shape": [1, 256, 1, 1], "seed": 13,
                "layers": [lin(1024)] + G + [lin(512)] + G + [lin(96), lin(7)]},
}


@pytest.fixture(params=["auto", "nohalo", "halostream", "halo0", "nolin4", "lin4tma", "lin4prod", "nopixpopc", "pixf32", "pixpacked", "noswap", "swapall",
                        "nofp4", "fp4all", "nopair", "pair224", "nosmall", "cg1", "nosplit", "split16"])
def tiling(bnn, request):
    """Every fused test runs with the automatic tile choice (one launch per weighted layer,
    swapped-operand conv kernels, A operand in TMEM and split-K for the small-batch linear
    layers), with the position-major conv kernel (noswap), with the halo-tile conv off or also
    streaming its weights, with the int8 linear kernel instead of lin4, with cta_group 1 forced,
    and with split-K off / forced to 16. The CUDA-core first conv
    (pix_popc) runs under "auto" (float input up to batch 512, else after the packer), "pixf32"
    (reading the float input itself, no packer launch) and "pixpacked"; the other settings put the
    pixel-input layer on the tensor-core kernels they select."""
    lib = bnn.load()
    p = request.param
    bnn._lib.check(lib.bnn_set_fused_tiling({"cg1": 1}.get(p, 0), 0))
    bnn._lib.check(lib.bnn_set_fused_split({"nosplit": 1, "split16": 16}.get(p, 0)))
    bnn._lib.check(lib.bnn_set_fused_swap({"noswap": 0, "swapall": 2}.get(p, 1)))
    bnn._lib.check(lib.bnn_set_fused_small_logits(0 if p == "nosmall" else 1))
    bnn._lib.check(lib.bnn_set_fused_pix_popc({"auto": 3, "pixf32": 1, "pixpacked": 2}.get(p, 0)))
    bnn._lib.check(lib.bnn_set_fused_fp4({"fp4": 1, "fp4all": 2, "nofp4": 0}.get(p, 1)))
    bnn._lib.check(lib.bnn_set_fused_fp4_pair({"nopair": 0, "pair224": 3}.get(p, 1)))
    bnn._lib.check(lib.bnn_set_fused_halo({"nohalo": 0, "halostream": 2}.get(p, 1)))
    # the pixel-input first conv on the halo FP4 kernel (opt-in: measured slower than pix_tile)
    bnn._lib.check(lib.bnn_set_fused_halo0(1 if p == "halo0" else 0))
    # lin4 images: TMA-loaded from a once-expanded e2m1 copy (forced on / off; auto by size)
    bnn._lib.check(lib.bnn_set_fused_lin4({"nolin4": 0, "lin4tma": 2, "lin4prod": 3}.get(p, 1)))
    yield p
    lib.bnn_set_fused_tiling(0, 0)
    lib.bnn_set_fused_split(0)
    lib.bnn_set_fused_swap(1)
    lib.bnn_set_fused_small_logits(1)
    lib.bnn_set_fused_pix_popc(3)
    lib.bnn_set_fused_fp4(1)
    lib.bnn_set_fused_fp4_pair(1)
    lib.bnn_set_fused_halo(1)
    lib.bnn_set_fused_halo0(0)
    lib.bnn_set_fused_lin4(1)


@pytest.fixture
def fused(bnn, tiling):
    def mk(spec=None, seed=1):
        net = bnn.Network(seed=seed) if spec is None else _net(bnn, spec)
        net.set_engine("fused")
        assert net.engine == "fused"
        return net
    return mk


@pytest.mark.parametrize("batch", [1, 2, 3, 5, 33, 128, 129])
def test_default_network_fused_vs_oracle(bnn, orc, fused, tiling, batch):
    net = fused()
    x = orc.fill_random((batch, 3, 32, 32), orc.mix64(1, INPUT_STREAM))
    got = net.forward(x)
    # 9 weighted layers, + pack_pixels when the first conv reads packed pixel words (the int8
    # tensor-core path and pix_popc after the packer); halo0 and pix_tile read the floats
    assert net.last_launches() == ((9 if tiling in ("auto", "pixf32", "halo0") else 10) +
                                   (1 if tiling == "lin4tma" else 0))  # + expand_act4 for fc1 (fc1 writes fc2's)
    assert np.array_equal(got, orc.net(seed=1).forward(x))


@pytest.mark.parametrize("bn", [32, 64, 128, 256])
def test_forced_tile_shapes_vs_oracle(bnn, orc, bn):
    lib = bnn.load()
    net = bnn.Network(seed=1)
    net.set_engine("fused")
    x = orc.fill_random((9, 3, 32, 32), orc.mix64(2, INPUT_STREAM))
    try:
        bnn._lib.check(lib.bnn_set_fused_tiling(1, bn))
        got = net.forward(x)
    finally:
        lib.bnn_set_fused_tiling(0, 0)
    assert np.array_equal(got, orc.net(seed=1).forward(x)), bn


def test_default_network_fused_equals_generic_large_batch(bnn, orc, fused):
    torch = pytest.importorskip("torch")
    net = fused(seed=4)
    x = torch.from_numpy(orc.fill_random((1000, 3, 32, 32), 12345)).cuda()
    a = net.forward_device(x).cpu().numpy()
    net.set_engine("generic")
    b = net.forward_device(x).cpu().numpy()
    assert np.array_equal(a, b)
    # and a slice checked against the oracle directly
    xs = x[:7].cpu().numpy()
    assert np.array_equal(a[:, :7], orc.net(seed=4).forward(xs))


def test_default_network_engine_is_fused_by_default(bnn):
    assert bnn.Network(seed=1).engine == "fused"


@pytest.mark.parametrize("name", sorted(FUSABLE))
@pytest.mark.parametrize("batch", [1, 6])
def test_fusable_topologies_vs_oracle(bnn, orc, fused, name, batch):
    spec = dict(FUSABLE[name])
    net = fused(spec)
    shape = (batch, *spec["input_shape"][1:])
    x = orc.fill_random(shape, orc.mix64(spec["seed"], INPUT_STREAM))
    got = net.forward(x)
    want = _oracle(orc, spec).forward(x)
    assert np.array_equal(got, want), name


def test_unfusable_topology_uses_generic_engine(bnn, orc):
    spec = {"input_shape": [1, 4, 12, 12], "seed": 99,
            "layers": [conv(40), {"kind": "htanh"}, {"kind": "affine_norm"}, lin(9)]}
    net = _net(bnn, spec)
    assert net.engine == "generic"
    with pytest.raises(bnn.ConfigError):
        net.set_engine("fused")
    x = orc.fill_random((3, 4, 12, 12), 5)
    assert np.array_equal(net.forward(x), _oracle(orc, spec).forward(x))


def test_graph_replay_matches_eager(bnn, orc):
    """Repeated forwards on a side stream are captured into a CUDA graph and replayed; the
    replayed logits must equal the eager ones and the oracle's, also after the input changes."""
    torch = pytest.importorskip("torch")
    net = bnn.Network(seed=6)
    st = torch.cuda.Stream()
    x = torch.from_numpy(orc.fill_random((37, 3, 32, 32), 77)).cuda()
    out = torch.empty((10, 37), device="cuda")
    want = orc.net(seed=6).forward(x.cpu().numpy())
    with torch.cuda.stream(st):
        for _ in range(4):  # eager, capture, replay, replay
            out.zero_()
            net.forward_device(x, out, st.cuda_stream)
            st.synchronize()
            assert np.array_equal(out.cpu().numpy(), want)
        x2 = torch.from_numpy(orc.fill_random((37, 3, 32, 32), 78)).cuda()
        x.copy_(x2)  # same buffer, new contents: the replayed graph reads them
        net.forward_device(x, out, st.cuda_stream)
        st.synchronize()
    assert np.array_equal(out.cpu().numpy(), orc.net(seed=6).forward(x2.cpu().numpy()))


def test_pipeline_host_buffers_vs_oracle(bnn, orc):
    """bnn_pipe_*: batches submitted from pinned host buffers come back with the oracle's
    logits, in order, with more batches in flight than buffer sets would allow unsynchronised."""
    torch = pytest.importorskip("torch")
    net = bnn.Network(seed=2)
    B, depth = 7, 3
    xs = [orc.fill_random((B, 3, 32, 32), orc.mix64(s, INPUT_STREAM)) for s in range(5)]
    want = [orc.net(seed=2).forward(x) for x in xs]
    hx = [torch.from_numpy(x).pin_memory() for x in xs]
    hy = [torch.empty((net.logits, B), dtype=torch.float32).pin_memory() for _ in range(depth)]
    pipe = net.pipeline(B, depth)
    seqs = []
    for i in range(12):
        if i >= depth:
            pipe.wait(seqs[i - depth])
            k = i - depth
            assert np.array_equal(hy[k % depth].numpy(), want[k % 5]), k
        seqs.append(pipe.submit(hx[i % 5].data_ptr(), hy[i % depth].data_ptr()))
    with pytest.raises(bnn.ConfigError):
        pipe.wait(seqs[0])  # no longer among the last `depth`
    for k in range(12 - depth, 12):
        pipe.wait(seqs[k])
        assert np.array_equal(hy[k % depth].numpy(), want[k % 5]), k
    pipe.close()
