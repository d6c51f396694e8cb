"""The round-2 fused kernels on shapes the default network does not exercise, each checked bit for
bit against the oracle, with the kernel each weighted layer ran asserted:

* halo4_kernel (csrc/halo.cu): 64/128/256-channel inputs (1, 2, 4 K steps per tap), pooled and
  unpooled, image widths 2..64 (canvases with several images per row, frame-only tiles, partial
  image groups), 1x1 / 1x3 / 3x1 "same" kernels, batches that leave the last tile partial;
* lin4_kernel (csrc/linear.cu): deep K (split-K completed in the launch), K not a multiple of
  256, feature counts not a multiple of 128, batches over one 256-image tile;
* the swap4 fallback for a conv whose K steps per tap are not a power of two.
"""
import numpy as np
import pytest

from conftest import INPUT_STREAM

pytestmark = pytest.mark.gpu


def conv(d, k=3, s=1, p=1):
    return {"kind": "conv", "out_channels": d, "kernel_size": k, "stride": s, "pad": p}


def lin(f):
    return {"kind": "linear", "out_features": f}


G = [{"kind": "affine_norm"}, {"kind": "htanh"}, {"kind": "sign"}]
POOL = [{"kind": "maxpool"}]

TOPOLOGIES = {
    # 64-channel input (1 K step per tap), unpooled, odd width: several images per canvas row
    "c64_odd": ([1, 3, 12, 10], [conv(64)] + G + [conv(64)] + G + [conv(96)] + G + [lin(10)]),
    # pooled 32 -> 16 -> 8 -> 4 -> 2, widths 32/16/8/4 through the pooled epilogue units
    "pool_chain": ([1, 3, 32, 32], [conv(64)] + G + [conv(128)] + POOL + G + [conv(128)] + POOL + G +
                   [conv(128)] + POOL + G + [conv(128)] + POOL + G + [lin(10)]),
    # 256-channel input (4 K steps per tap), 2x2 images pooled to 1x1
    "c256_tiny": ([1, 3, 4, 4], [conv(256)] + G + [conv(256)] + G + [conv(256)] + POOL + G + [lin(12)]),
    # 1x1 (pad 0) and 1x3 / 3x1 same convs on 128 channels, width 64 (two 32-column chunks)
    "kernels_1x1_1x3": ([1, 3, 6, 64], [conv(128)] + G +
                        [{"kind": "conv", "out_channels": 128, "kernel_size": 1, "pad": 0}] + G +
                        [{"kind": "conv", "out_channels": 128, "kernel_size": [1, 3], "pad": [0, 1]}] + G +
                        [{"kind": "conv", "out_channels": 64, "kernel_size": [3, 1], "pad": [1, 0]}] + G + [lin(10)]),
    # 192-channel input: 3 K steps per tap -> the swap4 fallback
    "c192_fallback": ([1, 3, 8, 8], [conv(192)] + G + [conv(128)] + G + [lin(10)]),
    # linear stack: deep K (split-K in the launch), K % 256 != 0, D % 128 != 0
    "fc_deep": ([1, 8192, 1, 1], [lin(256)] + G + [lin(200 + 24)] + G + [lin(96)] + [lin(10)]),
    "fc_ragged": ([1, 300, 1, 1], [lin(160)] + G + [lin(64)] + [lin(10)]),
}


def _kernels(bnn, net):
    lib = bnn.load()
    out = []
    for i, l in enumerate(net.layers):
        if l["kind"] in ("conv", "linear"):
            out.append(lib.bnn_net_layer_kernel(net.handle, i).decode())
    return out


@pytest.mark.parametrize("name", sorted(TOPOLOGIES))
@pytest.mark.parametrize("batch", [1, 5, 300])
def test_topology_vs_oracle(bnn, orc, name, batch):
    shape, layers = TOPOLOGIES[name]
    if batch == 300 and shape[2] * shape[3] > 64 * 8:
        batch = 40  # keep the oracle run short on the larger images
    net = bnn.Network(layers, tuple(shape[1:]), 31)
    net.set_engine("fused")
    x = orc.fill_random((batch, *shape[1:]), orc.mix64(31, INPUT_STREAM))
    got = net.forward(x)
    want = orc.net(layers, tuple(shape[1:]), 31).forward(x)
    assert np.array_equal(got, want), (name, batch)
    ks = _kernels(bnn, net)
    if name.startswith("fc_"):
        assert ks.count("lin4_kernel") >= 2, ks
    elif name == "c192_fallback":
        assert ks[1] == "fused_swap_mxf4", ks
    else:
        assert "halo4_kernel" in ks, ks


def test_deep_linear_splits_k(bnn):
    """fc 8192 -> 256 at batch 5: few output tiles, deep K -> lin4 with its K split over CTAs."""
    shape, layers = TOPOLOGIES["fc_deep"]
    net = bnn.Network(layers, tuple(shape[1:]), 31)
    x = np.zeros((5, *shape[1:]), dtype=np.float32)
    net.forward(x)
    assert _kernels(bnn, net)[0] == "lin4_kernel"


@pytest.mark.parametrize("mode", [1, 2, 3])  # auto, TMA-loaded images forced, producer-expanded forced
@pytest.mark.parametrize("batch", [1, 37, 600])
def test_lin4_tma_images_vs_oracle(bnn, orc, mode, batch):
    """lin4 with the images expanded once to e2m1 (expand_act4_kernel) and TMA-loaded, against
    the producer-expanded path and the oracle: K % 256 != 0, D % 128 != 0, split-K and not."""
    lib = bnn.load()
    layers = [lin(992)] + G + [lin(544)] + G + [lin(10)]
    net = bnn.Network(layers, (2336, 1, 1), 41)
    net.set_engine("fused")
    x = orc.fill_random((batch, 2336, 1, 1), orc.mix64(41, INPUT_STREAM))
    try:
        bnn._lib.check(lib.bnn_set_fused_lin4(mode))
        got = net.forward(x)
        ks = _kernels(bnn, net)
    finally:
        lib.bnn_set_fused_lin4(1)
    assert ks.count("lin4_kernel") >= 2, ks
    assert np.array_equal(got, orc.net(layers, (2336, 1, 1), 41).forward(x))
