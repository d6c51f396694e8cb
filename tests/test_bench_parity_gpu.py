"""Bit-exact parity of the benchmarked path itself: the default network's
logits at the batch sizes bench.py times, produced exactly as bench.py produces them --
Network.forward_device on a side stream, called three times (first sighting runs eagerly, the
second is captured into a CUDA graph, the third replays it) -- against FNV-1a hashes of the
UNMODIFIED reference's logits (tests/golden/default_net_batches.json, tools/make_golden_batches.py;
bench.cpp:23-33 hashing, bench.cpp:68-78 input stream)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, INPUT_STREAM

pytestmark = pytest.mark.gpu

HASHES = json.load(open(os.path.join(GOLD, "default_net_batches.json")))["fnv1a"]


@pytest.fixture(scope="module")
def net(bnn):
    return bnn.Network(seed=1)


def _timed_path(bnn, net, B):
    import torch

    from paper_1911_04477_b200 import _lib

    lib = bnn.load()
    st = torch.cuda.Stream()
    x = torch.empty((B, 3, 32, 32), dtype=torch.float32, device="cuda")
    _lib.check(lib.bnn_fill_random_f32(bnn.mix64(1, INPUT_STREAM), 0, x.numel(), x.data_ptr(), st.cuda_stream))
    logits = torch.empty((net.logits, B), dtype=torch.float32, device="cuda")
    out = []
    for _ in range(3):  # eager, capture, replay
        logits.fill_(float("nan"))
        with torch.cuda.stream(st):
            net.forward_device(x, logits, st.cuda_stream)
        st.synchronize()
        out.append(logits.cpu().numpy().copy())
    return out


@pytest.mark.parametrize("B", [int(b) for b in HASHES])
def test_default_network_benchmarked_batches_match_reference(bnn, net, B):
    for i, lg in enumerate(_timed_path(bnn, net, B)):
        assert bnn.fnv1a_hash(lg) == HASHES[str(B)], f"batch {B}, call {i} (eager/capture/replay)"


def test_headline_batch_full_logits(bnn, net):
    want = np.load(os.path.join(GOLD, "default_net_b256.npy"))
    for lg in _timed_path(bnn, net, 256):
        assert np.array_equal(lg, want)


def test_headline_batch_live_reference(bnn, net, ref):
    """The same 256 images through the compiled reference on this host, compared in full."""
    x = ref.fill_random((256, 3, 32, 32), ref.mix64(1, INPUT_STREAM))
    want = ref.net_default(1).forward(x, batch_threads=os.cpu_count() or 1)
    assert np.array_equal(_timed_path(bnn, net, 256)[2], want)


@pytest.mark.parametrize("B", [1024, 4096])
def test_shard_offsets_match_reference_columns(bnn, net, B):
    """A rank's shard (bench.py N > 1: fill_random at the shard's global element offset) gives
    the reference's columns of the global batch."""
    import torch

    from paper_1911_04477_b200 import _lib
    from paper_1911_04477_b200.shard import input_offset, shard_range

    world = 4
    lib = bnn.load()
    parts = []
    for r in range(world):
        lo, n = shard_range(B, world, r)
        x = torch.empty((n, 3, 32, 32), dtype=torch.float32, device="cuda")
        _lib.check(lib.bnn_fill_random_f32(bnn.mix64(1, INPUT_STREAM), input_offset(B, world, r), x.numel(),
                                           x.data_ptr(), 0))
        parts.append(net.forward_device(x).cpu().numpy())
    assert bnn.fnv1a_hash(np.ascontiguousarray(np.concatenate(parts, axis=1))) == HASHES[str(B)]
