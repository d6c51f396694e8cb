"""On-disk formats (csrc/io.cpp) against the compiled reference:
packed blobs (binarize.cpp:116-148), tensor blobs (tensor.cpp:123-150) and NetworkSpec JSON
files with weights blobs (network.cpp:203-306, 487-567). The blob tests are host-only (no GPU);
the network test runs the loaded network on the device and compares logits bit for bit."""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, INPUT_STREAM


def _rand_words(rng, lines, extent):
    wpl = (extent + 31) // 32
    w = rng.integers(0, 2**32, size=(lines, wpl), dtype=np.uint64).astype(np.uint32)
    pad = wpl * 32 - extent
    if pad:
        w[:, -1] &= np.uint32((1 << (32 - pad)) - 1)  # pad bits 0 (tensor.hpp:67-70)
    return w


@pytest.mark.parametrize("rows,cols,orient", [(1, 1, "rows"), (3, 40, "rows"), (33, 5, "cols"),
                                               (64, 96, "rows"), (7, 100, "cols")])
def test_packed_blob_roundtrip_with_reference(bnn, ref, tmp_path, rows, cols, orient):
    rng = np.random.default_rng(rows * 1000 + cols)
    lines, extent = (rows, cols) if orient == "rows" else (cols, rows)
    p = bnn.PackedBitMatrix(rows, cols, orient, _rand_words(rng, lines, extent))
    ours = tmp_path / "ours.pbm"
    bnn.save_packed_blob(p, ours)
    o, r, c, w = ref.load_packed_blob(ours)  # the reference reads our file
    assert (o, r, c) == ((0 if orient == "rows" else 1), rows, cols)
    assert np.array_equal(w, p.words)
    theirs = tmp_path / "theirs.pbm"
    ref.save_packed_blob(theirs, 0 if orient == "rows" else 1, rows, cols, p.words)
    assert ours.read_bytes() == theirs.read_bytes()  # byte-identical files
    q = bnn.load_packed_blob(theirs)
    assert (q.logical_rows, q.logical_cols, q.orientation) == (rows, cols, orient)
    assert np.array_equal(q.words, p.words)


def test_packed_blob_errors_match_reference(bnn, ref, tmp_path):
    rng = np.random.default_rng(5)
    p = bnn.PackedBitMatrix(4, 40, "rows", _rand_words(rng, 4, 40))
    good = tmp_path / "good.pbm"
    bnn.save_packed_blob(p, good)
    data = good.read_bytes()
    cases = {
        "truncated": (data[:10], "packed blob truncated"),
        "orient": (b"\x07" + data[1:], "packed blob has bad orientation byte"),
        "size": (data + b"\x00\x00\x00\x00", "packed blob size mismatch"),
        "pad": (data[:-4] + b"\xff\xff\xff\xff", "packed blob has nonzero pad bits"),
    }
    for name, (raw, msg) in cases.items():
        f = tmp_path / f"{name}.pbm"
        f.write_bytes(raw)
        with pytest.raises(bnn.IoError, match=msg):
            bnn.load_packed_blob(f)
        with pytest.raises(Exception, match=msg):  # the reference raises the same IoError
            ref.load_packed_blob(f)
    with pytest.raises(bnn.IoError, match="cannot open for reading"):
        bnn.load_packed_blob(tmp_path / "missing.pbm")


@pytest.mark.parametrize("shape", [(1, 1, 1, 1), (2, 3, 4, 5), (8, 9216, 1, 1)])
def test_tensor_blob_roundtrip_with_reference(bnn, ref, orc, tmp_path, shape):
    x = orc.fill_random(shape, 77)
    x.flat[::7] = -0.0
    ours = tmp_path / "ours.tb"
    bnn.save_tensor_blob(x, ours)
    assert np.array_equal(ref.load_tensor_blob(ours), x)
    theirs = tmp_path / "theirs.tb"
    ref.save_tensor_blob(theirs, x)
    assert ours.read_bytes() == theirs.read_bytes()
    y = bnn.load_tensor_blob(theirs)
    assert y.shape == shape and np.array_equal(y.view(np.uint32), x.view(np.uint32))  # -0.0 kept


def test_tensor_blob_errors(bnn, tmp_path):
    f = tmp_path / "t.tb"
    bnn.save_tensor_blob(np.zeros((1, 2, 3, 4), np.float32), f)
    data = f.read_bytes()
    (tmp_path / "short.tb").write_bytes(data[:20])
    with pytest.raises(bnn.IoError, match="tensor blob truncated"):
        bnn.load_tensor_blob(tmp_path / "short.tb")
    (tmp_path / "long.tb").write_bytes(data + b"\x00")
    with pytest.raises(bnn.IoError, match="tensor blob size mismatch"):
        bnn.load_tensor_blob(tmp_path / "long.tb")


def test_spec_info_reads_reference_fixture(bnn):
    import ctypes as C

    lib = bnn.load()
    shape = np.zeros(4, np.uint64)
    n = C.c_size_t()
    path = os.path.join(GOLD, "tiny_spec.json")
    assert lib.bnn_spec_info(path.encode(), shape.ctypes.data, C.byref(n)) == 0
    spec = json.load(open(path))
    assert list(shape) == spec["input_shape"] and n.value == len(spec["layers"])
    bad = b"/nonexistent/spec.json"
    assert lib.bnn_spec_info(bad, shape.ctypes.data, C.byref(n)) == 3  # ConfigError
    assert b"cannot open network spec" in lib.bnn_last_error()


def _blob_spec(tmp_path, ref, orc):
    """A NetworkSpec whose conv and first linear layer load their float weights from tensor
    blobs written by the reference (network.cpp:233-241, 258-266)."""
    wc = orc.fill_random((16, 3, 3, 3), 101)
    wl = orc.fill_random((12, 16 * 4 * 4, 1, 1), 102)
    ref.save_tensor_blob(tmp_path / "conv.tb", wc)
    ref.save_tensor_blob(tmp_path / "fc.tb", wl)
    spec = {"name": "blobs", "input_shape": [2, 3, 8, 8], "seed": 9, "binarize_weights": False,
            "kernel": "binary",
            "layers": [{"kind": "conv", "out_channels": 16, "kernel_size": 3, "pad": 1,
                        "weights_blob": str(tmp_path / "conv.tb")},
                       {"kind": "maxpool"}, {"kind": "affine_norm"}, {"kind": "htanh"}, {"kind": "sign"},
                       {"kind": "linear", "out_features": 12, "weights_blob": str(tmp_path / "fc.tb")},
                       {"kind": "sign"}, {"kind": "linear", "out_features": 5}]}
    path = tmp_path / "spec.json"
    path.write_text(json.dumps(spec))
    return path


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["blobs", "tiny_spec.json", "pad_injected_spec.json", "strided_spec.json"])
def test_network_from_spec_file_vs_reference(bnn, ref, orc, tmp_path, name):
    path = _blob_spec(tmp_path, ref, orc) if name == "blobs" else os.path.join(GOLD, name)
    net = bnn.Network.from_spec_file(path)
    want_net = ref.net_file(str(path))
    b = 5
    x = orc.fill_random((b, *net.input_chw), orc.mix64(3, INPUT_STREAM))
    got = net.forward(x)
    want = want_net.forward(x)
    assert np.array_equal(got, want), name


def test_spec_blob_shape_mismatch_is_shape_error(bnn, ref, orc, tmp_path):
    path = _blob_spec(tmp_path, ref, orc)
    ref.save_tensor_blob(tmp_path / "conv.tb", orc.fill_random((16, 3, 5, 5), 1))  # wrong kernel
    try:
        import torch

        if not torch.cuda.is_available():
            pytest.skip("network construction needs the device")
    except ImportError:
        pytest.skip("torch unavailable")
    with pytest.raises(bnn.ShapeError, match=r"layer 0 \(conv\): weights blob shape does not match"):
        bnn.Network.from_spec_file(path)
