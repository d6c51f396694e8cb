"""SURVEY.md §8(f) row f3 and the other ExecKernels: the bench / verify harness of the reference
(bench.cpp) over the device engines, checked against the UNMODIFIED reference (oracle/_ref).

* BinaryReference (sign(im2col) + float_gemm on sign(weights), network.cpp:81-94,128-131),
  Naive (network.cpp:96-111) and PerLayer (mixed kernels) network forwards are bit-identical
  to the reference's network_forward with the same ExecKernel.
* run_verify (bench.cpp:193-199) returns the reference's VerifySummary on the same network.
* The corrupted-bit hook (test_bench.cpp:159-173): one flipped packed weight bit of the logits
  layer moves a logit by 2, and verify fails.
* run_benchmark + emit_report write the reference's report schema; the reference's own
  parse_report reads it, and the logits hashes equal the reference's for the same config.
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLD, INPUT_STREAM

pytestmark = pytest.mark.gpu

SPECS = ["tiny_spec", "pad_injected_spec", "strided_spec"]


def _spec_net(bnn, name, binarize=None):
    return bnn.Network.from_spec_file(os.path.join(GOLD, f"{name}.json"), binarize)


def _input(ref, path):
    js = json.load(open(path))
    return ref.fill_random(tuple(js["input_shape"]), ref.mix64(js["seed"], INPUT_STREAM))


@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("engine", ["binary_reference", "naive", "float", "per_layer"])
def test_exec_kernels_match_reference(bnn, ref, name, engine):
    path = os.path.join(GOLD, f"{name}.json")
    net = bnn.Network.from_spec_file(path)
    rnet = ref.net_file(path)
    x = _input(ref, path)
    net.set_engine(engine)
    got = net.forward(x)
    want = rnet.forward(x, exec_kind=engine)
    assert np.array_equal(got, want)


def test_default_network_binary_reference_and_naive(bnn, ref):
    net = bnn.Network(seed=1)
    rnet = ref.net_default(1)
    x = ref.fill_random((2, 3, 32, 32), ref.mix64(1, INPUT_STREAM))
    for engine in ("binary_reference", "naive"):
        net.set_engine(engine)
        assert np.array_equal(net.forward(x), rnet.forward(x, exec_kind=engine, batch_threads=2)), engine
    net.set_engine("auto")
    assert net.engine == "fused"


def test_per_layer_mixed_kernels(bnn, ref, tmp_path):
    """ExecKernel::PerLayer with a float conv, a naive conv and binary linears in one network."""
    spec = {"name": "mixed", "input_shape": [3, 3, 8, 8], "seed": 5, "kernel": "binary",
            "layers": [{"kind": "conv", "out_channels": 8, "kernel_size": 3, "pad": 1, "kernel": "float"},
                       {"kind": "affine_norm"}, {"kind": "htanh"},
                       {"kind": "conv", "out_channels": 16, "kernel_size": 3, "pad": 1, "kernel": "naive"},
                       {"kind": "maxpool"}, {"kind": "sign"},
                       {"kind": "linear", "out_features": 33}, {"kind": "sign"},
                       {"kind": "linear", "out_features": 5}]}
    path = tmp_path / "mixed.json"
    path.write_text(json.dumps(spec))
    net = bnn.Network.from_spec_file(path)
    x = _input(ref, path)
    net.set_engine("per_layer")
    assert net.engine == "per_layer"
    assert np.array_equal(net.forward(x), ref.net_file(str(path)).forward(x, exec_kind="per_layer"))


@pytest.mark.parametrize("spec", [None, "tiny_spec", "pad_injected_spec"])
def test_run_verify_matches_reference(bnn, ref, spec):
    import ctypes as C

    path = None if spec is None else os.path.join(GOLD, f"{spec}.json")
    batch = 2 if spec is None else 4
    want = ref.run_verify(path, batch, 1)
    dev, n, ok, pad = C.c_double(), C.c_size_t(), C.c_int(), C.c_int()
    from paper_1911_04477_b200._lib import check

    check(bnn.load().bnn_run_verify(None if path is None else path.encode(), batch, 1, None, C.byref(dev),
                                    C.byref(n), C.byref(ok), C.byref(pad)))
    assert (dev.value, n.value, bool(ok.value), bool(pad.value)) == (
        want["max_abs_deviation"], want["compared"], want["pass"], want["pad_correction_exercised"])
    assert want["pass"] and want["compared"] % batch == 0


def test_corrupted_bit_is_detected(bnn, ref):
    """test_bench.cpp:159-173 through the Python mirror (Network.verify / set_layer_data)."""
    net = _spec_net(bnn, "tiny_spec", binarize=True)
    eng0 = net.engine  # "generic": the 33-feature hidden layer is not fusable (32-feature words)
    x = ref.fill_random((4, 3, 8, 8), 9)
    s = net.verify(x)
    assert s["pass"] and s["max_abs_deviation"] == 0.0 and s["compared"] == 20
    last = len(net.layers) - 1
    packed, _, _, _, _ = net.layer_data(last)
    bad = packed.copy()
    bad[0, 0] ^= 1
    net.set_layer_data(last, packed=bad)
    s = net.verify(x)
    assert not s["pass"] and s["max_abs_deviation"] >= 1.9
    net.set_layer_data(last, packed=packed)
    assert net.verify(x)["pass"]
    assert net.engine == eng0


def test_layer_data_is_the_reference_built_layer(bnn, ref):
    net = bnn.Network(seed=1, binarize_weights=True)
    rnet = ref.net_default(1, binarize=True)
    for i in (0, 1, 27):
        packed, weights, bias, scale, shift = net.layer_data(i)
        rp, rb, rs, rsh = rnet.layer_params(i)
        assert np.array_equal(packed.reshape(rp.shape), rp) and np.array_equal(bias, rb)
        assert np.array_equal(scale, rs) and np.array_equal(shift, rsh)
        if weights.size:
            assert set(np.unique(weights)) <= {-1.0, 1.0}  # binarize_weights applied to the float weights


def _keys(o):
    if isinstance(o, dict):
        return {k: _keys(v) for k, v in o.items()}
    if isinstance(o, list) and o and isinstance(o[0], dict):
        return [_keys(o[0])]
    return type(o).__name__ if not isinstance(o, (int, float)) else "num"


@pytest.mark.parametrize("spec", [None, "tiny_spec"])
def test_report_schema_and_hashes_match_reference(bnn, ref, tmp_path, spec):
    from paper_1911_04477_b200._lib import check

    path = None if spec is None else os.path.join(GOLD, f"{spec}.json")
    batch = 2 if spec is None else 4
    ours, theirs = tmp_path / "ours.json", tmp_path / "ref.json"
    # iterations 2, warmup 0 (the reference run below: 1 and 0; iterations is not compared)
    check(bnn.load().bnn_run_benchmark(None if path is None else path.encode(), batch, 2, 0, 1, 3, 1,
                                       str(ours).encode()))
    ref.run_benchmark(theirs, path, batch=batch, iterations=1, warmup=0, seed=1, kernels_mask=3)
    n, h = ref.parse_report(ours)  # the reference's parser accepts our report
    a, b = json.load(open(ours)), json.load(open(theirs))
    assert _keys(a) == _keys(b)
    assert n == 2 and int(a["kernels"][0]["logits_hash"], 16) == h
    assert [k["kernel"] for k in a["kernels"]] == ["binary", "float"]
    for ka, kb in zip(a["kernels"], b["kernels"]):
        assert ka["logits_hash"] == kb["logits_hash"], ka["kernel"]
    assert a["weight_memory"] == b["weight_memory"]
    assert a["network"] == b["network"]
    assert {k: v for k, v in a["config"].items() if k != "iterations"} == \
        {k: v for k, v in b["config"].items() if k != "iterations"}
    assert [s["baseline"] for s in a["speedups"]] == ["float"]
