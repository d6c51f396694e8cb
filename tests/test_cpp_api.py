"""The C++ drop-in API (include/bnn_b200.hpp): the library exports the reference-signature
symbols (CPU), and the compiled C++ test program passes on the GPU (the reference's unit
cases re-expressed through namespace bnn, checked against the C oracle)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1911_04477_b200", "libbnn_b200.so")
BIN = os.path.join(ROOT, "paper_1911_04477_b200", "bin", "test_cpp_api")

CPP_SYMBOLS = ["bnn::pack_rows(", "bnn::pack_cols(", "bnn::xnor_gemm(", "bnn::conv_forward_binary(",
               "bnn::linear_forward_packed(", "bnn::linear_forward(", "bnn::sign(", "bnn::htanh(",
               "bnn::unpack(", "bnn::to_float(", "bnn::bias_add(", "bnn::maxpool2(", "bnn::affine_norm(",
               "bnn::flatten_to_columns(", "bnn::output_dims(", "bnn::fill_random(", "bnn::mix64(",
               "bnn::PackedBitMatrix::make(", "bnn::build_default_network(", "bnn::DeviceNetwork::forward(",
               "bnn::im2col_sign_pack(", "bnn::reshape_output(", "bnn::flatten_weights(",
               # the network / harness / lowering entry points of network.hpp, bench.hpp, lowering.hpp
               "bnn::build_network(", "bnn::network_forward(bnn::Network const&", "bnn::load_network_spec(",
               "bnn::save_network_spec(", "bnn::im2col(", "bnn::col2im(", "bnn::float_gemm(", "bnn::naive_conv(",
               "bnn::conv_forward_float(", "bnn::conv_forward_binary_reference(", "bnn::conv_forward_naive(",
               "bnn::linear_forward_binary_reference(", "bnn::run_benchmark(", "bnn::run_verify(",
               "bnn::verify_network(", "bnn::emit_report(", "bnn::parse_report(", "bnn::print_report(",
               "bnn::median(", "bnn::fnv1a_hash(bnn::FloatMatrix const&", "bnn::parse_kernel_choice(",
               "bnn::parse_layer_kind(", "bnn::to_string(bnn::LayerKind"]


def test_library_exports_reference_cpp_api():
    if not os.path.exists(LIB):
        pytest.skip("libbnn_b200.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", LIB], capture_output=True, text=True).stdout
    missing = [s for s in CPP_SYMBOLS if s not in out]
    assert not missing, missing


@pytest.mark.gpu
def test_cpp_api_program():
    assert os.path.exists(BIN), "build with __graft_entry__.build()"
    r = subprocess.run([BIN, ROOT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
