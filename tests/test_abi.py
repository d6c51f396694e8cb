"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every symbol
include/bnn_cuda.h declares, and its host-only helpers behave like the reference. No
compute calls (there is no GPU here): compute entry points must fail loudly, not fall back.
"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, gpu_available

HEADER = os.path.join(ROOT, "include", "bnn_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(bnn_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_abi():
    names = declared_functions()
    for must in ("bnn_sign_pack_cols_f32", "bnn_sign_pack_rows_f32", "bnn_im2col_sign_pack_f32",
                 "bnn_xnor_gemm_s32", "bnn_conv_forward_binary_f32", "bnn_linear_forward_packed_f32",
                 "bnn_net_forward", "bnn_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(bnn):
    lib_path = bnn.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True,
                         check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    # and the Python binding covers them all
    assert set(declared_functions()) <= set(bnn.EXPORTS)


def test_library_is_sm100a_only(bnn):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bnn.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_words_per_line_and_output_dims(bnn):
    lib = bnn.load()
    assert [lib.bnn_words_per_line(e) for e in (1, 31, 32, 33, 576, 9216)] == [1, 1, 1, 2, 18, 288]
    assert bnn.output_dims(bnn.ConvGeometry(3, 3, 1, 1, 1, 1, 1, 1), 32, 32) == (32, 32)
    assert bnn.output_dims(bnn.ConvGeometry(2, 2, 2, 2, 0, 0, 1, 1), 32, 32) == (16, 16)
    with pytest.raises(bnn.ShapeError, match="height"):
        bnn.output_dims(bnn.ConvGeometry(3, 3, 2, 2, 0, 0, 1, 1), 32, 32)
    with pytest.raises(bnn.ShapeError, match="width"):
        bnn.output_dims(bnn.ConvGeometry(2, 3, 2, 2, 0, 0, 1, 1), 32, 32)
    with pytest.raises(bnn.ShapeError, match="kernel larger"):
        bnn.output_dims(bnn.ConvGeometry(5, 5, 1, 1, 0, 0, 1, 1), 3, 3)


def test_mix64_matches_oracle(bnn, orc, golden):
    _, meta = golden
    for k, v in meta["mix64"].items():
        s, c = (int(t) for t in k.split(","))
        assert bnn.mix64(s, c) == v == orc.mix64(s, c)


def test_default_spec_matches_reference_topology(bnn, orc):
    from paper_1911_04477_b200._lib import LayerSpec

    lib = bnn.load()
    arr = (LayerSpec * 64)()
    n = lib.bnn_default_spec(C.addressof(arr), 64)
    oarr, on = orc.default_spec()
    assert n == on == 36
    for i in range(n):
        assert (arr[i].kind, arr[i].out_channels, arr[i].kernel_h, arr[i].pad_h, arr[i].out_features) == \
               (oarr[i].kind, oarr[i].out_channels, oarr[i].kernel_h, oarr[i].pad_h, oarr[i].out_features)
    # the Python spec helper agrees too
    kinds = [l["kind"] for l in bnn.default_layers()]
    assert len(kinds) == 36 and kinds.count("conv") == 6 and kinds.count("linear") == 3


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu(bnn):
    lib = bnn.load()
    rc = lib.bnn_xnor_gemm_s32(None, 1, None, 1, 1, 1, 1, None, 1, None)
    assert rc == 4  # BNN_E_CUDA, never a silent CPU fallback
    with pytest.raises(bnn.CudaError):
        bnn.xnor_gemm(bnn.PackedBitMatrix.make(1, 32, "rows"), bnn.PackedBitMatrix.make(32, 1, "cols"), 32)


def test_host_side_shape_checks_match_reference(bnn):
    w = bnn.PackedBitMatrix.make(2, 40, "rows")
    x = bnn.PackedBitMatrix.make(40, 2, "cols")
    # test_kernels.cpp:161-170
    with pytest.raises(bnn.ShapeError):
        bnn.xnor_gemm(w, x, 39)
    with pytest.raises(bnn.ShapeError):
        bnn.xnor_gemm(x, x, 40)
    with pytest.raises(bnn.ShapeError):
        bnn.xnor_gemm(w, bnn.PackedBitMatrix.make(72, 2, "cols"), 40)
    p = bnn.PackedBitMatrix.make(1, 40, "rows")
    assert p.words_per_line == 2 and p.pad_bits_per_line == 24 and p.pad_mask() == 0xFFFFFF00


def test_oracle_is_not_linked_into_the_product(bnn):
    out = subprocess.run(["nm", "-D", bnn.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out and "bnnref" not in out
    src = open(os.path.join(ROOT, "paper_1911_04477_b200", "api.py")).read()
    assert "oracle" not in src.replace("oracle/", "")
