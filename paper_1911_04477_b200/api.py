"""Python mirror of the reference operator API (namespace bnn, /root/reference/proj/include/bnn).

Same names, argument meaning and error behaviour as the reference C++ functions, so the
parity tests read like the reference's own tests. Host (numpy) arguments in, host results
out; every computation runs on the B200 through the C ABI (include/bnn_cuda.h). PyTorch is
used only as the device-memory / stream plumbing for the entry points that have no
``bnn_host_*`` twin.

Reference → here:
    sign / htanh (binarize.hpp:9-16)             sign / htanh
    pack_rows / pack_cols (binarize.hpp:19-23)   pack_rows / pack_cols (strict: EncodingError)
    unpack (binarize.hpp:27)                     unpack
    im2col / col2im (lowering.hpp:11-18)         im2col / col2im (float), im2col_sign_pack (K2)
    xnor_gemm (kernels.hpp:53-54)                xnor_gemm
    conv_forward_binary (network.hpp:117-119)    conv_forward_binary
    linear_forward_packed (network.hpp:133-134)  linear_forward_packed
    linear_forward (network.hpp:130-132)         linear_forward (kernel "binary" / "float")
    float_gemm, conv_forward_float (kernels.hpp:44, network.hpp:114-116)
    conv_forward_binary_reference, linear_forward_binary_reference, conv_forward_naive
    maxpool2 / affine_norm / flatten_to_columns  maxpool2 / affine_norm / flatten_to_columns
    fill_random* / mix64 / unit_random           fill_random / mix64 / unit_random
    build_network + network_forward (ExecKernel) Network (engine "auto"/"float"/"binary_reference"/...)
    verify_network (bench.cpp:172-191)           Network.verify
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ConfigError, ConvGeom, EncodingError, LayerSpec, ShapeError, check, load

ROW_PACKED, COL_PACKED = "rows", "cols"


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ------------------------------------------------------------------------- L0 types


@dataclass
class ConvGeometry:
    """ConvGeometry (tensor.hpp:101-111)."""

    kernel_h: int = 1
    kernel_w: int = 1
    stride_h: int = 1
    stride_w: int = 1
    pad_h: int = 0
    pad_w: int = 0
    in_channels: int = 1
    out_channels: int = 1

    def patch_len(self) -> int:
        return self.kernel_h * self.kernel_w * self.in_channels

    def c(self) -> ConvGeom:
        return ConvGeom(self.kernel_h, self.kernel_w, self.stride_h, self.stride_w, self.pad_h,
                        self.pad_w, self.in_channels, self.out_channels)

    @classmethod
    def of(cls, g) -> "ConvGeometry":
        if isinstance(g, ConvGeometry):
            return g
        return cls(*[int(v) for v in g])


def words_per_line(extent: int) -> int:
    return (int(extent) + 31) // 32


@dataclass
class PackedBitMatrix:
    """PackedBitMatrix (tensor.hpp:63-98): ``words`` is [lines, words_per_line] uint32."""

    logical_rows: int
    logical_cols: int
    orientation: str
    words: np.ndarray

    @classmethod
    def make(cls, rows: int, cols: int, orientation: str) -> "PackedBitMatrix":
        if rows < 1 or cols < 1:
            raise ShapeError("extent 'rows'/'cols' must be >= 1")
        lines, extent = (rows, cols) if orientation == ROW_PACKED else (cols, rows)
        return cls(rows, cols, orientation, np.zeros((lines, words_per_line(extent)), np.uint32))

    def lines(self) -> int:
        return self.logical_rows if self.orientation == ROW_PACKED else self.logical_cols

    def packed_extent(self) -> int:
        return self.logical_cols if self.orientation == ROW_PACKED else self.logical_rows

    @property
    def words_per_line(self) -> int:
        return words_per_line(self.packed_extent())

    @property
    def pad_bits_per_line(self) -> int:
        return self.words_per_line * 32 - self.packed_extent()

    def pad_mask(self) -> int:
        pad = self.pad_bits_per_line
        return 0 if pad == 0 else (0xFFFFFFFF << (32 - pad)) & 0xFFFFFFFF

    def byte_size(self) -> int:
        return self.words.size * 4


# tensor.cpp:46-63
def output_dims(geom, in_h: int, in_w: int) -> tuple[int, int]:
    g = ConvGeometry.of(geom).c()
    oh, ow = C.c_size_t(), C.c_size_t()
    check(load().bnn_output_dims(C.byref(g), in_h, in_w, C.byref(oh), C.byref(ow)))
    return oh.value, ow.value


# tensor.cpp:65-77 (host arithmetic, identical to the device generator)
def mix64(seed: int, counter: int) -> int:
    return int(load().bnn_mix64(seed, counter))


def fill_random(shape, seed: int, offset: int = 0) -> np.ndarray:
    """fill_random / fill_random_matrix / fill_random_vector, generated on the device."""
    import torch

    n = int(np.prod(shape))
    if n == 0:
        raise ShapeError("extent must be >= 1")
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    check(load().bnn_fill_random_f32(seed, offset, n, out.data_ptr(), _stream()))
    return out.cpu().numpy().reshape(shape)


def _stream() -> int:
    import torch

    return torch.cuda.current_stream().cuda_stream


def _dev(a: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# -------------------------------------------------------------------- binarize


def _unary(fn, x):
    x = _f32(x)
    dx = _dev(x)
    out = dx.clone()
    check(fn(dx.data_ptr(), x.size, out.data_ptr(), _stream()))
    return out.cpu().numpy().reshape(x.shape)


def sign(x) -> np.ndarray:
    """binarize.cpp:19-27: v >= 0 -> +1 else -1."""
    return _unary(load().bnn_sign_f32, x)


def htanh(x) -> np.ndarray:
    """binarize.cpp:29-37: clamp to [-1, 1]."""
    return _unary(load().bnn_htanh_f32, x)


def _pack(x, orientation: str, apply_sign: bool) -> PackedBitMatrix:
    x = _f32(x)
    if x.ndim != 2:
        raise ShapeError("pack: expected a matrix")
    rows, cols = x.shape
    p = PackedBitMatrix.make(rows, cols, orientation)
    check(load().bnn_host_sign_pack(_p(x), rows, cols, 0 if orientation == ROW_PACKED else 1,
                                    int(apply_sign), _p(p.words)))
    return p


def pack_rows(w) -> PackedBitMatrix:
    """binarize.cpp:39-53. Entries must be exactly +-1 (EncodingError names the entry)."""
    return _pack(w, ROW_PACKED, False)


def pack_cols(x) -> PackedBitMatrix:
    """binarize.cpp:55-73."""
    return _pack(x, COL_PACKED, False)


def sign_pack_rows(w) -> PackedBitMatrix:
    """pack_rows(sign(w)) fused (network.cpp:247)."""
    return _pack(w, ROW_PACKED, True)


def sign_pack_cols(x) -> PackedBitMatrix:
    """pack_cols(sign(x)) fused (network.cpp:123)."""
    return _pack(x, COL_PACKED, True)


def unpack(p: PackedBitMatrix) -> np.ndarray:
    """binarize.cpp:75-90."""
    import torch

    out = torch.empty((p.logical_rows, p.logical_cols), dtype=torch.float32, device="cuda")
    dw = _dev(p.words)
    check(load().bnn_unpack_f32(dw.data_ptr(), p.words_per_line, p.logical_rows, p.logical_cols,
                                0 if p.orientation == ROW_PACKED else 1, out.data_ptr(), _stream()))
    return out.cpu().numpy()


# -------------------------------------------------------------------- lowering


def im2col_sign_pack(x, geom) -> PackedBitMatrix:
    """pack_cols(sign(im2col(x, b, geom))) for every b (lowering.cpp:7-43, network.cpp:72).

    Returns a col-packed matrix of logical shape [K, B*oh*ow]: line b*oh*ow + j holds
    image b's patch column j.
    """
    import torch

    x = _f32(x)
    if x.ndim != 4:
        raise ShapeError("im2col: expected a [B, C, H, W] tensor")
    g = ConvGeometry.of(geom)
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    K = g.patch_len()
    lines = x.shape[0] * oh * ow
    wpl = words_per_line(K)
    out = torch.zeros((lines, wpl), dtype=torch.int32, device="cuda")
    gc = g.c()
    dx = _dev(x)
    check(load().bnn_im2col_sign_pack_f32(dx.data_ptr(), *x.shape, C.byref(gc), out.data_ptr(),
                                          wpl, _stream()))
    return PackedBitMatrix(K, lines, COL_PACKED, out.cpu().numpy().view(np.uint32))


# --------------------------------------------------------------------- kernels


def xnor_gemm(w: PackedBitMatrix, x: PackedBitMatrix, inner_len: int, threads: int = 1) -> np.ndarray:
    """kernels.cpp:53-88; returns IntMatrix data as int32 [D, N]. ``threads`` is accepted for
    signature parity and ignored (the CUDA grid replaces parallel_rows, kernels.cpp:12-29)."""
    if w.orientation != ROW_PACKED:
        raise ShapeError("xnor_gemm: weight operand must be row-packed")
    if x.orientation != COL_PACKED:
        raise ShapeError("xnor_gemm: input operand must be column-packed")
    if w.logical_cols != inner_len or x.logical_rows != inner_len:
        raise ShapeError(f"xnor_gemm: inner extents {w.logical_cols}/{x.logical_rows} do not "
                         f"match L={inner_len}")
    if w.words_per_line != x.words_per_line:
        raise ShapeError("xnor_gemm: words-per-line mismatch")
    M, N = w.logical_rows, x.logical_cols
    out = np.empty((M, N), np.int32)
    ww = np.ascontiguousarray(w.words, np.uint32)
    xw = np.ascontiguousarray(x.words, np.uint32)
    check(load().bnn_host_xnor_gemm(_p(ww), M, _p(xw), N, inner_len, _p(out)))
    return out


def to_float(m: np.ndarray) -> np.ndarray:
    """kernels.cpp:90-95, on the device."""
    import torch

    m = np.ascontiguousarray(m, np.int32)
    dm = _dev(m)
    out = torch.empty(m.shape, dtype=torch.float32, device="cuda")
    check(load().bnn_to_float_s32(dm.data_ptr(), m.size, out.data_ptr(), _stream()))
    return out.cpu().numpy()


def bias_add(a: np.ndarray, bias) -> np.ndarray:
    """kernels.cpp:97-107, on the device: a[d, j] += bias[d]."""
    a = _f32(a)
    bias = _f32(bias)
    if bias.size != a.shape[0]:
        raise ShapeError(f"bias_add: bias length {bias.size} does not match {a.shape[0]} rows")
    da, db = _dev(a), _dev(bias)
    check(load().bnn_bias_add_f32(da.data_ptr(), a.shape[0], a.size // max(1, a.shape[0]), db.data_ptr(),
                                  _stream()))
    return da.cpu().numpy()


def float_gemm(w, x, threads: int = 1) -> np.ndarray:
    """kernels.cpp:33-51 (the control group's float GEMM), on the CUDA cores: the reference's
    k-ascending FMA chain per output, bit-identical."""
    import torch

    w, x = _f32(w), _f32(x)
    if w.shape[1] != x.shape[0]:
        raise ShapeError(f"float_gemm: inner extents differ, {w.shape[1]} vs {x.shape[0]}")
    dw, dx = _dev(w), _dev(x)
    out = torch.empty((w.shape[0], x.shape[1]), dtype=torch.float32, device="cuda")
    check(load().bnn_float_gemm_f32(dw.data_ptr(), w.shape[0], w.shape[1], dx.data_ptr(), x.shape[1], None, 0,
                                    out.data_ptr(), _stream()))
    return out.cpu().numpy()


def im2col(x, batch_index: int, geom) -> np.ndarray:
    """lowering.cpp:7-43: the float [K, oh*ow] patch matrix of batch slice ``batch_index``."""
    import torch

    x = _f32(x)
    g = ConvGeometry.of(geom)
    if x.shape[1] != g.in_channels:
        raise ShapeError(f"im2col: input has {x.shape[1]} channels, geometry expects {g.in_channels}")
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    out = torch.empty((g.patch_len(), oh * ow), dtype=torch.float32, device="cuda")
    gc = g.c()
    dx = _dev(x)
    check(load().bnn_im2col_f32(dx.data_ptr(), *x.shape, batch_index, 1, C.byref(gc), out.data_ptr(), _stream()))
    return out.cpu().numpy()


def col2im(m, geom, out_h: int, out_w: int) -> np.ndarray:
    """lowering.cpp:45-84, the adjoint of im2col: [K, out_h*out_w] -> [1, C, in_h, in_w]."""
    import torch

    m = _f32(m)
    g = ConvGeometry.of(geom)
    gc = g.c()
    ih, iw = C.c_size_t(), C.c_size_t()
    lib = load()
    check(lib.bnn_col2im_f32(None, m.shape[0], m.shape[1], C.byref(gc), out_h, out_w, None, C.byref(ih), C.byref(iw),
                             None))
    out = torch.empty((1, g.in_channels, ih.value, iw.value), dtype=torch.float32, device="cuda")
    dm = _dev(m)
    check(lib.bnn_col2im_f32(dm.data_ptr(), m.shape[0], m.shape[1], C.byref(gc), out_h, out_w, out.data_ptr(), None,
                             None, _stream()))
    return out.cpu().numpy()


# --------------------------------------------------------------------- layers


def conv_forward_binary(x, packed_w: PackedBitMatrix, bias, geom, threads: int = 1) -> np.ndarray:
    """network.cpp:65-79: [B, C, H, W] -> [B, D, oh, ow]."""
    x = _f32(x)
    g = ConvGeometry.of(geom)
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    bias = _f32(bias)
    if packed_w.orientation != ROW_PACKED or packed_w.logical_cols != g.patch_len() or \
            packed_w.logical_rows != g.out_channels:
        raise ShapeError("conv_forward_binary: packed weights do not match the geometry")
    if bias.size != g.out_channels:
        raise ShapeError(f"bias_add: bias length {bias.size} does not match {g.out_channels} rows")
    out = np.empty((x.shape[0], g.out_channels, oh, ow), np.float32)
    gc = g.c()
    pw = np.ascontiguousarray(packed_w.words, np.uint32)
    check(load().bnn_host_conv_forward_binary(_p(x), *x.shape, _p(pw), _p(bias), C.byref(gc), _p(out)))
    return out


def linear_forward_packed(x, packed_w: PackedBitMatrix, bias, threads: int = 1) -> np.ndarray:
    """network.cpp:121-126: x [K, N] (features x batch) -> [M, N]."""
    x = _f32(x)
    bias = _f32(bias)
    K, N = x.shape
    if packed_w.logical_cols != K:
        raise ShapeError(f"xnor_gemm: inner extents {packed_w.logical_cols}/{K} do not match "
                         f"L={packed_w.logical_cols}")
    if bias.size != packed_w.logical_rows:
        raise ShapeError(f"bias_add: bias length {bias.size} does not match "
                         f"{packed_w.logical_rows} rows")
    out = np.empty((packed_w.logical_rows, N), np.float32)
    pw = np.ascontiguousarray(packed_w.words, np.uint32)
    check(load().bnn_host_linear_forward_packed(_p(x), K, N, _p(pw), packed_w.logical_rows, _p(bias),
                                                _p(out)))
    return out


def linear_forward(x, w, bias, kernel: str = "binary", threads: int = 1) -> np.ndarray:
    """network.cpp:113-119: binary packs the weights per call; float (and naive) run float_gemm."""
    if kernel == "binary":
        return linear_forward_packed(x, sign_pack_rows(w), bias, threads)
    if kernel not in ("float", "naive"):
        raise ConfigError(f"unknown kernel choice '{kernel}', expected binary|float|naive")
    return bias_add(float_gemm(w, x), bias)


def linear_forward_binary_reference(x, w_pm1, bias, threads: int = 1) -> np.ndarray:
    """network.cpp:128-131: float_gemm(w_pm1, sign(x)) + bias, on the device."""
    return bias_add(float_gemm(w_pm1, sign(x)), bias)


def conv_forward_float(x, w_flat, bias, geom, threads: int = 1) -> np.ndarray:
    """network.cpp:50-63: float im2col + float_gemm + bias on the device (bit-identical)."""
    import torch

    x, w_flat, bias = _f32(x), _f32(w_flat), _f32(bias)
    g = ConvGeometry.of(geom)
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    if w_flat.shape[1] != g.patch_len():
        raise ShapeError(f"float_gemm: inner extents differ, {w_flat.shape[1]} vs {g.patch_len()}")
    if bias.size != w_flat.shape[0]:
        raise ShapeError(f"bias_add: bias length {bias.size} does not match {w_flat.shape[0]} rows")
    out = torch.empty((x.shape[0], g.out_channels, oh, ow), dtype=torch.float32, device="cuda")
    dx, dw, db = _dev(x), _dev(w_flat), _dev(bias)
    gc = g.c()
    check(load().bnn_conv_forward_float_f32(dx.data_ptr(), *x.shape, dw.data_ptr(), db.data_ptr(), C.byref(gc),
                                            out.data_ptr(), _stream()))
    return out.cpu().numpy()


def conv_forward_binary_reference(x, w_pm1, bias, geom, threads: int = 1) -> np.ndarray:
    """network.cpp:81-94: sign(im2col(x)) then float_gemm(w_pm1) + bias, on the device."""
    import torch

    x, w_pm1, bias = _f32(x), _f32(w_pm1), _f32(bias)
    g = ConvGeometry.of(geom)
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    B, K, N = x.shape[0], g.patch_len(), x.shape[0] * oh * ow
    lib = load()
    dx, dw, db = _dev(x), _dev(w_pm1), _dev(bias)
    cols = torch.empty((K, N), dtype=torch.float32, device="cuda")
    gc = g.c()
    st = _stream()
    check(lib.bnn_im2col_f32(dx.data_ptr(), *x.shape, 0, B, C.byref(gc), cols.data_ptr(), st))
    check(lib.bnn_sign_f32(cols.data_ptr(), K * N, cols.data_ptr(), st))
    out = torch.empty((B, g.out_channels, oh, ow), dtype=torch.float32, device="cuda")
    check(lib.bnn_float_gemm_f32(dw.data_ptr(), w_pm1.shape[0], K, cols.data_ptr(), N, db.data_ptr(), oh * ow,
                                 out.data_ptr(), st))
    return out.cpu().numpy()


def conv_forward_naive(x, w, bias, geom) -> np.ndarray:
    """network.cpp:96-111: direct convolution (w [D, C, kH, kW]) + bias, on the device."""
    import torch

    x, w, bias = _f32(x), _f32(w), _f32(bias)
    g = ConvGeometry.of(geom)
    oh, ow = output_dims(g, x.shape[2], x.shape[3])
    if bias.size != g.out_channels:
        raise ShapeError("conv: bias length does not match output channels")
    out = torch.empty((x.shape[0], g.out_channels, oh, ow), dtype=torch.float32, device="cuda")
    dx, dw, db = _dev(x), _dev(w), _dev(bias)
    gc = g.c()
    check(load().bnn_conv_forward_naive_f32(dx.data_ptr(), *x.shape, dw.data_ptr(), db.data_ptr(), C.byref(gc),
                                            out.data_ptr(), _stream()))
    return out.cpu().numpy()


def maxpool2(x) -> np.ndarray:
    """network.cpp:133-149."""
    import torch

    x = _f32(x)
    b, c, h, w = x.shape
    out = torch.empty((b, c, h // 2, w // 2), dtype=torch.float32, device="cuda")
    dx = _dev(x)
    check(load().bnn_maxpool2_f32(dx.data_ptr(), b, c, h, w, out.data_ptr(), _stream()))
    return out.cpu().numpy()


def affine_norm(x, scale, shift) -> np.ndarray:
    """network.cpp:151-175 (tensor [B,C,H,W] per channel, or matrix [F, N] per row)."""
    x = _f32(x)
    scale, shift = _f32(scale), _f32(shift)
    if x.ndim == 4:
        channels, plane = x.shape[1], x.shape[2] * x.shape[3]
        what = "channels"
    else:
        channels, plane = x.shape[0], x.shape[1]
        what = "features"
    if scale.size != channels or shift.size != channels:
        raise ShapeError(f"affine_norm: parameter length does not match {what}")
    dx, ds, dt = _dev(x), _dev(scale), _dev(shift)  # keep alive until the kernel has run
    out = dx.clone()
    check(load().bnn_affine_f32(dx.data_ptr(), x.size, channels, plane, ds.data_ptr(),
                                dt.data_ptr(), out.data_ptr(), _stream()))
    return out.cpu().numpy()


def flatten_to_columns(x) -> np.ndarray:
    """network.cpp:177-184: [B, C, H, W] -> [C*H*W, B]."""
    import torch

    x = _f32(x)
    B = x.shape[0]
    F = x.size // B
    out = torch.empty((F, B), dtype=torch.float32, device="cuda")
    dx = _dev(x)
    check(load().bnn_flatten_to_columns_f32(dx.data_ptr(), B, F, out.data_ptr(), _stream()))
    return out.cpu().numpy()


def fnv1a_hash(m: np.ndarray) -> int:
    """bench.cpp:23-33: FNV-1a over the float bytes (bnn_fnv1a_f32)."""
    m = _f32(m)
    h = C.c_uint64()
    dm = _dev(m.reshape(-1))
    check(load().bnn_fnv1a_f32(dm.data_ptr(), m.size, C.byref(h), _stream()))
    return int(h.value)


# --------------------------------------------------------------------- network

KINDS = {"conv": 0, "linear": 1, "maxpool": 2, "affine_norm": 3, "sign": 4, "htanh": 5}


def _pair(v, default):
    if v is None:
        return default, default
    if isinstance(v, (list, tuple)):
        return int(v[0]), int(v[1])
    return int(v), int(v)


KERNELS = {"float": 0, "binary": 1, "naive": 2}


def layer_specs(layers, default_kernel: str = "binary") -> "C.Array":
    """Layer dicts in the reference NetworkSpec JSON vocabulary (network.cpp:487-536)."""
    arr = (LayerSpec * len(layers))()
    for i, l in enumerate(layers):
        k = l["kind"]
        if k not in KINDS:
            raise ConfigError(f"unknown layer kind '{k}'")
        arr[i].kind = KINDS[k]
        kern = l.get("kernel", default_kernel)
        if kern not in KERNELS:
            raise ConfigError(f"unknown kernel choice '{kern}', expected binary|float|naive")
        arr[i].kernel = KERNELS[kern]
        if "seed" in l:
            arr[i].has_seed, arr[i].seed = 1, int(l["seed"])
        arr[i].stride_h = arr[i].stride_w = 1
        if k == "conv":
            kh, kw = _pair(l.get("kernel_size"), 0)
            if kh == 0:
                raise ConfigError("conv layer needs kernel_size")
            arr[i].out_channels = int(l["out_channels"])
            arr[i].kernel_h, arr[i].kernel_w = kh, kw
            arr[i].stride_h, arr[i].stride_w = _pair(l.get("stride"), 1)
            arr[i].pad_h, arr[i].pad_w = _pair(l.get("pad"), 0)
        elif k == "linear":
            arr[i].out_features = int(l["out_features"])
        if k in ("conv", "linear") and l.get("weights_blob"):
            arr[i].weights_blob = str(l["weights_blob"]).encode()  # the array keeps the bytes alive
    return arr


def default_layers() -> list[dict]:
    """build_default_network (network.cpp:422-465) as NetworkSpec layer dicts."""
    out = []
    na = [{"kind": "affine_norm"}, {"kind": "htanh"}, {"kind": "sign"}]
    for i, d in enumerate((128, 128, 256, 256, 512, 512)):
        out.append({"kind": "conv", "out_channels": d, "kernel_size": 3, "pad": 1})
        if i % 2 == 1:
            out.append({"kind": "maxpool"})
        out += [dict(v) for v in na]
    for i, f in enumerate((1024, 1024, 10)):
        out.append({"kind": "linear", "out_features": f})
        if i < 2:
            out += [dict(v) for v in na]
    return out


# ------------------------------------------------------------------ on-disk formats (csrc/io.cpp)


def save_packed_blob(p: PackedBitMatrix, path) -> None:
    """save_packed_blob (binarize.cpp:116-127)."""
    o = 0 if p.orientation == ROW_PACKED else 1
    w = np.ascontiguousarray(p.words, np.uint32)
    check(load().bnn_save_packed_blob(str(path).encode(), o, p.logical_rows, p.logical_cols, _p(w)))


def load_packed_blob(path) -> PackedBitMatrix:
    """load_packed_blob (binarize.cpp:129-148): IoError on a truncated / mismatched / dirty blob."""
    lib = load()
    o, r, c = C.c_int(), C.c_uint64(), C.c_uint64()
    check(lib.bnn_load_packed_blob(str(path).encode(), C.byref(o), C.byref(r), C.byref(c), None, 0))
    p = PackedBitMatrix.make(r.value, c.value, ROW_PACKED if o.value == 0 else COL_PACKED)
    check(lib.bnn_load_packed_blob(str(path).encode(), C.byref(o), C.byref(r), C.byref(c), _p(p.words), p.words.size))
    return p


def save_tensor_blob(x, path) -> None:
    """save_tensor_blob (tensor.cpp:123-134): x is [batch, channels, height, width]."""
    x = _f32(x)
    if x.ndim != 4:
        raise ShapeError("tensor blob needs a 4-d [batch, channels, height, width] array")
    shape = np.asarray(x.shape, np.uint64)
    check(load().bnn_save_tensor_blob(str(path).encode(), _p(shape), _p(x)))


def load_tensor_blob(path) -> np.ndarray:
    """load_tensor_blob (tensor.cpp:136-150)."""
    lib = load()
    shape = np.zeros(4, np.uint64)
    check(lib.bnn_load_tensor_blob(str(path).encode(), _p(shape), None, 0))
    out = np.zeros(tuple(int(v) for v in shape), np.float32)
    check(lib.bnn_load_tensor_blob(str(path).encode(), _p(shape), _p(out), out.size))
    return out


class Network:
    """build_network + network_forward(ExecKernel::Binary) on the current CUDA device."""

    def __init__(self, layers=None, input_chw=(3, 32, 32), seed: int = 1,
                 binarize_weights: bool = False):
        lib = load()
        self.layers = default_layers() if layers is None else list(layers)
        arr = layer_specs(self.layers)
        h = C.c_void_p()
        check(lib.bnn_net_create(C.addressof(arr), len(self.layers), *input_chw, seed,
                                 int(binarize_weights), C.byref(h)))
        self._h = h
        self.input_chw = tuple(input_chw)
        self.logits = int(lib.bnn_net_logits(h))

    @classmethod
    def from_spec_file(cls, path, binarize_weights=None) -> "Network":
        """load_network_spec (network.cpp:487-536) + build_network: a NetworkSpec JSON file,
        layers may take their float weights from a ``weights_blob`` tensor blob."""
        import json as _json

        lib = load()
        h = C.c_void_p()
        check(lib.bnn_net_create_from_spec(str(path).encode(), -1 if binarize_weights is None else int(binarize_weights),
                                           C.byref(h)))
        self = cls.__new__(cls)
        spec = _json.load(open(path))
        self.layers = spec["layers"]
        shape = np.zeros(4, np.uint64)
        n = C.c_size_t()
        check(lib.bnn_spec_info(str(path).encode(), _p(shape), C.byref(n)))
        self._h = h
        self.input_chw = tuple(int(v) for v in shape[1:])
        self.logits = int(lib.bnn_net_logits(h))
        return self

    @classmethod
    def from_spec(cls, spec: dict) -> "Network":
        shape = spec.get("input_shape", [1, 3, 32, 32])
        return cls(spec["layers"], tuple(shape[1:]), int(spec.get("seed", 1)),
                   bool(spec.get("binarize_weights", False)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib._lib is not None:
            _lib._lib.bnn_net_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _check_input(self, shape) -> None:
        """network.cpp:332-337: the input must be [B, C, H, W] with the network's C, H, W."""
        if len(shape) != 4 or tuple(int(v) for v in shape[1:]) != self.input_chw or int(shape[0]) < 1:
            got = "x".join(str(int(v)) for v in shape[1:]) if len(shape) == 4 else f"a {len(shape)}-d array"
            raise ShapeError(f"network input is {got}, network expects " + "x".join(str(v) for v in self.input_chw))

    def forward(self, x) -> np.ndarray:
        """Host buffers in and out (H2D, forward, D2H): [B, C, H, W] -> [features, B]."""
        x = _f32(x)
        self._check_input(x.shape)
        out = np.empty((self.logits, x.shape[0]), np.float32)
        check(load().bnn_host_net_forward(self._h, _p(x), x.shape[0], _p(out)))
        return out

    def forward_device(self, x, out=None, stream=None):
        """torch CUDA tensors in and out, stream-ordered."""
        import torch

        self._check_input(tuple(x.shape))
        if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
            raise ShapeError("forward_device: x must be a contiguous float32 CUDA tensor")
        B = x.shape[0]
        if out is None:
            out = torch.empty((self.logits, B), dtype=torch.float32, device=x.device)
        elif out.dtype != torch.float32 or not out.is_cuda or not out.is_contiguous() or out.numel() < self.logits * B:
            raise ShapeError(f"forward_device: out must be a contiguous float32 CUDA tensor of {self.logits}x{B}")
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(load().bnn_net_forward(self._h, x.data_ptr(), B, out.data_ptr(), st))
        return out

    ENGINES = {"auto": 0, "generic": 1, "fused": 2, "float": 3, "binary_reference": 4, "naive": 5,
               "per_layer": 6}

    def pipeline(self, batch: int, depth: int = 3) -> "Pipeline":
        """A serving pipeline of host-buffer batches (bnn_pipe_*)."""
        return Pipeline(self, batch, depth)

    def set_engine(self, name: str) -> None:
        """Select the device engine (the reference's ExecKernel): "fused" (Binary: one tcgen05
        launch per weighted layer, packed-bit activations), "generic" (Binary, one kernel per
        reference op), "auto" (fused when the topology allows it), "float" (ExecKernel::Float),
        "binary_reference" (ExecKernel::BinaryReference), "naive" (ExecKernel::Naive) or
        "per_layer" (each layer's own kernel). All are bit-exact with the reference."""
        if name not in self.ENGINES:
            raise ConfigError(f"unknown engine '{name}'")
        check(load().bnn_net_set_engine(self._h, self.ENGINES[name]))

    @property
    def engine(self) -> str:
        names = {v: k for k, v in self.ENGINES.items()}
        return names[int(load().bnn_net_engine(self._h))]

    def forward_with(self, x, engine: str) -> np.ndarray:
        """network_forward(net, x, {ExecKernel}) with the engine switched for this call only."""
        prev = int(load().bnn_net_engine(self._h))
        prev_name = "auto" if prev in (1, 2) else {v: k for k, v in self.ENGINES.items()}[prev]
        self.set_engine(engine)
        try:
            return self.forward(x)
        finally:
            self.set_engine(prev_name)

    def verify(self, x, tolerance: float = 1e-4) -> dict:
        """verify_network (bench.cpp:172-191): Binary (the fused engine) against BinaryReference
        (sign(im2col) + float_gemm on sign(weights)), both on the device; the max |delta logit|
        is reduced on the device (bnn_max_abs_diff_f32)."""
        import torch

        x = _f32(x)
        self._check_input(x.shape)
        dx = _dev(x)
        got = torch.empty((self.logits, x.shape[0]), dtype=torch.float32, device="cuda")
        want = torch.empty_like(got)
        st = _stream()
        self.forward_device(dx, got, st)
        lib = load()
        prev = int(lib.bnn_net_engine(self._h))
        check(lib.bnn_net_set_engine(self._h, self.ENGINES["binary_reference"]))
        try:
            check(lib.bnn_net_forward(self._h, dx.data_ptr(), x.shape[0], want.data_ptr(), st))
        finally:
            lib.bnn_net_set_engine(self._h, 0 if prev in (1, 2) else prev)
        dev = C.c_double()
        check(lib.bnn_max_abs_diff_f32(got.data_ptr(), want.data_ptr(), got.numel(), C.byref(dev), st))
        return {"batch": int(x.shape[0]), "compared": int(got.numel()), "max_abs_deviation": dev.value,
                "tolerance": tolerance, "pass": dev.value <= tolerance}

    def layer_data(self, i: int):
        """BuiltLayer parameters of layer i: (packed words, float weights, bias, scale, shift)."""
        lib = load()
        rows, cols = C.c_size_t(), C.c_size_t()
        check(lib.bnn_net_layer_params(self._h, i, None, C.byref(rows), C.byref(cols), None, None, None))
        r, c = rows.value, cols.value
        packed = np.zeros((r, words_per_line(c) if c else 0), np.uint32)
        weights = np.zeros((r, c), np.float32)
        bias = np.zeros(r, np.float32)
        n_aff = self._affine_width(i) if self.layers[i]["kind"] == "affine_norm" else 0
        scale, shift = np.zeros(n_aff, np.float32), np.zeros(n_aff, np.float32)
        check(lib.bnn_net_layer_data(self._h, i, _p(packed) if r else None, _p(weights) if r else None,
                                     _p(bias) if r else None, _p(scale) if n_aff else None,
                                     _p(shift) if n_aff else None))
        return packed, weights, bias, scale, shift

    def set_layer_data(self, i: int, packed=None, weights=None, bias=None, scale=None, shift=None) -> None:
        """Replace layer i's parameters on the device (the reference's net.layers[i] test hook)."""
        arrs = [None if a is None else np.ascontiguousarray(a, dt)
                for a, dt in ((packed, np.uint32), (weights, np.float32), (bias, np.float32), (scale, np.float32),
                              (shift, np.float32))]
        check(load().bnn_net_set_layer_data(self._h, i, *[None if a is None else _p(a) for a in arrs]))

    def last_launches(self) -> int:
        return int(load().bnn_net_last_launches(self._h))

    def device_bytes(self) -> int:
        return int(load().bnn_net_device_bytes(self._h))

    def layer_params(self, i: int):
        lib = load()
        rows, cols = C.c_size_t(), C.c_size_t()
        check(lib.bnn_net_layer_params(self._h, i, None, C.byref(rows), C.byref(cols), None, None, None))
        r, c = rows.value, cols.value
        n_aff = 0
        spec = self.layers[i]
        packed = np.zeros((r, words_per_line(c) if c else 0), np.uint32)
        bias = np.zeros(r, np.float32)
        if spec["kind"] == "affine_norm":
            n_aff = self._affine_width(i)
        scale = np.zeros(n_aff, np.float32)
        shift = np.zeros(n_aff, np.float32)
        check(lib.bnn_net_layer_params(self._h, i, _p(packed) if r else None, None, None,
                                       _p(bias) if r else None, _p(scale) if n_aff else None,
                                       _p(shift) if n_aff else None))
        return packed, bias, scale, shift

    def _affine_width(self, i: int) -> int:
        c, h, w = self.input_chw
        flat = False
        for l in self.layers[:i]:
            k = l["kind"]
            if k == "conv":
                c = int(l["out_channels"])
                oh, ow = output_dims(ConvGeometry(*_pair(l["kernel_size"], 0), *_pair(l.get("stride"), 1),
                                                  *_pair(l.get("pad"), 0), c, c), h, w)
                h, w = oh, ow
            elif k == "linear":
                c, flat = int(l["out_features"]), True
            elif k == "maxpool":
                h, w = h // 2, w // 2
        return c


class Pipeline:
    """Host buffers in and out, batches pipelined (bnn_pipe_*): submit() copies a batch in,
    runs the network and copies its logits back, asynchronously; wait(seq) blocks until batch
    seq's logits are in the buffer passed to submit(). Host buffers should be pinned (e.g.
    torch pin_memory tensors) for the copies to overlap the forward of the previous batch."""

    def __init__(self, net: "Network", batch: int, depth: int = 3):
        h = C.c_void_p()
        check(load().bnn_pipe_create(net._h, batch, depth, C.byref(h)))
        self._h, self._net, self.batch, self.depth = h, net, batch, depth

    def submit(self, x_ptr: int, logits_ptr: int) -> int:
        """x_ptr: host float32 [batch, C, H, W]; logits_ptr: host float32 [features, batch]."""
        seq = C.c_uint64()
        check(load().bnn_pipe_submit(self._h, C.c_void_p(x_ptr), C.c_void_p(logits_ptr), C.byref(seq)))
        return seq.value

    def wait(self, seq: int) -> None:
        check(load().bnn_pipe_wait(self._h, seq))

    def close(self) -> None:
        if self._h:
            load().bnn_pipe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
