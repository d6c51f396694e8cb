"""ctypes binding of the C ABI (include/bnn_cuda.h) exported by libbnn_b200.so.

The library is built in-tree (paper_1911_04477_b200/build.py). There is no fallback:
if the shared object is missing or the device is not an sm_100 part, every compute call
raises instead of silently running something else.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libbnn_b200.so")

_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64
_I = C.c_int


class BnnError(RuntimeError):
    """Base of the reference's exception family (tensor.hpp:11-25)."""

    code = -1


class ShapeError(BnnError):
    code = 1


class EncodingError(BnnError):
    code = 2


class ConfigError(BnnError):
    code = 3


class CudaError(BnnError):
    code = 4


class IoError(BnnError):
    code = 5


_ERRORS = {1: ShapeError, 2: EncodingError, 3: ConfigError, 4: CudaError, 5: IoError}


class ConvGeom(C.Structure):
    """bnn_conv_geom == ConvGeometry (tensor.hpp:101-111), same field order."""

    _fields_ = [("kernel_h", _U64), ("kernel_w", _U64), ("stride_h", _U64), ("stride_w", _U64),
                ("pad_h", _U64), ("pad_w", _U64), ("in_channels", _U64), ("out_channels", _U64)]


class LayerSpec(C.Structure):
    """bnn_layer_spec == LayerSpec (network.hpp:23-39); kernel = KernelChoice (0 float, 1 binary,
    2 naive), used by the per-layer engine."""

    _fields_ = [("kind", C.c_uint32), ("has_seed", C.c_uint32), ("seed", _U64),
                ("out_channels", _U64), ("kernel_h", _U64), ("kernel_w", _U64),
                ("stride_h", _U64), ("stride_w", _U64), ("pad_h", _U64), ("pad_w", _U64),
                ("out_features", _U64), ("weights_blob", C.c_char_p), ("kernel", C.c_uint32),
                ("reserved", C.c_uint32)]


_SIGS = {
    "bnn_last_error": (C.c_char_p, []),
    "bnn_version": (_I, []),
    "bnn_last_gemm_kernel": (C.c_char_p, []),
    "bnn_set_gemm_policy": (_I, [_I]),
    "bnn_words_per_line": (_SZ, [_SZ]),
    "bnn_output_dims": (_I, [_P, _SZ, _SZ, C.POINTER(_SZ), C.POINTER(_SZ)]),
    "bnn_sign_pack_cols_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _P]),
    "bnn_sign_pack_rows_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _P]),
    "bnn_pack_cols_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _P, _P]),
    "bnn_pack_rows_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _P, _P]),
    "bnn_unpack_f32": (_I, [_P, _SZ, _SZ, _SZ, _I, _P, _P]),
    "bnn_im2col_sign_pack_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _SZ, _P]),
    "bnn_xnor_gemm_s32": (_I, [_P, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P, _SZ, _P]),
    "bnn_xnor_gemm_bias_f32": (_I, [_P, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P, _SZ, _P, _P]),
    "bnn_conv_forward_binary_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _SZ, _P, _P, _P, _P]),
    "bnn_linear_forward_packed_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _SZ, _P, _P, _P]),
    "bnn_sign_f32": (_I, [_P, _SZ, _P, _P]),
    "bnn_htanh_f32": (_I, [_P, _SZ, _P, _P]),
    "bnn_maxpool2_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P]),
    "bnn_affine_f32": (_I, [_P, _SZ, _SZ, _SZ, _P, _P, _P, _P]),
    "bnn_flatten_to_columns_f32": (_I, [_P, _SZ, _SZ, _P, _P]),
    "bnn_to_float_s32": (_I, [_P, _SZ, _P, _P]),
    "bnn_bias_add_f32": (_I, [_P, _SZ, _SZ, _P, _P]),
    "bnn_fill_random_f32": (_I, [_U64, _U64, _SZ, _P, _P]),
    "bnn_mix64": (_U64, [_U64, _U64]),
    "bnn_fnv1a_f32": (_I, [_P, _SZ, C.POINTER(_U64), _P]),
    "bnn_default_spec": (_SZ, [_P, _SZ]),
    "bnn_net_create": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _U64, _I, C.POINTER(_P)]),
    "bnn_net_destroy": (None, [_P]),
    "bnn_net_logits": (_SZ, [_P]),
    "bnn_net_num_layers": (_SZ, [_P]),
    "bnn_net_layer_params": (_I, [_P, _SZ, _P, C.POINTER(_SZ), C.POINTER(_SZ), _P, _P, _P]),
    "bnn_net_layer_data": (_I, [_P, _SZ, _P, _P, _P, _P, _P]),
    "bnn_net_set_layer_data": (_I, [_P, _SZ, _P, _P, _P, _P, _P]),
    "bnn_net_set_layer_kernel": (_I, [_P, _SZ, _I]),
    "bnn_im2col_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P, _P]),
    "bnn_col2im_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _SZ, _P, C.POINTER(_SZ), C.POINTER(_SZ), _P]),
    "bnn_conv_forward_naive_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P, _P]),
    "bnn_max_abs_diff_f32": (_I, [_P, _P, _SZ, C.POINTER(C.c_double), _P]),
    "bnn_run_verify": (_I, [C.c_char_p, _SZ, _U64, C.c_char_p, C.POINTER(C.c_double), C.POINTER(_SZ),
                            C.POINTER(_I), C.POINTER(_I)]),
    "bnn_run_benchmark": (_I, [C.c_char_p, _SZ, _SZ, _SZ, _U64, _I, _I, C.c_char_p]),
    "bnn_net_forward": (_I, [_P, _P, _SZ, _P, _P]),
    "bnn_net_last_launches": (_SZ, [_P]),
    "bnn_net_set_engine": (_I, [_P, _I]),
    "bnn_net_engine": (_I, [_P]),
    "bnn_net_set_graphs": (_I, [_P, _I]),
    "bnn_set_fused_tiling": (_I, [_I, _I]),
    "bnn_set_fused_split": (_I, [_I]),
    "bnn_debug_timeline": (_I, [_I]),
    "bnn_set_fused_swap": (_I, [_I]),
    "bnn_set_fused_small_logits": (_I, [_I]),
    "bnn_set_fused_pix_popc": (_I, [_I]),
    "bnn_set_fused_fp4": (_I, [_I]),
    "bnn_set_fused_halo": (_I, [_I]),
    "bnn_set_fused_halo0": (_I, [_I]),
    "bnn_set_fused_lin4": (_I, [_I]),
    "bnn_set_fused_fp4_pair": (_I, [_I]),
    "bnn_float_gemm_f32": (_I, [_P, _SZ, _SZ, _P, _SZ, _P, _SZ, _P, _P]),
    "bnn_net_layer_kernel": (C.c_char_p, [_P, _SZ]),
    "bnn_conv_forward_float_f32": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P, _P]),
    "bnn_save_packed_blob": (_I, [C.c_char_p, _I, _U64, _U64, _P]),
    "bnn_load_packed_blob": (_I, [C.c_char_p, C.POINTER(_I), C.POINTER(_U64), C.POINTER(_U64), _P, _SZ]),
    "bnn_save_tensor_blob": (_I, [C.c_char_p, _P, _P]),
    "bnn_load_tensor_blob": (_I, [C.c_char_p, _P, _P, _SZ]),
    "bnn_net_create_from_spec": (_I, [C.c_char_p, _I, _P]),
    "bnn_spec_info": (_I, [C.c_char_p, _P, C.POINTER(_SZ)]),
    "bnn_net_set_timing": (_I, [_P, _I]),
    "bnn_net_timing": (_I, [_P, _P, _P, _P]),
    "bnn_net_reset_timing": (_I, [_P]),
    "bnn_net_layer_shape": (_I, [_P, _SZ, _P]),
    "bnn_net_device_bytes": (_SZ, [_P]),
    "bnn_probe_popc_peak": (_I, [C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "bnn_probe_bmma_peak": (_I, [C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "bnn_probe_umma_peak": (_I, [_I, _I, C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "bnn_host_sign_pack": (_I, [_P, _SZ, _SZ, _I, _I, _P]),
    "bnn_host_xnor_gemm": (_I, [_P, _SZ, _P, _SZ, _SZ, _P]),
    "bnn_host_conv_forward_binary": (_I, [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P]),
    "bnn_host_linear_forward_packed": (_I, [_P, _SZ, _SZ, _P, _SZ, _P, _P]),
    "bnn_host_net_forward": (_I, [_P, _P, _SZ, _P]),
    "bnn_pipe_create": (_I, [_P, _SZ, _I, _P]),
    "bnn_pipe_submit": (_I, [_P, _P, _P, _P]),
    "bnn_pipe_wait": (_I, [_P, _U64]),
    "bnn_pipe_destroy": (_I, [_P]),
}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libbnn_b200.so (RTLD_GLOBAL not needed) and attach the C signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().bnn_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, BnnError)(last_error())
