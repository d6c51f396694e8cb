"""B200-native (sm_100a) binarized-layer hot path of arXiv 1911.04477.

sign-binarize + bit-pack encoder (K1), binary im2col (K2) and the xnor-popcount GEMM (K3)
behind the reference's operator API. The compute lives in ``libbnn_b200.so`` (CUDA C++
behind the C ABI of ``include/bnn_cuda.h``); this package is the Python mirror of the
reference interface (``api``) plus the ctypes binding (``_lib``).
"""
from ._lib import (BnnError, ConfigError, CudaError, EncodingError, IoError, ShapeError,  # noqa: F401
                   EXPORTS, LIB_PATH, load)
from .api import (COL_PACKED, ROW_PACKED, ConvGeometry, Network, PackedBitMatrix, Pipeline,  # noqa: F401
                  affine_norm, bias_add, col2im, conv_forward_binary, conv_forward_binary_reference,
                  conv_forward_float, conv_forward_naive, default_layers, fill_random, flatten_to_columns,
                  float_gemm, fnv1a_hash, htanh, im2col, im2col_sign_pack, linear_forward,
                  linear_forward_binary_reference, linear_forward_packed, load_packed_blob,
                  load_tensor_blob, maxpool2, mix64, output_dims, pack_cols, pack_rows, save_packed_blob,
                  save_tensor_blob, sign, sign_pack_cols, sign_pack_rows, to_float, unpack,
                  words_per_line, xnor_gemm)
