"""TEST INFRASTRUCTURE ONLY — CPU checkers for the binarized-layer hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker or the timed CPU
baseline. The product (``paper_1911_04477_b200``) never imports it.

Two checkers live here:

* ``Oracle`` — ``bnn_oracle.c``, a plain-C restatement of the reference algorithm
  (each function cites the reference file:line it follows), built into
  ``oracle/_build/libbnn_oracle.so``.
* ``RefLib`` — the UNMODIFIED reference C++ sources (/root/reference/proj/src)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libbnnref_{v3,v4}.so`` behind
  ``ref_shim.cpp``. Parity of ``Oracle`` is pinned against it and against the
  reference's own known-answer tests (tests/test_oracle.py, tests/golden/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64


def _fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _uptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _iptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def words_per_line(extent: int) -> int:
    return (extent + 31) // 32


def build(ref: bool = True) -> None:
    """Build the checkers (the C restatement always; the reference when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _Layer(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("has_seed", C.c_uint32), ("seed", _U64),
                ("out_channels", _U64), ("kernel_h", _U64), ("kernel_w", _U64),
                ("stride_h", _U64), ("stride_w", _U64), ("pad_h", _U64), ("pad_w", _U64),
                ("out_features", _U64)]


KINDS = {"conv": 0, "linear": 1, "maxpool": 2, "affine_norm": 3, "sign": 4, "htanh": 5}


def layer_array(layers):
    """layers: list of dicts in the reference NetworkSpec JSON vocabulary (network.cpp:487-536)."""
    arr = (_Layer * len(layers))()
    for i, l in enumerate(layers):
        k = l["kind"]
        arr[i].kind = KINDS[k]
        if "seed" in l:
            arr[i].has_seed, arr[i].seed = 1, int(l["seed"])
        if k == "conv":
            ks = l["kernel_size"]
            kh, kw = (ks, ks) if isinstance(ks, int) else ks
            st = l.get("stride", 1)
            sh, sw = (st, st) if isinstance(st, int) else st
            pd = l.get("pad", 0)
            ph, pw = (pd, pd) if isinstance(pd, int) else pd
            arr[i].out_channels = l["out_channels"]
            arr[i].kernel_h, arr[i].kernel_w = kh, kw
            arr[i].stride_h, arr[i].stride_w = sh, sw
            arr[i].pad_h, arr[i].pad_w = ph, pw
        elif k == "linear":
            arr[i].out_features = l["out_features"]
            arr[i].stride_h = arr[i].stride_w = 1
        else:
            arr[i].stride_h = arr[i].stride_w = 1
    return arr


class Oracle:
    """ctypes view of oracle/_build/libbnn_oracle.so (the C restatement)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_build", "libbnn_oracle.so")
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_mix64.restype = _U64
        L.orc_mix64.argtypes = [_U64, _U64]
        L.orc_fill_random.argtypes = [_SZ, _U64, _U64, _P]
        L.orc_sign.argtypes = [_P, _SZ, _P]
        L.orc_htanh.argtypes = [_P, _SZ, _P]
        L.orc_pack.argtypes = [_P, _SZ, _SZ, C.c_int, C.c_int, _P, C.POINTER(_SZ), C.POINTER(_SZ)]
        L.orc_unpack.argtypes = [_P, _SZ, _SZ, C.c_int, _P]
        L.orc_xnor_gemm.argtypes = [_P, _SZ, _P, _SZ, _SZ, _P]
        L.orc_output_dims.argtypes = [_P, _SZ, _SZ, C.POINTER(_SZ), C.POINTER(_SZ)]
        L.orc_im2col.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P]
        L.orc_conv_forward_binary.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, _P]
        L.orc_linear_forward_packed.argtypes = [_P, _SZ, _SZ, _P, _SZ, _P, _P]
        L.orc_maxpool2.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _P]
        L.orc_affine_tensor.argtypes = [_P, _SZ, _SZ, _SZ, _P, _P, _P]
        L.orc_affine_matrix.argtypes = [_P, _SZ, _SZ, _P, _P, _P]
        L.orc_fnv1a.restype = _U64
        L.orc_fnv1a.argtypes = [_P, _SZ]
        L.orc_default_spec.restype = _SZ
        L.orc_default_spec.argtypes = [_P, _SZ]
        L.orc_net_build.restype = _P
        L.orc_net_build.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _U64, C.c_int]
        L.orc_net_free.argtypes = [_P]
        L.orc_net_logits.restype = _SZ
        L.orc_net_logits.argtypes = [_P]
        L.orc_net_layer_params.restype = _SZ
        L.orc_net_layer_params.argtypes = [_P, _SZ, _P, _P, _P, _P]
        L.orc_net_forward.argtypes = [_P, _P, _SZ, _P]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def mix64(self, seed, counter):
        return int(self.lib.orc_mix64(seed, counter))

    def fill_random(self, shape, seed, offset=0):
        n = int(np.prod(shape))
        out = np.empty(n, np.float32)
        self.lib.orc_fill_random(n, seed, offset, out.ctypes.data)
        return out.reshape(shape)

    def sign(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.orc_sign(x.ctypes.data, x.size, out.ctypes.data)
        return out

    def htanh(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self.lib.orc_htanh(x.ctypes.data, x.size, out.ctypes.data)
        return out

    def pack(self, x, orientation, apply_sign=False):
        """orientation 'rows' (pack_rows) or 'cols' (pack_cols); returns [lines, wpl] u32."""
        x = np.ascontiguousarray(x, np.float32)
        rows, cols = x.shape
        o = 0 if orientation == "rows" else 1
        lines, extent = (rows, cols) if o == 0 else (cols, rows)
        out = np.zeros((lines, words_per_line(extent)), np.uint32)
        br, bc = _SZ(), _SZ()
        rc = self.lib.orc_pack(x.ctypes.data, rows, cols, o, int(apply_sign), out.ctypes.data,
                               C.byref(br), C.byref(bc))
        if rc:
            e = OracleError(rc, self.lib.orc_last_error().decode())
            e.position = (br.value, bc.value)
            raise e
        return out

    def unpack(self, words, rows, cols, orientation):
        words = np.ascontiguousarray(words, np.uint32)
        out = np.empty((rows, cols), np.float32)
        self.lib.orc_unpack(words.ctypes.data, rows, cols, 0 if orientation == "rows" else 1,
                            out.ctypes.data)
        return out

    def xnor_gemm(self, w, x, inner_len):
        w = np.ascontiguousarray(w, np.uint32)
        x = np.ascontiguousarray(x, np.uint32)
        out = np.empty((w.shape[0], x.shape[0]), np.int32)
        self._check(self.lib.orc_xnor_gemm(w.ctypes.data, w.shape[0], x.ctypes.data, x.shape[0],
                                           inner_len, out.ctypes.data))
        return out

    @staticmethod
    def _geom(g):
        return np.asarray(g, np.uint64)

    def output_dims(self, geom, h, w):
        g = self._geom(geom)
        oh, ow = _SZ(), _SZ()
        self._check(self.lib.orc_output_dims(g.ctypes.data, h, w, C.byref(oh), C.byref(ow)))
        return oh.value, ow.value

    def im2col(self, x, batch_index, geom):
        x = np.ascontiguousarray(x, np.float32)
        g = self._geom(geom)
        oh, ow = self.output_dims(geom, x.shape[2], x.shape[3])
        out = np.empty((int(g[0] * g[1] * g[6]), oh * ow), np.float32)
        self._check(self.lib.orc_im2col(x.ctypes.data, *x.shape, batch_index, g.ctypes.data,
                                        out.ctypes.data))
        return out

    def conv_forward_binary(self, x, packed_w, bias, geom):
        x = np.ascontiguousarray(x, np.float32)
        g = self._geom(geom)
        oh, ow = self.output_dims(geom, x.shape[2], x.shape[3])
        out = np.empty((x.shape[0], int(g[7]), oh, ow), np.float32)
        pw = np.ascontiguousarray(packed_w, np.uint32)
        b = np.ascontiguousarray(bias, np.float32)
        self._check(self.lib.orc_conv_forward_binary(x.ctypes.data, *x.shape, pw.ctypes.data,
                                                     b.ctypes.data, g.ctypes.data, out.ctypes.data))
        return out

    def linear_forward_packed(self, x, packed_w, bias):
        x = np.ascontiguousarray(x, np.float32)
        pw = np.ascontiguousarray(packed_w, np.uint32)
        b = np.ascontiguousarray(bias, np.float32)
        out = np.empty((pw.shape[0], x.shape[1]), np.float32)
        self._check(self.lib.orc_linear_forward_packed(x.ctypes.data, x.shape[0], x.shape[1],
                                                       pw.ctypes.data, pw.shape[0], b.ctypes.data,
                                                       out.ctypes.data))
        return out

    def maxpool2(self, x):
        x = np.ascontiguousarray(x, np.float32)
        b, c, h, w = x.shape
        out = np.empty((b, c, h // 2, w // 2), np.float32)
        self._check(self.lib.orc_maxpool2(x.ctypes.data, b, c, h, w, out.ctypes.data))
        return out

    def affine_tensor(self, x, scale, shift):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        s = np.ascontiguousarray(scale, np.float32)
        t = np.ascontiguousarray(shift, np.float32)
        self.lib.orc_affine_tensor(x.ctypes.data, x.shape[0], x.shape[1], x.shape[2] * x.shape[3],
                                   s.ctypes.data, t.ctypes.data, out.ctypes.data)
        return out

    def affine_matrix(self, x, scale, shift):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        s = np.ascontiguousarray(scale, np.float32)
        t = np.ascontiguousarray(shift, np.float32)
        self.lib.orc_affine_matrix(x.ctypes.data, x.shape[0], x.shape[1], s.ctypes.data,
                                   t.ctypes.data, out.ctypes.data)
        return out

    def fnv1a(self, x):
        x = np.ascontiguousarray(x, np.float32)
        return int(self.lib.orc_fnv1a(x.ctypes.data, x.size))

    def default_spec(self):
        arr = (_Layer * 64)()
        n = self.lib.orc_default_spec(C.addressof(arr), 64)
        return arr, n

    def net(self, layers=None, input_chw=(3, 32, 32), seed=1, binarize=False):
        if layers is None:
            arr, n = self.default_spec()
        else:
            arr, n = layer_array(layers), len(layers)
        h = self.lib.orc_net_build(C.addressof(arr), n, *input_chw, seed, int(binarize))
        if not h:
            raise OracleError(1, self.lib.orc_last_error().decode())
        return OracleNet(self, h, n, input_chw)


class OracleNet:
    def __init__(self, orc, handle, n_layers, input_chw):
        self.orc, self.h, self.n_layers, self.input_chw = orc, handle, n_layers, input_chw
        self.logits = int(orc.lib.orc_net_logits(handle))

    def __del__(self):
        try:
            self.orc.lib.orc_net_free(self.h)
        except Exception:
            pass

    def forward(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty((self.logits, x.shape[0]), np.float32)
        self.orc._check(self.orc.lib.orc_net_forward(self.h, x.ctypes.data, x.shape[0],
                                                     out.ctypes.data))
        return out


def cpu_has(flag: str) -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return flag in line.split()
    except OSError:
        pass
    return False


def ref_isa() -> str:
    return "v4" if all(cpu_has(f) for f in ("avx512f", "avx512bw", "avx512vl", "avx512_vpopcntdq",
                                               "avx512_bitalg")) else "v3"


class RefLib:
    """ctypes view of the compiled UNMODIFIED reference (oracle/_ref/libbnnref_<isa>.so)."""

    def __init__(self, isa: str | None = None):
        self.isa = isa or ref_isa()
        path = os.path.join(HERE, "_ref", f"libbnnref_{self.isa}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is present")
        L = self.lib = C.CDLL(path)
        L.bnnref_last_error.restype = C.c_char_p
        L.bnnref_mix64.restype = _U64
        L.bnnref_mix64.argtypes = [_U64, _U64]
        L.bnnref_fill_random.argtypes = [_SZ, _U64, _P]
        L.bnnref_output_dims.argtypes = [_P, _SZ, _SZ, C.POINTER(_SZ), C.POINTER(_SZ)]
        L.bnnref_sign.argtypes = [_P, _SZ, _P]
        L.bnnref_htanh.argtypes = [_P, _SZ, _P]
        L.bnnref_pack.argtypes = [_P, _SZ, _SZ, C.c_int, C.c_int, _P]
        L.bnnref_unpack.argtypes = [_P, _SZ, _SZ, C.c_int, _P]
        L.bnnref_xnor_gemm.argtypes = [_P, _SZ, _P, _SZ, _SZ, C.c_uint, _P]
        L.bnnref_im2col.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _SZ, _P, _P]
        L.bnnref_conv_forward_binary.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P, C.c_uint, _P]
        L.bnnref_linear_forward_packed.argtypes = [_P, _SZ, _SZ, _P, _SZ, _P, C.c_uint, _P]
        L.bnnref_maxpool2.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _P]
        L.bnnref_affine_norm_tensor.argtypes = [_P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P]
        L.bnnref_affine_norm_matrix.argtypes = [_P, _SZ, _SZ, _P, _P, _P]
        L.bnnref_fnv1a.restype = _U64
        L.bnnref_fnv1a.argtypes = [_P, _SZ]
        L.bnnref_net_build_default.restype = _P
        L.bnnref_net_build_default.argtypes = [_U64, C.c_int]
        L.bnnref_net_build_file.restype = _P
        L.bnnref_net_build_file.argtypes = [C.c_char_p, C.c_int]
        L.bnnref_net_free.argtypes = [_P]
        L.bnnref_save_packed_blob.argtypes = [C.c_char_p, C.c_int, _SZ, _SZ, _P]
        L.bnnref_load_packed_blob.argtypes = [C.c_char_p, _P, _P]
        L.bnnref_save_tensor_blob.argtypes = [C.c_char_p, _P, _P]
        L.bnnref_load_tensor_blob.argtypes = [C.c_char_p, _P, _P]
        L.bnnref_net_info.argtypes = [_P, _P]
        L.bnnref_net_layer_info.argtypes = [_P, _SZ, _P]
        L.bnnref_net_layer_params.argtypes = [_P, _SZ, _P, _P, _P, _P]
        L.bnnref_net_forward.argtypes = [_P, _P, _SZ, C.c_int, C.c_uint, C.c_uint, _P]
        L.bnnref_run_verify.argtypes = [C.c_char_p, _SZ, _U64, C.POINTER(C.c_double), C.POINTER(_SZ),
                                        C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.bnnref_run_benchmark.argtypes = [C.c_char_p, _SZ, _SZ, _SZ, _U64, C.c_int, C.c_char_p]
        L.bnnref_parse_report.argtypes = [C.c_char_p, C.POINTER(_SZ), C.POINTER(_U64)]

    def run_verify(self, spec_path=None, batch=64, seed=1):
        """run_verify (bench.cpp:193-199) -> the VerifySummary fields."""
        dev, n, ok, pad = C.c_double(), C.c_size_t(), C.c_int(), C.c_int()
        self._check(self.lib.bnnref_run_verify(None if spec_path is None else str(spec_path).encode(), batch, seed,
                                               C.byref(dev), C.byref(n), C.byref(ok), C.byref(pad)))
        return {"max_abs_deviation": dev.value, "compared": n.value, "pass": bool(ok.value),
                "pad_correction_exercised": bool(pad.value)}

    def run_benchmark(self, out_path, spec_path=None, batch=4, iterations=2, warmup=1, seed=1, kernels_mask=3):
        """run_benchmark + emit_report (bench.cpp:102-170, 219-257) into out_path."""
        self._check(self.lib.bnnref_run_benchmark(None if spec_path is None else str(spec_path).encode(), batch,
                                                  iterations, warmup, seed, kernels_mask, str(out_path).encode()))

    def parse_report(self, path):
        """parse_report (bench.cpp:259-303): (kernel count, first kernel's logits hash)."""
        n, h = C.c_size_t(), C.c_uint64()
        self._check(self.lib.bnnref_parse_report(str(path).encode(), C.byref(n), C.byref(h)))
        return n.value, h.value

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.bnnref_last_error().decode())

    def mix64(self, seed, counter):
        return int(self.lib.bnnref_mix64(seed, counter))

    def fill_random(self, shape, seed):
        n = int(np.prod(shape))
        out = np.empty(n, np.float32)
        self._check(self.lib.bnnref_fill_random(n, seed, out.ctypes.data))
        return out.reshape(shape)

    def sign(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._check(self.lib.bnnref_sign(x.ctypes.data, x.size, out.ctypes.data))
        return out

    def htanh(self, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        self._check(self.lib.bnnref_htanh(x.ctypes.data, x.size, out.ctypes.data))
        return out

    def pack(self, x, orientation, apply_sign=False):
        x = np.ascontiguousarray(x, np.float32)
        rows, cols = x.shape
        o = 0 if orientation == "rows" else 1
        lines, extent = (rows, cols) if o == 0 else (cols, rows)
        out = np.zeros((lines, words_per_line(extent)), np.uint32)
        self._check(self.lib.bnnref_pack(x.ctypes.data, rows, cols, o, int(apply_sign),
                                         out.ctypes.data))
        return out

    def unpack(self, words, rows, cols, orientation):
        words = np.ascontiguousarray(words, np.uint32)
        out = np.empty((rows, cols), np.float32)
        self._check(self.lib.bnnref_unpack(words.ctypes.data, rows, cols,
                                           0 if orientation == "rows" else 1, out.ctypes.data))
        return out

    def xnor_gemm(self, w, x, inner_len, threads=1):
        w = np.ascontiguousarray(w, np.uint32)
        x = np.ascontiguousarray(x, np.uint32)
        out = np.empty((w.shape[0], x.shape[0]), np.int32)
        self._check(self.lib.bnnref_xnor_gemm(w.ctypes.data, w.shape[0], x.ctypes.data, x.shape[0],
                                              inner_len, threads, out.ctypes.data))
        return out

    def output_dims(self, geom, h, w):
        g = np.asarray(geom, np.uint64)
        oh, ow = _SZ(), _SZ()
        self._check(self.lib.bnnref_output_dims(g.ctypes.data, h, w, C.byref(oh), C.byref(ow)))
        return oh.value, ow.value

    def im2col(self, x, batch_index, geom):
        x = np.ascontiguousarray(x, np.float32)
        g = np.asarray(geom, np.uint64)
        oh, ow = self.output_dims(geom, x.shape[2], x.shape[3])
        out = np.empty((int(g[0] * g[1] * g[6]), oh * ow), np.float32)
        self._check(self.lib.bnnref_im2col(x.ctypes.data, *x.shape, batch_index, g.ctypes.data,
                                           out.ctypes.data))
        return out

    def conv_forward_binary(self, x, packed_w, bias, geom, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        g = np.asarray(geom, np.uint64)
        oh, ow = self.output_dims(geom, x.shape[2], x.shape[3])
        out = np.empty((x.shape[0], int(g[7]), oh, ow), np.float32)
        pw = np.ascontiguousarray(packed_w, np.uint32)
        b = np.ascontiguousarray(bias, np.float32)
        self._check(self.lib.bnnref_conv_forward_binary(x.ctypes.data, *x.shape, pw.ctypes.data,
                                                        b.ctypes.data, g.ctypes.data, threads,
                                                        out.ctypes.data))
        return out

    def linear_forward_packed(self, x, packed_w, bias, threads=1):
        x = np.ascontiguousarray(x, np.float32)
        pw = np.ascontiguousarray(packed_w, np.uint32)
        b = np.ascontiguousarray(bias, np.float32)
        out = np.empty((pw.shape[0], x.shape[1]), np.float32)
        self._check(self.lib.bnnref_linear_forward_packed(x.ctypes.data, x.shape[0], x.shape[1],
                                                          pw.ctypes.data, pw.shape[0], b.ctypes.data,
                                                          threads, out.ctypes.data))
        return out

    def maxpool2(self, x):
        x = np.ascontiguousarray(x, np.float32)
        b, c, h, w = x.shape
        out = np.empty((b, c, h // 2, w // 2), np.float32)
        self._check(self.lib.bnnref_maxpool2(x.ctypes.data, b, c, h, w, out.ctypes.data))
        return out

    def affine_tensor(self, x, scale, shift):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        s = np.ascontiguousarray(scale, np.float32)
        t = np.ascontiguousarray(shift, np.float32)
        self._check(self.lib.bnnref_affine_norm_tensor(x.ctypes.data, *x.shape, s.ctypes.data,
                                                       t.ctypes.data, out.ctypes.data))
        return out

    def affine_matrix(self, x, scale, shift):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty_like(x)
        s = np.ascontiguousarray(scale, np.float32)
        t = np.ascontiguousarray(shift, np.float32)
        self._check(self.lib.bnnref_affine_norm_matrix(x.ctypes.data, *x.shape, s.ctypes.data,
                                                       t.ctypes.data, out.ctypes.data))
        return out

    def fnv1a(self, x):
        x = np.ascontiguousarray(x, np.float32)
        return int(self.lib.bnnref_fnv1a(x.ctypes.data, x.size))

    def save_packed_blob(self, path, orientation, rows, cols, words):
        w = np.ascontiguousarray(words, np.uint32)
        self._check(self.lib.bnnref_save_packed_blob(str(path).encode(), int(orientation), rows, cols, w.ctypes.data))

    def load_packed_blob(self, path):
        """-> (orientation 0/1, rows, cols, words [lines, wpl])"""
        d = np.zeros(3, np.uint64)
        self._check(self.lib.bnnref_load_packed_blob(str(path).encode(), d.ctypes.data, None))
        o, r, c = (int(v) for v in d)
        lines, extent = (r, c) if o == 0 else (c, r)
        w = np.zeros((lines, words_per_line(extent)), np.uint32)
        self._check(self.lib.bnnref_load_packed_blob(str(path).encode(), d.ctypes.data, w.ctypes.data))
        return o, r, c, w

    def save_tensor_blob(self, path, x):
        x = np.ascontiguousarray(x, np.float32)
        shape = np.asarray(x.shape, np.uint64)
        self._check(self.lib.bnnref_save_tensor_blob(str(path).encode(), shape.ctypes.data, x.ctypes.data))

    def load_tensor_blob(self, path):
        shape = np.zeros(4, np.uint64)
        self._check(self.lib.bnnref_load_tensor_blob(str(path).encode(), shape.ctypes.data, None))
        out = np.zeros(tuple(int(v) for v in shape), np.float32)
        self._check(self.lib.bnnref_load_tensor_blob(str(path).encode(), shape.ctypes.data, out.ctypes.data))
        return out

    def net_default(self, seed=1, binarize=False):
        h = self.lib.bnnref_net_build_default(seed, int(binarize))
        if not h:
            raise OracleError(1, self.lib.bnnref_last_error().decode())
        return RefNet(self, h)

    def net_file(self, path, binarize=-1):
        h = self.lib.bnnref_net_build_file(path.encode(), int(binarize))
        if not h:
            raise OracleError(3, self.lib.bnnref_last_error().decode())
        return RefNet(self, h)


class RefNet:
    def __init__(self, ref, handle):
        self.ref, self.h = ref, handle
        dims = np.zeros(6, np.uint64)
        ref.lib.bnnref_net_info(handle, dims.ctypes.data)
        self.input_shape = tuple(int(v) for v in dims[:4])
        self.logits = int(dims[4])
        self.n_layers = int(dims[5])

    def __del__(self):
        try:
            self.ref.lib.bnnref_net_free(self.h)
        except Exception:
            pass

    def layer_info(self, i):
        info = np.zeros(18, np.uint64)
        self.ref.lib.bnnref_net_layer_info(self.h, i, info.ctypes.data)
        return [int(v) for v in info]

    def layer_params(self, i):
        info = self.layer_info(i)
        rows, wpl, nb, na = info[1], info[3], info[4], info[5]
        packed = np.zeros((rows, wpl), np.uint32)
        bias = np.zeros(nb, np.float32)
        scale = np.zeros(na, np.float32)
        shift = np.zeros(na, np.float32)
        self.ref.lib.bnnref_net_layer_params(self.h, i, packed.ctypes.data, bias.ctypes.data,
                                             scale.ctypes.data, shift.ctypes.data)
        return packed, bias, scale, shift

    def forward(self, x, exec_kind="binary", threads=1, batch_threads=1):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty((self.logits, x.shape[0]), np.float32)
        ek = {"per_layer": 0, "float": 1, "binary": 2, "naive": 3, "binary_reference": 4}[exec_kind]  # ExecKernel (network.hpp:91)
        self.ref._check(self.ref.lib.bnnref_net_forward(self.h, x.ctypes.data, x.shape[0], ek,
                                                        threads, batch_threads, out.ctypes.data))
        return out
