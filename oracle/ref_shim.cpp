// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference CPU library (bnncore), compiled
// straight from /root/reference/proj/src with -Dbnn=bnnref by oracle/Makefile.
// It exposes the reference's hot-path operators with plain pointers so the
// Python tests (tests/), the golden-vector generator (tools/make_golden.py) and
// bench.py's CPU-baseline leg can call the real reference implementation.
//
// Every function forwards to the reference symbol named in its comment; the
// only logic here is marshalling between flat buffers and the reference types
// (FloatTensor / FloatMatrix / PackedBitMatrix, tensor.hpp:28-98).
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "bnn/bench.hpp"
#include "bnn/binarize.hpp"
#include "bnn/kernels.hpp"
#include "bnn/lowering.hpp"
#include "bnn/network.hpp"
#include "bnn/tensor.hpp"

using namespace bnnref;  // the reference namespace, renamed by -Dbnn=bnnref

namespace {

thread_local std::string g_err;

// 0 ok, 1 ShapeError, 2 EncodingError, 3 ConfigError, 5 IoError, 9 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const EncodingError& e) {
        g_err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

FloatMatrix make_matrix(const float* x, std::size_t rows, std::size_t cols) {
    FloatMatrix m(rows, cols);
    std::memcpy(m.data.data(), x, rows * cols * sizeof(float));
    return m;
}

FloatTensor make_tensor(const float* x, std::size_t b, std::size_t c, std::size_t h,
                        std::size_t w) {
    FloatTensor t(b, c, h, w);
    std::memcpy(t.data.data(), x, t.data.size() * sizeof(float));
    return t;
}

PackedBitMatrix make_packed(const std::uint32_t* words, std::size_t rows, std::size_t cols,
                            PackOrientation o) {
    PackedBitMatrix p = PackedBitMatrix::make(rows, cols, o);
    std::memcpy(p.words.data(), words, p.words.size() * sizeof(std::uint32_t));
    return p;
}

ConvGeometry make_geom(const std::size_t g[8]) {
    return ConvGeometry{g[0], g[1], g[2], g[3], g[4], g[5], g[6], g[7]};
}

}  // namespace

extern "C" {

const char* bnnref_last_error() { return g_err.c_str(); }

// tensor.cpp:65-71
std::uint64_t bnnref_mix64(std::uint64_t seed, std::uint64_t counter) { return mix64(seed, counter); }

// tensor.cpp:73-77 / 85-89 (fill_random_matrix is the same stream over a flat index)
int bnnref_fill_random(std::size_t n, std::uint64_t seed, float* out) {
    return guarded([&] {
        FloatMatrix m = fill_random_matrix(1, n, seed);
        std::memcpy(out, m.data.data(), n * sizeof(float));
    });
}

// tensor.cpp:46-63
int bnnref_output_dims(const std::size_t geom[8], std::size_t in_h, std::size_t in_w,
                       std::size_t* out_h, std::size_t* out_w) {
    return guarded([&] {
        auto [h, w] = output_dims(make_geom(geom), in_h, in_w);
        *out_h = h;
        *out_w = w;
    });
}

// binarize.cpp:19-27
int bnnref_sign(const float* x, std::size_t n, float* out) {
    return guarded([&] {
        FloatMatrix s = sign(make_matrix(x, 1, n));
        std::memcpy(out, s.data.data(), n * sizeof(float));
    });
}

// binarize.cpp:29-37
int bnnref_htanh(const float* x, std::size_t n, float* out) {
    return guarded([&] {
        FloatMatrix s = htanh(make_matrix(x, 1, n));
        std::memcpy(out, s.data.data(), n * sizeof(float));
    });
}

// binarize.cpp:39-73. orientation 0 = pack_rows, 1 = pack_cols. apply_sign != 0
// runs sign() first (the hot-path composition pack_cols(sign(x)), network.cpp:72,123).
int bnnref_pack(const float* x, std::size_t rows, std::size_t cols, int orientation,
                int apply_sign, std::uint32_t* out) {
    return guarded([&] {
        FloatMatrix m = make_matrix(x, rows, cols);
        if (apply_sign) m = sign(std::move(m));
        PackedBitMatrix p = orientation == 0 ? pack_rows(m) : pack_cols(m);
        std::memcpy(out, p.words.data(), p.words.size() * sizeof(std::uint32_t));
    });
}

// binarize.cpp:75-90
int bnnref_unpack(const std::uint32_t* words, std::size_t rows, std::size_t cols,
                  int orientation, float* out) {
    return guarded([&] {
        FloatMatrix m = unpack(make_packed(words, rows, cols,
                                           orientation == 0 ? PackOrientation::RowPacked
                                                            : PackOrientation::ColPacked));
        std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    });
}

// kernels.cpp:53-88. w: M lines (row-packed [M, L]); x: N lines (col-packed [L, N]).
int bnnref_xnor_gemm(const std::uint32_t* w, std::size_t m, const std::uint32_t* x,
                     std::size_t n, std::size_t inner_len, unsigned threads, std::int32_t* out) {
    return guarded([&] {
        PackedBitMatrix pw = make_packed(w, m, inner_len, PackOrientation::RowPacked);
        PackedBitMatrix px = make_packed(x, inner_len, n, PackOrientation::ColPacked);
        IntMatrix r = xnor_gemm(pw, px, inner_len, threads);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(std::int32_t));
    });
}

// lowering.cpp:7-43
int bnnref_im2col(const float* x, std::size_t b, std::size_t c, std::size_t h, std::size_t w,
                  std::size_t batch_index, const std::size_t geom[8], float* out) {
    return guarded([&] {
        FloatMatrix m = im2col(make_tensor(x, b, c, h, w), batch_index, make_geom(geom));
        std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
    });
}

// network.cpp:65-79. packed_w: D lines of ceil(K/32) words (row-packed sign weights).
int bnnref_conv_forward_binary(const float* x, std::size_t b, std::size_t c, std::size_t h,
                               std::size_t w, const std::uint32_t* packed_w, const float* bias,
                               const std::size_t geom[8], unsigned threads, float* out) {
    return guarded([&] {
        const ConvGeometry g = make_geom(geom);
        PackedBitMatrix pw =
            make_packed(packed_w, g.out_channels, g.patch_len(), PackOrientation::RowPacked);
        std::vector<float> bv(bias, bias + g.out_channels);
        FloatTensor y = conv_forward_binary(make_tensor(x, b, c, h, w), pw, bv, g, threads);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// network.cpp:121-126. x: [K, N] features x batch; packed_w: M lines x ceil(K/32).
int bnnref_linear_forward_packed(const float* x, std::size_t k, std::size_t n,
                                 const std::uint32_t* packed_w, std::size_t m, const float* bias,
                                 unsigned threads, float* out) {
    return guarded([&] {
        PackedBitMatrix pw = make_packed(packed_w, m, k, PackOrientation::RowPacked);
        std::vector<float> bv(bias, bias + m);
        FloatMatrix y = linear_forward_packed(make_matrix(x, k, n), pw, bv, threads);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// network.cpp:133-149
int bnnref_maxpool2(const float* x, std::size_t b, std::size_t c, std::size_t h, std::size_t w,
                    float* out) {
    return guarded([&] {
        FloatTensor y = maxpool2(make_tensor(x, b, c, h, w));
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// network.cpp:151-165 (tensor form, per channel)
int bnnref_affine_norm_tensor(const float* x, std::size_t b, std::size_t c, std::size_t h,
                              std::size_t w, const float* scale, const float* shift, float* out) {
    return guarded([&] {
        std::vector<float> s(scale, scale + c), t(shift, shift + c);
        FloatTensor y = affine_norm(make_tensor(x, b, c, h, w), s, t);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// network.cpp:167-175 (matrix form, per row feature)
int bnnref_affine_norm_matrix(const float* x, std::size_t rows, std::size_t cols,
                              const float* scale, const float* shift, float* out) {
    return guarded([&] {
        std::vector<float> s(scale, scale + rows), t(shift, shift + rows);
        FloatMatrix y = affine_norm(make_matrix(x, rows, cols), s, t);
        std::memcpy(out, y.data.data(), y.data.size() * sizeof(float));
    });
}

// bench.cpp:23-33
std::uint64_t bnnref_fnv1a(const float* x, std::size_t n) {
    return fnv1a_hash(make_matrix(x, 1, n));
}

// ------------------------------------------------------------- networks

struct RefNet {
    Network net;
};

// network.cpp:422-465 + network.cpp:203-306
void* bnnref_net_build_default(std::uint64_t seed, int binarize_weights) {
    RefNet* r = nullptr;
    int rc = guarded([&] {
        NetworkSpec spec = build_default_network(KernelChoice::Binary, seed);
        spec.binarize_weights = binarize_weights != 0;
        r = new RefNet{build_network(spec)};
    });
    return rc == 0 ? r : nullptr;
}

// network.cpp:487-536 + network.cpp:203-306. binarize < 0 keeps the file's value.
void* bnnref_net_build_file(const char* path, int binarize_weights) {
    RefNet* r = nullptr;
    int rc = guarded([&] {
        NetworkSpec spec = load_network_spec(path);
        if (binarize_weights >= 0) spec.binarize_weights = binarize_weights != 0;
        r = new RefNet{build_network(spec)};
    });
    return rc == 0 ? r : nullptr;
}

void bnnref_net_free(void* h) { delete static_cast<RefNet*>(h); }

// save_packed_blob / load_packed_blob (binarize.cpp:116-148)
int bnnref_save_packed_blob(const char* path, int orientation, std::size_t rows, std::size_t cols,
                            const std::uint32_t* words) {
    return guarded([&] {
        PackedBitMatrix p = PackedBitMatrix::make(rows, cols, static_cast<PackOrientation>(orientation));
        std::memcpy(p.words.data(), words, p.words.size() * 4);
        save_packed_blob(p, path);
    });
}

// dims[0] = orientation, dims[1] = rows, dims[2] = cols; words NULL: header only
int bnnref_load_packed_blob(const char* path, std::size_t dims[3], std::uint32_t* words) {
    return guarded([&] {
        PackedBitMatrix p = load_packed_blob(path);
        dims[0] = static_cast<std::size_t>(p.orientation);
        dims[1] = p.logical_rows;
        dims[2] = p.logical_cols;
        if (words) std::memcpy(words, p.words.data(), p.words.size() * 4);
    });
}

// save_tensor_blob / load_tensor_blob (tensor.cpp:123-150)
int bnnref_save_tensor_blob(const char* path, const std::size_t shape[4], const float* data) {
    return guarded([&] { save_tensor_blob(make_tensor(data, shape[0], shape[1], shape[2], shape[3]), path); });
}

int bnnref_load_tensor_blob(const char* path, std::size_t shape[4], float* data) {
    return guarded([&] {
        FloatTensor t = load_tensor_blob(path);
        shape[0] = t.batch, shape[1] = t.channels, shape[2] = t.height, shape[3] = t.width;
        if (data) std::memcpy(data, t.data.data(), t.data.size() * 4);
    });
}

// dims[0..3] = default input shape (B, C, H, W), dims[4] = logits, dims[5] = layer count
void bnnref_net_info(void* h, std::size_t dims[6]) {
    const Network& n = static_cast<RefNet*>(h)->net;
    dims[0] = n.spec.input_shape[0];
    dims[1] = n.in_channels;
    dims[2] = n.in_h;
    dims[3] = n.in_w;
    dims[4] = n.logits;
    dims[5] = n.layers.size();
}

// Per-layer parameters, so the device network build can be checked field by field.
// info[0] kind (LayerKind order), [1] rows of packed weights, [2] cols (L),
// [3] words per line, [4] bias len, [5] scale/shift len, [6..13] geometry,
// [14..17] out (C, H, W, flat)
void bnnref_net_layer_info(void* h, std::size_t i, std::size_t info[18]) {
    const BuiltLayer& l = static_cast<RefNet*>(h)->net.layers[i];
    std::memset(info, 0, 18 * sizeof(std::size_t));
    info[0] = static_cast<std::size_t>(l.spec.kind);
    info[1] = l.packed_weights.logical_rows;
    info[2] = l.packed_weights.logical_cols;
    info[3] = l.packed_weights.words_per_line;
    info[4] = l.bias.size();
    info[5] = l.scale.size();
    const ConvGeometry& g = l.geom;
    const std::size_t gv[8] = {g.kernel_h, g.kernel_w, g.stride_h, g.stride_w,
                               g.pad_h,    g.pad_w,    g.in_channels, g.out_channels};
    for (int k = 0; k < 8; ++k) info[6 + k] = gv[k];
    info[14] = l.out_channels;
    info[15] = l.out_h;
    info[16] = l.out_w;
    info[17] = l.out_flat ? 1 : 0;
}

void bnnref_net_layer_params(void* h, std::size_t i, std::uint32_t* packed, float* bias,
                             float* scale, float* shift) {
    const BuiltLayer& l = static_cast<RefNet*>(h)->net.layers[i];
    if (packed && !l.packed_weights.words.empty())
        std::memcpy(packed, l.packed_weights.words.data(), l.packed_weights.byte_size());
    if (bias && !l.bias.empty()) std::memcpy(bias, l.bias.data(), l.bias.size() * sizeof(float));
    if (scale && !l.scale.empty())
        std::memcpy(scale, l.scale.data(), l.scale.size() * sizeof(float));
    if (shift && !l.shift.empty())
        std::memcpy(shift, l.shift.data(), l.shift.size() * sizeof(float));
}

// network.cpp:330-420. exec: the ExecKernel value (0 PerLayer, 1 Float, 2 Binary, 3 Naive,
// 4 BinaryReference).
// x: [B, C, H, W]; logits: [features, B] (network.hpp:104-105).
// batch_threads > 1 splits the batch into contiguous shards, one std::thread per
// shard, each calling the reference network_forward on its slice (re-entrant,
// SPEC.md:301); the [features, shard] results are reassembled column-wise.
int bnnref_net_forward(void* h, const float* x, std::size_t batch, int exec, unsigned threads,
                       unsigned batch_threads, float* logits) {
    return guarded([&] {
        const Network& net = static_cast<RefNet*>(h)->net;
        const ExecKernel ek = static_cast<ExecKernel>(exec);
        const std::size_t per = net.in_channels * net.in_h * net.in_w;
        const std::size_t feats = net.logits;
        unsigned shards = batch_threads < 1 ? 1 : batch_threads;
        if (shards > batch) shards = static_cast<unsigned>(batch);
        const std::size_t chunk = (batch + shards - 1) / shards;
        std::vector<std::string> errs(shards);
        auto run = [&](unsigned s) {
            const std::size_t lo = s * chunk, hi = std::min(batch, lo + chunk);
            if (lo >= hi) return;
            try {
                FloatTensor xs = make_tensor(x + lo * per, hi - lo, net.in_channels, net.in_h,
                                             net.in_w);
                FloatMatrix y = network_forward(net, xs, ForwardOptions{ek, threads, nullptr});
                for (std::size_t f = 0; f < feats; ++f)
                    for (std::size_t j = 0; j < hi - lo; ++j)
                        logits[f * batch + lo + j] = y.at(f, j);
            } catch (const std::exception& e) {
                errs[s] = e.what();
            }
        };
        if (shards == 1) {
            run(0);
        } else {
            std::vector<std::thread> pool;
            for (unsigned s = 0; s < shards; ++s) pool.emplace_back(run, s);
            for (auto& t : pool) t.join();
        }
        for (auto& e : errs)
            if (!e.empty()) throw ShapeError(e);
    });
}

// run_verify (bench.cpp:193-199): spec_path NULL -> the default network.
int bnnref_run_verify(const char* spec_path, std::size_t batch, std::uint64_t seed, double* max_dev,
                      std::size_t* compared, int* pass, int* pad_exercised) {
    return guarded([&] {
        BenchConfig cfg;
        cfg.spec_path = spec_path ? spec_path : "";
        cfg.batch = batch;
        cfg.seed = seed;
        const VerifySummary s = run_verify(cfg);
        *max_dev = s.max_abs_deviation;
        *compared = s.compared;
        *pass = s.pass ? 1 : 0;
        *pad_exercised = s.pad_correction_exercised ? 1 : 0;
    });
}

// run_benchmark (bench.cpp:102-170) + emit_report (bench.cpp:219-257). kernels_mask: bit 0
// Binary, bit 1 Float, bit 2 Naive, in that order.
int bnnref_run_benchmark(const char* spec_path, std::size_t batch, std::size_t iterations,
                         std::size_t warmup, std::uint64_t seed, int kernels_mask,
                         const char* out_path) {
    return guarded([&] {
        BenchConfig cfg;
        cfg.spec_path = spec_path ? spec_path : "";
        cfg.batch = batch;
        cfg.iterations = iterations;
        cfg.warmup = warmup;
        cfg.seed = seed;
        cfg.kernels.clear();
        if (kernels_mask & 1) cfg.kernels.push_back(KernelChoice::Binary);
        if (kernels_mask & 2) cfg.kernels.push_back(KernelChoice::Float);
        if (kernels_mask & 4) cfg.kernels.push_back(KernelChoice::Naive);
        emit_report(run_benchmark(cfg), out_path);
    });
}

// parse_report (bench.cpp:259-303): 1 when the reference parser accepts the file; the
// network name and the first kernel's logits hash come back for cross-checking.
int bnnref_parse_report(const char* path, std::size_t* n_kernels, std::uint64_t* first_hash) {
    return guarded([&] {
        const BenchReport r = parse_report(path);
        *n_kernels = r.kernels.size();
        *first_hash = r.kernels.empty() ? 0 : r.kernels.front().logits_hash;
    });
}

}  // extern "C"
