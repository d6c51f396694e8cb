// C++ reference-signature API (include/bnn_b200.hpp) over the C ABI (include/bnn_cuda.h).
//
// Every function keeps the reference's contract (argument checks, exception type and message,
// return-by-value) and does its arithmetic on the device: host buffers are copied in, the
// sm_100a kernels run on the legacy default stream, results are copied back. Layout-only
// operations with no arithmetic (reshape_output, flatten_weights: a row-major reinterpretation,
// lowering.cpp:87-102) stay host memcpys like the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "bnn_b200.hpp"
#include "bnn_cuda.h"
#include "cpp_internal.hpp"

namespace bnn {
namespace {

using namespace cppi;

// unary elementwise op (0 sign, 1 htanh) on the device
std::vector<float> unary(const std::vector<float>& x, int op) {
    std::vector<float> out(x.size());
    if (x.empty()) return out;
    Dev d(x.size() * 4);
    d.put(x.data(), x.size() * 4);
    check(op == 0 ? bnn_sign_f32(d.as<float>(), x.size(), d.as<float>(), nullptr)
                  : bnn_htanh_f32(d.as<float>(), x.size(), d.as<float>(), nullptr));
    d.get(out.data(), out.size() * 4);
    return out;
}

PackedBitMatrix pack(const FloatMatrix& m, PackOrientation o, bool apply_sign) {
    PackedBitMatrix p = PackedBitMatrix::make(m.rows, m.cols, o);
    check(bnn_host_sign_pack(m.data.data(), m.rows, m.cols, o == PackOrientation::RowPacked ? 0 : 1,
                             apply_sign ? 1 : 0, p.words.data()));
    return p;
}

std::vector<float> generate(std::size_t n, std::uint64_t seed) {
    std::vector<float> out(n);
    Dev d(n * 4);
    check(bnn_fill_random_f32(seed, 0, n, d.as<float>(), nullptr));
    d.get(out.data(), n * 4);
    return out;
}

}  // namespace

FloatTensor::FloatTensor(std::size_t n, std::size_t c, std::size_t h, std::size_t w)
    : batch(n), channels(c), height(h), width(w) {
    check_extent(n, "batch");
    check_extent(c, "channels");
    check_extent(h, "height");
    check_extent(w, "width");
    data.assign(n * c * h * w, 0.0f);
}

FloatMatrix::FloatMatrix(std::size_t r, std::size_t c) : rows(r), cols(c) {
    check_extent(r, "rows");
    check_extent(c, "cols");
    data.assign(r * c, 0.0f);
}

PackedBitMatrix PackedBitMatrix::make(std::size_t rows, std::size_t cols, PackOrientation o) {
    check_extent(rows, "rows");
    check_extent(cols, "cols");
    PackedBitMatrix p;
    p.logical_rows = rows, p.logical_cols = cols, p.orientation = o;
    p.words_per_line = bnn_words_per_line(p.packed_extent());
    p.pad_bits_per_line = p.words_per_line * kWordBits - p.packed_extent();
    p.words.assign(p.words_per_line * p.lines(), 0u);
    return p;
}

std::pair<std::size_t, std::size_t> output_dims(const ConvGeometry& geom, std::size_t in_h, std::size_t in_w) {
    const bnn_conv_geom g = to_c(geom);
    std::size_t oh = 0, ow = 0;
    check(bnn_output_dims(&g, in_h, in_w, &oh, &ow));
    return {oh, ow};
}

std::uint64_t mix64(std::uint64_t seed, std::uint64_t counter) { return bnn_mix64(seed, counter); }

float unit_random(std::uint64_t seed, std::uint64_t index) {
    const std::uint32_t top = static_cast<std::uint32_t>(bnn_mix64(seed, index) >> 40);
    return static_cast<float>(top) * 0x1.0p-23f - 1.0f;
}

FloatTensor fill_random(std::size_t n, std::size_t c, std::size_t h, std::size_t w, std::uint64_t seed) {
    FloatTensor t(n, c, h, w);
    t.data = generate(t.size(), seed);
    return t;
}

FloatMatrix fill_random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed) {
    FloatMatrix m(rows, cols);
    m.data = generate(m.data.size(), seed);
    return m;
}

std::vector<float> fill_random_vector(std::size_t len, std::uint64_t seed) { return generate(len, seed); }

FloatTensor sign(FloatTensor x) {
    x.data = unary(x.data, 0);
    return x;
}
FloatMatrix sign(FloatMatrix x) {
    x.data = unary(x.data, 0);
    return x;
}
FloatTensor htanh(FloatTensor x) {
    x.data = unary(x.data, 1);
    return x;
}
FloatMatrix htanh(FloatMatrix x) {
    x.data = unary(x.data, 1);
    return x;
}

PackedBitMatrix pack_rows(const FloatMatrix& w) { return pack(w, PackOrientation::RowPacked, false); }
PackedBitMatrix pack_cols(const FloatMatrix& x) { return pack(x, PackOrientation::ColPacked, false); }
PackedBitMatrix sign_pack_rows(const FloatMatrix& w) { return pack(w, PackOrientation::RowPacked, true); }
PackedBitMatrix sign_pack_cols(const FloatMatrix& x) { return pack(x, PackOrientation::ColPacked, true); }

FloatMatrix unpack(const PackedBitMatrix& p) {
    FloatMatrix m(p.logical_rows, p.logical_cols);
    Dev dw(p.byte_size()), dm(m.data.size() * 4);
    dw.put(p.words.data(), p.byte_size());
    check(bnn_unpack_f32(dw.as<std::uint32_t>(), p.words_per_line, p.logical_rows, p.logical_cols,
                         p.orientation == PackOrientation::RowPacked ? 0 : 1, dm.as<float>(), nullptr));
    dm.get(m.data.data(), m.data.size() * 4);
    return m;
}

PackedBitMatrix im2col_sign_pack(const FloatTensor& x, std::size_t batch_index, const ConvGeometry& geom) {
    if (batch_index >= x.batch) throw ShapeError("im2col: batch index out of range");
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    PackedBitMatrix p = PackedBitMatrix::make(geom.patch_len(), oh * ow, PackOrientation::ColPacked);
    const std::size_t img = x.channels * x.height * x.width;
    Dev dx(img * 4), dw(p.byte_size());
    dx.put(x.data.data() + batch_index * img, img * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_im2col_sign_pack_f32(dx.as<float>(), 1, x.channels, x.height, x.width, &g, dw.as<std::uint32_t>(),
                                   p.words_per_line, nullptr));
    dw.get(p.words.data(), p.byte_size());
    return p;
}

FloatTensor reshape_output(const FloatMatrix& m, std::size_t out_h, std::size_t out_w) {
    if (m.cols != out_h * out_w)
        throw ShapeError("reshape_output: matrix has " + std::to_string(m.cols) + " columns, expected " +
                         std::to_string(out_h * out_w));
    FloatTensor t(1, m.rows, out_h, out_w);
    std::memcpy(t.data.data(), m.data.data(), m.data.size() * sizeof(float));
    return t;
}

FloatMatrix flatten_weights(const FloatTensor& w) {
    FloatMatrix m(w.batch, w.channels * w.height * w.width);
    std::memcpy(m.data.data(), w.data.data(), w.data.size() * sizeof(float));
    return m;
}

IntMatrix xnor_gemm(const PackedBitMatrix& w, const PackedBitMatrix& x, std::size_t inner_len, unsigned) {
    // kernels.cpp:55-68 checks, in the reference's order and words
    if (w.orientation != PackOrientation::RowPacked) throw ShapeError("xnor_gemm: weight operand must be row-packed");
    if (x.orientation != PackOrientation::ColPacked) throw ShapeError("xnor_gemm: input operand must be column-packed");
    if (w.logical_cols != inner_len || x.logical_rows != inner_len)
        throw ShapeError("xnor_gemm: inner extents " + std::to_string(w.logical_cols) + "/" +
                         std::to_string(x.logical_rows) + " do not match L=" + std::to_string(inner_len));
    if (w.words_per_line != x.words_per_line) throw ShapeError("xnor_gemm: words-per-line mismatch");
    IntMatrix out(w.logical_rows, x.logical_cols);
    check(bnn_host_xnor_gemm(w.words.data(), w.logical_rows, x.words.data(), x.logical_cols, inner_len,
                             out.data.data()));
    return out;
}

FloatMatrix to_float(const IntMatrix& m) {
    FloatMatrix out(m.rows, m.cols);
    Dev da(m.data.size() * 4), df(m.data.size() * 4);
    da.put(m.data.data(), m.data.size() * 4);
    check(bnn_to_float_s32(da.as<std::int32_t>(), m.data.size(), df.as<float>(), nullptr));
    df.get(out.data.data(), out.data.size() * 4);
    return out;
}

FloatMatrix bias_add(FloatMatrix a, std::span<const float> bias) {
    if (bias.size() != a.rows)
        throw ShapeError("bias_add: bias length " + std::to_string(bias.size()) + " does not match " +
                         std::to_string(a.rows) + " rows");
    Dev da(a.data.size() * 4), db(bias.size() * 4);
    da.put(a.data.data(), a.data.size() * 4);
    db.put(bias.data(), bias.size() * 4);
    check(bnn_bias_add_f32(da.as<float>(), a.rows, a.cols, db.as<float>(), nullptr));
    da.get(a.data.data(), a.data.size() * 4);
    return a;
}

FloatTensor conv_forward_binary(const FloatTensor& x, const PackedBitMatrix& packed_w, std::span<const float> bias,
                                const ConvGeometry& geom, unsigned) {
    if (packed_w.orientation != PackOrientation::RowPacked || packed_w.logical_rows != geom.out_channels ||
        packed_w.logical_cols != geom.patch_len())
        throw ShapeError("conv_forward_binary: packed weights must be row-packed [out_channels, patch_len]");
    if (bias.size() != geom.out_channels)
        throw ShapeError("bias_add: bias length " + std::to_string(bias.size()) + " does not match " +
                         std::to_string(geom.out_channels) + " rows");
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    FloatTensor out(x.batch, geom.out_channels, oh, ow);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_host_conv_forward_binary(x.data.data(), x.batch, x.channels, x.height, x.width, packed_w.words.data(),
                                       bias.data(), &g, out.data.data()));
    return out;
}

FloatMatrix linear_forward_packed(const FloatMatrix& x, const PackedBitMatrix& packed_w, std::span<const float> bias,
                                  unsigned) {
    if (packed_w.orientation != PackOrientation::RowPacked || packed_w.logical_cols != x.rows)
        throw ShapeError("xnor_gemm: inner extents " + std::to_string(packed_w.logical_cols) + "/" +
                         std::to_string(x.rows) + " do not match L=" + std::to_string(packed_w.logical_cols));
    if (bias.size() != packed_w.logical_rows)
        throw ShapeError("bias_add: bias length " + std::to_string(bias.size()) + " does not match " +
                         std::to_string(packed_w.logical_rows) + " rows");
    FloatMatrix out(packed_w.logical_rows, x.cols);
    check(bnn_host_linear_forward_packed(x.data.data(), x.rows, x.cols, packed_w.words.data(), packed_w.logical_rows,
                                         bias.data(), out.data.data()));
    return out;
}

FloatMatrix linear_forward(const FloatMatrix& x, const FloatMatrix& w, std::span<const float> bias,
                           KernelChoice kernel, unsigned threads) {  // network.cpp:113-120
    if (kernel == KernelChoice::Binary)
        return linear_forward_packed(x, pack_rows(sign(w)), bias, threads);  // packs per call
    return bias_add(float_gemm(w, x, threads), bias);
}

FloatTensor maxpool2(const FloatTensor& x) {
    if (x.height % 2 != 0 || x.width % 2 != 0)
        throw ShapeError("maxpool2: spatial extents must be even, got " + std::to_string(x.height) + "x" +
                         std::to_string(x.width));
    FloatTensor out(x.batch, x.channels, x.height / 2, x.width / 2);
    Dev dx(x.size() * 4), dy(out.size() * 4);
    dx.put(x.data.data(), x.size() * 4);
    check(bnn_maxpool2_f32(dx.as<float>(), x.batch, x.channels, x.height, x.width, dy.as<float>(), nullptr));
    dy.get(out.data.data(), out.size() * 4);
    return out;
}

namespace {
std::vector<float> affine(const std::vector<float>& x, std::size_t channels, std::size_t plane,
                          std::span<const float> scale, std::span<const float> shift) {
    std::vector<float> out(x.size());
    Dev dx(x.size() * 4), ds(channels * 4), dt(channels * 4);
    dx.put(x.data(), x.size() * 4);
    ds.put(scale.data(), channels * 4);
    dt.put(shift.data(), channels * 4);
    check(bnn_affine_f32(dx.as<float>(), x.size(), channels, plane, ds.as<float>(), dt.as<float>(), dx.as<float>(),
                         nullptr));
    dx.get(out.data(), out.size() * 4);
    return out;
}
}  // namespace

FloatTensor affine_norm(FloatTensor x, std::span<const float> scale, std::span<const float> shift) {
    if (scale.size() != x.channels || shift.size() != x.channels)
        throw ShapeError("affine_norm: parameter length does not match channels");
    x.data = affine(x.data, x.channels, x.height * x.width, scale, shift);
    return x;
}

FloatMatrix affine_norm(FloatMatrix x, std::span<const float> scale, std::span<const float> shift) {
    if (scale.size() != x.rows || shift.size() != x.rows)
        throw ShapeError("affine_norm: parameter length does not match features");
    x.data = affine(x.data, x.rows, x.cols, scale, shift);
    return x;
}

FloatMatrix flatten_to_columns(const FloatTensor& x) {
    const std::size_t features = x.channels * x.height * x.width;
    FloatMatrix m(features, x.batch);
    Dev dx(x.size() * 4), dm(x.size() * 4);
    dx.put(x.data.data(), x.size() * 4);
    check(bnn_flatten_to_columns_f32(dx.as<float>(), x.batch, features, dm.as<float>(), nullptr));
    dm.get(m.data.data(), m.data.size() * 4);
    return m;
}

NetworkSpec build_default_network(KernelChoice kernel, std::uint64_t seed) {
    bnn_layer_spec buf[64];
    const std::size_t n = bnn_default_spec(buf, 64);
    NetworkSpec spec;
    spec.name = "bnn-cifar10";
    spec.seed = seed;
    for (std::size_t i = 0; i < n; ++i) {
        LayerSpec l;
        l.kind = static_cast<LayerKind>(buf[i].kind);
        l.out_channels = buf[i].out_channels;
        l.kernel_h = buf[i].kernel_h, l.kernel_w = buf[i].kernel_w;
        l.stride_h = buf[i].stride_h, l.stride_w = buf[i].stride_w;
        l.pad_h = buf[i].pad_h, l.pad_w = buf[i].pad_w;
        l.out_features = buf[i].out_features;
        if (l.kind == LayerKind::Conv || l.kind == LayerKind::Linear) l.kernel = kernel;
        spec.layers.push_back(l);
    }
    return spec;
}

DeviceNetwork::DeviceNetwork(const NetworkSpec& spec) {
    std::vector<bnn_layer_spec> layers;
    for (const LayerSpec& l : spec.layers) {
        bnn_layer_spec c{};
        c.kernel = static_cast<std::uint32_t>(l.kernel);
        c.kind = static_cast<std::uint32_t>(l.kind);
        c.has_seed = l.seed.has_value() ? 1 : 0;
        c.seed = l.seed.value_or(0);
        c.out_channels = l.out_channels;
        c.kernel_h = l.kernel_h, c.kernel_w = l.kernel_w;
        c.stride_h = l.stride_h, c.stride_w = l.stride_w;
        c.pad_h = l.pad_h, c.pad_w = l.pad_w;
        c.out_features = l.out_features;
        c.weights_blob = l.weights_blob.empty() ? nullptr : l.weights_blob.c_str();
        layers.push_back(c);
    }
    in_chw_ = {spec.input_shape[1], spec.input_shape[2], spec.input_shape[3]};
    check(bnn_net_create(layers.data(), layers.size(), in_chw_[0], in_chw_[1], in_chw_[2], spec.seed,
                         spec.binarize_weights ? 1 : 0, &net_));
}

DeviceNetwork DeviceNetwork::from_spec_file(const std::string& path) {
    DeviceNetwork n;
    std::uint64_t shape[4];
    check(bnn_spec_info(path.c_str(), shape, nullptr));
    n.in_chw_ = {shape[1], shape[2], shape[3]};
    check(bnn_net_create_from_spec(path.c_str(), -1, &n.net_));
    return n;
}

DeviceNetwork::~DeviceNetwork() {
    if (net_) bnn_net_destroy(net_);
}

void save_packed_blob(const PackedBitMatrix& p, const std::string& path) {  // binarize.cpp:116-127
    check(bnn_save_packed_blob(path.c_str(), int(p.orientation), p.logical_rows, p.logical_cols, p.words.data()));
}

PackedBitMatrix load_packed_blob(const std::string& path) {  // binarize.cpp:129-148
    int o = 0;
    std::uint64_t r = 0, c = 0;
    check(bnn_load_packed_blob(path.c_str(), &o, &r, &c, nullptr, 0));
    PackedBitMatrix p = PackedBitMatrix::make(r, c, static_cast<PackOrientation>(o));
    check(bnn_load_packed_blob(path.c_str(), &o, &r, &c, p.words.data(), p.words.size()));
    return p;
}

void save_tensor_blob(const FloatTensor& t, const std::string& path) {  // tensor.cpp:123-134
    const std::uint64_t shape[4] = {t.batch, t.channels, t.height, t.width};
    check(bnn_save_tensor_blob(path.c_str(), shape, t.data.data()));
}

FloatTensor load_tensor_blob(const std::string& path) {  // tensor.cpp:136-150
    std::uint64_t shape[4];
    check(bnn_load_tensor_blob(path.c_str(), shape, nullptr, 0));
    FloatTensor t(shape[0], shape[1], shape[2], shape[3]);
    check(bnn_load_tensor_blob(path.c_str(), shape, t.data.data(), t.data.size()));
    return t;
}

std::size_t DeviceNetwork::logits() const { return bnn_net_logits(net_); }

FloatMatrix DeviceNetwork::forward(const FloatTensor& x) {
    if (x.channels != in_chw_[0] || x.height != in_chw_[1] || x.width != in_chw_[2])  // network.cpp:332-337
        throw ShapeError("network input is " + std::to_string(x.channels) + "x" + std::to_string(x.height) + "x" +
                         std::to_string(x.width) + ", network expects " + std::to_string(in_chw_[0]) + "x" +
                         std::to_string(in_chw_[1]) + "x" + std::to_string(in_chw_[2]));
    FloatMatrix out(logits(), x.batch);
    check(bnn_host_net_forward(net_, x.data.data(), x.batch, out.data.data()));
    return out;
}

FloatMatrix network_forward(DeviceNetwork& net, const FloatTensor& x) { return net.forward(x); }

}  // namespace bnn
