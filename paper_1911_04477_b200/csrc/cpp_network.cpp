// C++ reference-signature API, part 2: the float control group, the BinaryReference / naive
// layer forwards, float im2col / col2im, and the network entry points build_network +
// network_forward(const Network&, x, ForwardOptions) (include/bnn_b200.hpp, mirroring
// /root/reference/proj/include/bnn/{kernels,lowering,network}.hpp). Every arithmetic step runs on
// the device through the C ABI (bnn_cuda.h); host code only checks arguments (the reference's
// checks, order and messages), moves buffers and keeps the reference-shaped host mirror of the
// network's parameters.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>

#include "bnn_b200.hpp"
#include "bnn_cuda.h"
#include "cpp_internal.hpp"

namespace bnn {

using namespace cppi;

namespace {

void float_gemm_into(const float* dw, std::size_t M, std::size_t K, const float* dx, std::size_t N, const float* dbias,
                     std::size_t P, float* dout) {
    check(bnn_float_gemm_f32(dw, M, K, dx, N, dbias, P, dout, nullptr));
}

void check_bias(std::size_t len, std::size_t rows) {  // bias_add, kernels.cpp:97-101
    if (len != rows)
        throw ShapeError("bias_add: bias length " + std::to_string(len) + " does not match " + std::to_string(rows) +
                         " rows");
}

void check_gemm(std::size_t w_cols, std::size_t x_rows) {  // float_gemm, kernels.cpp:33-37
    if (w_cols != x_rows)
        throw ShapeError("float_gemm: inner extents differ, " + std::to_string(w_cols) + " vs " +
                         std::to_string(x_rows));
}

void check_im2col(const FloatTensor& x, const ConvGeometry& g) {  // lowering.cpp:8-10
    if (x.channels != g.in_channels)
        throw ShapeError("im2col: input has " + std::to_string(x.channels) + " channels, geometry expects " +
                         std::to_string(g.in_channels));
}

}  // namespace

// ----------------------------------------------------------------------- kernels.hpp / lowering.hpp

FloatMatrix float_gemm(const FloatMatrix& w, const FloatMatrix& x, unsigned) {  // kernels.cpp:33-51
    check_gemm(w.cols, x.rows);
    FloatMatrix out(w.rows, x.cols);
    Dev dw(w.data.size() * 4), dx(x.data.size() * 4), dy(out.data.size() * 4);
    dw.put(w.data.data(), w.data.size() * 4);
    dx.put(x.data.data(), x.data.size() * 4);
    float_gemm_into(dw.as<float>(), w.rows, w.cols, dx.as<float>(), x.cols, nullptr, 0, dy.as<float>());
    dy.get(out.data.data(), out.data.size() * 4);
    return out;
}

FloatMatrix im2col(const FloatTensor& x, std::size_t batch_index, const ConvGeometry& geom) {  // lowering.cpp:7-43
    check_im2col(x, geom);
    if (batch_index >= x.batch)
        throw ShapeError("im2col: batch index " + std::to_string(batch_index) + " out of range " +
                         std::to_string(x.batch));
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    FloatMatrix m(geom.patch_len(), oh * ow);
    const std::size_t img = x.channels * x.height * x.width;
    Dev dx(img * 4), dm(m.data.size() * 4);
    dx.put(x.data.data() + batch_index * img, img * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_im2col_f32(dx.as<float>(), 1, x.channels, x.height, x.width, 0, 1, &g, dm.as<float>(), nullptr));
    dm.get(m.data.data(), m.data.size() * 4);
    return m;
}

FloatTensor col2im(const FloatMatrix& m, const ConvGeometry& geom, std::size_t out_h, std::size_t out_w) {
    const bnn_conv_geom g = to_c(geom);
    std::size_t in_h = 0, in_w = 0;  // lowering.cpp:47-59 checks, extents only
    check(bnn_col2im_f32(nullptr, m.rows, m.cols, &g, out_h, out_w, nullptr, &in_h, &in_w, nullptr));
    FloatTensor x(1, geom.in_channels, in_h, in_w);
    Dev dm(m.data.size() * 4), dx(x.data.size() * 4);
    dm.put(m.data.data(), m.data.size() * 4);
    check(bnn_col2im_f32(dm.as<float>(), m.rows, m.cols, &g, out_h, out_w, dx.as<float>(), nullptr, nullptr, nullptr));
    dx.get(x.data.data(), x.data.size() * 4);
    return x;
}

FloatTensor naive_conv(const FloatTensor& x, std::size_t batch_index, const FloatTensor& w,
                       const ConvGeometry& geom) {  // kernels.cpp:109-147
    if (batch_index >= x.batch) throw ShapeError("naive_conv: batch index out of range");
    if (w.batch != geom.out_channels || w.channels != geom.in_channels || w.height != geom.kernel_h ||
        w.width != geom.kernel_w)
        throw ShapeError("naive_conv: weight shape does not match geometry");
    if (x.channels != geom.in_channels) throw ShapeError("naive_conv: input channels do not match geometry");
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    FloatTensor out(1, geom.out_channels, oh, ow);
    const std::size_t img = x.channels * x.height * x.width;
    Dev dx(img * 4), dw(w.data.size() * 4), dy(out.data.size() * 4);
    dx.put(x.data.data() + batch_index * img, img * 4);
    dw.put(w.data.data(), w.data.size() * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_conv_forward_naive_f32(dx.as<float>(), 1, x.channels, x.height, x.width, dw.as<float>(), nullptr, &g,
                                     dy.as<float>(), nullptr));
    dy.get(out.data.data(), out.data.size() * 4);
    return out;
}

// ------------------------------------------------------------------------------- network.hpp ops

FloatTensor conv_forward_float(const FloatTensor& x, const FloatMatrix& w_flat, std::span<const float> bias,
                               const ConvGeometry& geom, unsigned) {  // network.cpp:50-63
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    check_im2col(x, geom);
    check_gemm(w_flat.cols, geom.patch_len());
    check_bias(bias.size(), w_flat.rows);
    FloatTensor out(x.batch, geom.out_channels, oh, ow);
    Dev dx(x.size() * 4), dw(w_flat.data.size() * 4), db(bias.size() * 4), dy(out.size() * 4);
    dx.put(x.data.data(), x.size() * 4);
    dw.put(w_flat.data.data(), w_flat.data.size() * 4);
    db.put(bias.data(), bias.size() * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_conv_forward_float_f32(dx.as<float>(), x.batch, x.channels, x.height, x.width, dw.as<float>(),
                                     db.as<float>(), &g, dy.as<float>(), nullptr));
    dy.get(out.data.data(), out.size() * 4);
    return out;
}

FloatTensor conv_forward_binary_reference(const FloatTensor& x, const FloatMatrix& w_pm1, std::span<const float> bias,
                                          const ConvGeometry& geom, unsigned) {  // network.cpp:81-94
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    check_im2col(x, geom);
    check_gemm(w_pm1.cols, geom.patch_len());
    check_bias(bias.size(), w_pm1.rows);
    FloatTensor out(x.batch, geom.out_channels, oh, ow);
    const std::size_t K = geom.patch_len(), N = x.batch * oh * ow;
    Dev dx(x.size() * 4), dcol(K * N * 4), dw(w_pm1.data.size() * 4), db(bias.size() * 4), dy(out.size() * 4);
    dx.put(x.data.data(), x.size() * 4);
    dw.put(w_pm1.data.data(), w_pm1.data.size() * 4);
    db.put(bias.data(), bias.size() * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_im2col_f32(dx.as<float>(), x.batch, x.channels, x.height, x.width, 0, x.batch, &g, dcol.as<float>(),
                         nullptr));
    check(bnn_sign_f32(dcol.as<float>(), K * N, dcol.as<float>(), nullptr));  // sign(im2col(x, b))
    float_gemm_into(dw.as<float>(), w_pm1.rows, K, dcol.as<float>(), N, db.as<float>(), oh * ow, dy.as<float>());
    dy.get(out.data.data(), out.size() * 4);
    return out;
}

FloatTensor conv_forward_naive(const FloatTensor& x, const FloatTensor& w, std::span<const float> bias,
                               const ConvGeometry& geom) {  // network.cpp:96-111
    const auto [oh, ow] = output_dims(geom, x.height, x.width);
    if (bias.size() != geom.out_channels) throw ShapeError("conv: bias length does not match output channels");
    if (w.batch != geom.out_channels || w.channels != geom.in_channels || w.height != geom.kernel_h ||
        w.width != geom.kernel_w)
        throw ShapeError("naive_conv: weight shape does not match geometry");
    if (x.channels != geom.in_channels) throw ShapeError("naive_conv: input channels do not match geometry");
    FloatTensor out(x.batch, geom.out_channels, oh, ow);
    Dev dx(x.size() * 4), dw(w.data.size() * 4), db(bias.size() * 4), dy(out.size() * 4);
    dx.put(x.data.data(), x.size() * 4);
    dw.put(w.data.data(), w.data.size() * 4);
    db.put(bias.data(), bias.size() * 4);
    const bnn_conv_geom g = to_c(geom);
    check(bnn_conv_forward_naive_f32(dx.as<float>(), x.batch, x.channels, x.height, x.width, dw.as<float>(),
                                     db.as<float>(), &g, dy.as<float>(), nullptr));
    dy.get(out.data.data(), out.size() * 4);
    return out;
}

FloatMatrix linear_forward_binary_reference(const FloatMatrix& x, const FloatMatrix& w_pm1, std::span<const float> bias,
                                            unsigned) {  // network.cpp:128-131
    check_gemm(w_pm1.cols, x.rows);
    check_bias(bias.size(), w_pm1.rows);
    FloatMatrix out(w_pm1.rows, x.cols);
    Dev dx(x.data.size() * 4), dw(w_pm1.data.size() * 4), db(bias.size() * 4), dy(out.data.size() * 4);
    dx.put(x.data.data(), x.data.size() * 4);
    dw.put(w_pm1.data.data(), w_pm1.data.size() * 4);
    db.put(bias.data(), bias.size() * 4);
    check(bnn_sign_f32(dx.as<float>(), x.data.size(), dx.as<float>(), nullptr));  // sign(x)
    float_gemm_into(dw.as<float>(), w_pm1.rows, w_pm1.cols, dx.as<float>(), x.cols, db.as<float>(), 0, dy.as<float>());
    dy.get(out.data.data(), out.data.size() * 4);
    return out;
}

// ----------------------------------------------------------------------------------- the network

namespace detail {

// The device network plus what its parameters were last synchronised from, so network_forward
// notices a caller's edits of net.layers (the reference reads them on every forward).
struct DeviceEngine {
    bnn_net* net = nullptr;
    std::mutex mu;  // one forward at a time per engine (the arena is shared)
    int policy = -1;
    struct Snap {
        std::vector<std::uint32_t> packed;
        std::vector<float> bias, scale, shift;
        std::uint64_t weights_hash = 0;
        KernelChoice kernel = KernelChoice::Float;
    };
    std::vector<Snap> snap;
    ~DeviceEngine() {
        if (net) bnn_net_destroy(net);
    }
};

}  // namespace detail

namespace {

// 64-bit multiply-xorshift hash over the float weights (detects edits of BuiltLayer::weights
// without keeping a second copy of them).
std::uint64_t words_hash(const std::vector<float>& v) {
    std::uint64_t h = 0x9E3779B97F4A7C15ull ^ v.size();
    const auto* p = reinterpret_cast<const unsigned char*>(v.data());
    const std::size_t n = v.size() * sizeof(float);
    std::size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        std::uint64_t w;
        std::memcpy(&w, p + i, 8);
        h = (h ^ w) * 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
    }
    for (; i < n; ++i) h = (h ^ p[i]) * 0x94D049BB133111EBull;
    return h;
}

bnn_layer_spec to_c_layer(const LayerSpec& l) {
    bnn_layer_spec c{};
    c.kind = static_cast<std::uint32_t>(l.kind);
    c.has_seed = l.seed.has_value() ? 1 : 0;
    c.seed = l.seed.value_or(0);
    c.out_channels = l.out_channels;
    c.kernel_h = l.kernel_h, c.kernel_w = l.kernel_w;
    c.stride_h = l.stride_h, c.stride_w = l.stride_w;
    c.pad_h = l.pad_h, c.pad_w = l.pad_w;
    c.out_features = l.out_features;
    c.weights_blob = l.weights_blob.empty() ? nullptr : l.weights_blob.c_str();
    c.kernel = static_cast<std::uint32_t>(l.kernel);
    return c;
}

void take_snapshot(detail::DeviceEngine& e, const Network& net) {
    e.snap.assign(net.layers.size(), {});
    for (std::size_t i = 0; i < net.layers.size(); ++i) {
        const BuiltLayer& L = net.layers[i];
        auto& s = e.snap[i];
        s.packed = L.packed_weights.words, s.bias = L.bias, s.scale = L.scale, s.shift = L.shift;
        s.weights_hash = L.has_weights() ? words_hash(L.weights.data) : 0;
        s.kernel = L.spec.kernel;
    }
}

// Re-upload the parameters the caller changed since the last forward (the ones the requested
// graph reads: packed bits for Binary, float weights for Float / BinaryReference / Naive).
void sync(detail::DeviceEngine& e, const Network& net, bool float_weights) {
    if (net.layers.size() != e.snap.size())
        throw ShapeError("network_forward: layer count changed since build_network");
    for (std::size_t i = 0; i < net.layers.size(); ++i) {
        const BuiltLayer& L = net.layers[i];
        auto& s = e.snap[i];
        const std::uint32_t* packed = nullptr;
        const float *weights = nullptr, *bias = nullptr, *scale = nullptr, *shift = nullptr;
        if (L.has_weights()) {
            if (L.packed_weights.words != s.packed) {
                if (L.packed_weights.words.size() != s.packed.size())
                    throw ShapeError("layer " + std::to_string(i) + ": packed weights resized");
                packed = L.packed_weights.words.data();
            }
            if (L.bias != s.bias) {
                if (L.bias.size() != s.bias.size()) throw ShapeError("layer " + std::to_string(i) + ": bias resized");
                bias = L.bias.data();
            }
            if (float_weights) {
                const std::uint64_t h = words_hash(L.weights.data);
                if (h != s.weights_hash) {
                    if (L.weights.rows * L.weights.cols != L.weights.data.size() ||
                        L.weights.data.size() != L.packed_weights.logical_rows * L.packed_weights.logical_cols)
                        throw ShapeError("layer " + std::to_string(i) + ": weights resized");
                    weights = L.weights.data.data();
                    s.weights_hash = h;
                }
            }
            if (L.spec.kernel != s.kernel) {
                check(bnn_net_set_layer_kernel(e.net, i, static_cast<int>(L.spec.kernel)));
                s.kernel = L.spec.kernel;
            }
        }
        if (L.spec.kind == LayerKind::AffineNorm) {
            if (L.scale != s.scale) {
                if (L.scale.size() != s.scale.size()) throw ShapeError("layer " + std::to_string(i) + ": scale resized");
                scale = L.scale.data();
            }
            if (L.shift != s.shift) {
                if (L.shift.size() != s.shift.size()) throw ShapeError("layer " + std::to_string(i) + ": shift resized");
                shift = L.shift.data();
            }
        }
        if (packed || weights || bias || scale || shift) {
            check(bnn_net_set_layer_data(e.net, i, packed, weights, bias, scale, shift));
            if (packed) s.packed = L.packed_weights.words;
            if (bias) s.bias = L.bias;
            if (scale) s.scale = L.scale;
            if (shift) s.shift = L.shift;
        }
    }
}

int engine_for(ExecKernel k) {
    switch (k) {
        case ExecKernel::PerLayer: return BNN_ENGINE_PER_LAYER;
        case ExecKernel::Float: return BNN_ENGINE_FLOAT;
        case ExecKernel::Binary: return BNN_ENGINE_AUTO;
        case ExecKernel::Naive: return BNN_ENGINE_NAIVE;
        case ExecKernel::BinaryReference: return BNN_ENGINE_BINARY_REFERENCE;
    }
    return BNN_ENGINE_AUTO;
}

}  // namespace

Network build_network(const NetworkSpec& spec) {  // network.cpp:203-306
    Network net;
    net.spec = spec;
    net.in_channels = spec.input_shape[1];
    net.in_h = spec.input_shape[2];
    net.in_w = spec.input_shape[3];
    if (spec.layers.empty()) throw ShapeError("network has no layers");
    std::vector<bnn_layer_spec> cl;
    for (const LayerSpec& l : spec.layers) cl.push_back(to_c_layer(l));
    auto eng = std::make_shared<detail::DeviceEngine>();
    check(bnn_net_create(cl.data(), cl.size(), net.in_channels, net.in_h, net.in_w, spec.seed,
                         spec.binarize_weights ? 1 : 0, &eng->net));
    // the host mirror of the device parameters (BuiltLayer, network.hpp:57-77)
    std::size_t ch = net.in_channels;
    for (std::size_t i = 0; i < spec.layers.size(); ++i) {
        BuiltLayer L;
        L.spec = spec.layers[i];
        std::size_t sh[8];
        check(bnn_net_layer_shape(eng->net, i, sh));
        const std::size_t rows = sh[1], cols = sh[2];
        if (L.spec.kind == LayerKind::Conv)
            L.geom = ConvGeometry{L.spec.kernel_h, L.spec.kernel_w, L.spec.stride_h, L.spec.stride_w,
                                  L.spec.pad_h,    L.spec.pad_w,    ch,               L.spec.out_channels};
        if (L.spec.kind == LayerKind::Linear) L.in_features = cols, L.out_features = rows;
        if (L.has_weights()) {
            L.weights = FloatMatrix(rows, cols);
            L.packed_weights = PackedBitMatrix::make(rows, cols, PackOrientation::RowPacked);
            L.bias.assign(rows, 0.0f);
            check(bnn_net_layer_data(eng->net, i, L.packed_weights.words.data(), L.weights.data.data(), L.bias.data(),
                                     nullptr, nullptr));
            if (L.spec.kind == LayerKind::Conv) {
                L.weight_tensor = FloatTensor(rows, ch, L.spec.kernel_h, L.spec.kernel_w);
                L.weight_tensor.data = L.weights.data;  // flatten_weights is the identity on memory
            }
            net.parameter_count += L.weights.data.size() + L.bias.size();
        }
        if (L.spec.kind == LayerKind::AffineNorm) {
            L.scale.assign(ch, 0.0f);
            L.shift.assign(ch, 0.0f);
            check(bnn_net_layer_data(eng->net, i, nullptr, nullptr, nullptr, L.scale.data(), L.shift.data()));
            net.parameter_count += 2 * ch;
        }
        L.out_channels = sh[4], L.out_h = sh[5], L.out_w = sh[6], L.out_flat = sh[7] != 0;
        ch = L.out_channels;
        net.layers.push_back(std::move(L));
    }
    net.logits = bnn_net_logits(eng->net);
    take_snapshot(*eng, net);
    net.device = std::move(eng);
    return net;
}

FloatMatrix network_forward(const Network& net, const FloatTensor& x, const ForwardOptions& opts) {
    if (x.channels != net.in_channels || x.height != net.in_h || x.width != net.in_w)  // network.cpp:332-337
        throw ShapeError("network input is " + std::to_string(x.channels) + "x" + std::to_string(x.height) + "x" +
                         std::to_string(x.width) + ", network expects " + std::to_string(net.in_channels) + "x" +
                         std::to_string(net.in_h) + "x" + std::to_string(net.in_w));
    if (opts.layer_seconds && opts.layer_seconds->size() != net.layers.size())
        opts.layer_seconds->assign(net.layers.size(), 0.0);
    if (!net.device) throw ConfigError("network_forward: the network was not made by build_network");
    detail::DeviceEngine& e = *net.device;
    std::lock_guard<std::mutex> lock(e.mu);
    const int policy = engine_for(opts.kernel);
    bool float_weights = policy != BNN_ENGINE_AUTO;
    if (policy == BNN_ENGINE_PER_LAYER) {
        float_weights = false;
        for (const BuiltLayer& L : net.layers) float_weights |= L.has_weights() && L.spec.kernel != KernelChoice::Binary;
    }
    sync(e, net, float_weights);
    if (policy != e.policy) {
        check(bnn_net_set_engine(e.net, policy));
        e.policy = policy;
    }
    if (opts.layer_seconds) {
        check(bnn_net_set_timing(e.net, 1));
        check(bnn_net_reset_timing(e.net));
    }
    FloatMatrix out(net.logits, x.batch);
    const int rc = bnn_host_net_forward(e.net, x.data.data(), x.batch, out.data.data());
    if (opts.layer_seconds) {
        std::vector<double> ms(net.layers.size(), 0.0);
        const int rt = bnn_net_timing(e.net, ms.data(), nullptr, nullptr);
        bnn_net_set_timing(e.net, 0);
        check(rc);
        check(rt);
        for (std::size_t i = 0; i < ms.size(); ++i) (*opts.layer_seconds)[i] += ms[i] * 1e-3;
    }
    check(rc);
    return out;
}

}  // namespace bnn
