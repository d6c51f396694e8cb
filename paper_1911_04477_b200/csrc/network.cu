// Device network engine: build_network + network_forward for ExecKernel::Binary
// (network.cpp:203-420) on one GPU and one stream.
//
// Build: parameters are generated ON THE DEVICE with the reference's counter-based
// generator (bit-identical to fill_random, tensor.cpp:65-96) from the reference seeds
// (base = layer seed or mix64(net seed, i); weights mix64(base,1), bias mix64(base,2),
// affine scale mix64(base,3) -> 1 + 0.5u, shift mix64(base,4); network.cpp:217-290) and
// packed once with K1 (pack_rows(sign(W)), network.cpp:247,271). Nothing is packed inside
// a forward.
//
// Forward (general topology): conv = K2 binary im2col + K3 GEMM with the fused
// to_float+bias+reshape epilogue; linear = flatten_to_columns (when coming from a tensor)
// + K1 pack_cols(sign) + K3; maxpool / affine / htanh / sign = K4. Activations ping-pong
// between two arena buffers sized for the largest layer at the requested batch.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "bnn_common.cuh"
#include <cstring>

#include "fused.cuh"

namespace bnnk {

int launch_pack_cols(const float*, size_t, size_t, uint32_t*, size_t, unsigned long long*,
                     cudaStream_t);
int launch_pack_rows_e2m1(const float* x, size_t D, size_t L, void* out4, cudaStream_t s);
int launch_pack_rows(const float*, size_t, size_t, uint32_t*, size_t, unsigned long long*,
                     cudaStream_t);
int launch_im2col_sign_pack(const float*, size_t, size_t, size_t, size_t, const bnn_conv_geom*,
                            uint32_t*, size_t, cudaStream_t);
int gemm_f32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t, const float*,
             size_t, float*, cudaStream_t);
int launch_maxpool2(const float*, size_t, size_t, size_t, size_t, float*, cudaStream_t);
int launch_affine(const float*, size_t, size_t, size_t, const float*, const float*, float*,
                  cudaStream_t);
int launch_transpose(const float*, size_t, size_t, float*, cudaStream_t);
int launch_fill_random(uint64_t, uint64_t, size_t, float*, cudaStream_t);
int launch_affine_scale(float*, size_t, cudaStream_t);
int launch_unary(int, const float*, size_t, float*, cudaStream_t);
int make_tmap_2d_s8(CUtensorMap* map, const void* base, size_t rows, size_t K, size_t ld, uint32_t box_rows);
int launch_float_gemm(const float*, const float*, size_t, size_t, size_t, const float*, size_t, float*, cudaStream_t);
int launch_im2col_f32(const float*, size_t, size_t, size_t, size_t, const bnn_conv_geom*, float*, cudaStream_t);
int launch_naive_conv(const float*, size_t, size_t, size_t, size_t, const float*, const float*, const bnn_conv_geom*,
                      float*, cudaStream_t);

namespace {

const char* kind_name(uint32_t k) {
    static const char* names[] = {"conv", "linear", "maxpool", "affine_norm", "sign", "htanh"};
    return k < 6 ? names[k] : "?";
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t b) {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, b ? b : 16);
        if (e != cudaSuccess)
            return fail(BNN_E_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        bytes = b;
        return BNN_OK;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct Layer {
    bnn_layer_spec spec{};
    bnn_conv_geom geom{};
    size_t rows = 0, cols = 0, wpl = 0;  // packed weights: rows lines x wpl words, L = cols
    DevBuf wf;                           // float weights [rows, cols] (the float control group)
    DevBuf packed, bias, scale, shift;
    DevBuf wpm1;                         // sign(wf), made on first use by the BinaryReference graph
    size_t n_affine = 0;
    size_t in_c = 0, in_h = 0, in_w = 0;  // input shape (per image)
    bool in_flat = false;
    size_t out_c = 0, out_h = 0, out_w = 0;
    bool out_flat = false;
};

// One fused launch (fused.cu): a weighted layer plus the glue that follows it.
struct FusedStage {
    size_t layer = 0, last = 0;  // weighted layer index, last layer folded into it
    int in_mode = FIN_BITS, epi = FEPI_BITS;
    FusedGeom g{};               // batch-independent fields
    int Dpad = 0, Kpad = 0;
    bool pre_encode = false;     // first layer is linear: K1 sign-packs each image's features first
    bool small_logits = false;   // tiny final layer: CUDA-core popcount kernel (wbits)
    bool pix_popc = false;       // pixel-input first conv with K <= 32: CUDA-core kernel
    bool halo0 = false;          // pixel-input first conv through halo4 (float input, C padded to 64)
    DevBuf w4h;                  // its e2m1 weights [Dpad, K'/2], K' = KH*KW*64
    CUtensorMap tm4h;
    PixParams pix{};             // its per-channel weight words, thresholds and flips
    const char* kname = "";      // kernel the last forward ran for this stage
    DevBuf w8, prm, wbits;
    DevBuf w4;                   // FP4 (e2m1) weights [Dpad, Kpad4 / 2] for the mxf4 swapped kernel
    CUtensorMap tm4;             // its weight map (box 128 rows x 128 bytes)
    bool fp4_ok = false;              // int8 +-1 weights [Dpad, Kpad] (engine K order), float4 params
    CUtensorMap tm[5];           // weight tile maps, box rows 16, 32, 64, 128, 256 (= BN / cta_group)
    size_t out_words_per_image = 0;
};

}  // namespace bnnk

struct bnn_net {
    std::vector<std::unique_ptr<bnnk::Layer>> layers;
    size_t in_c = 0, in_h = 0, in_w = 0, logits = 0;
    bool binarize = false;          // NetworkSpec::binarize_weights
    size_t max_act_per_image = 0;   // floats
    size_t max_lines_words_per_image = 0;
    // activation arena
    size_t arena_batch = 0;
    bnnk::DevBuf act[2], lines;
    size_t last_launches = 0;
    size_t weight_bytes = 0;
    // per-layer CUDA-event timing (the device analogue of ForwardOptions::layer_seconds,
    // network.hpp:93-97): events are recorded on the forward stream and resolved lazily.
    bool timing = false;
    struct Pending { size_t layer; int what; cudaEvent_t a, b; };  // what: 0 layer, 1 gemm
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> pool;
    std::vector<double> layer_ms, gemm_ms;
    std::vector<size_t> gemm_launches;
    // fused engine (fused.cu): one launch per weighted layer, packed-bit activations
    int engine_policy = 0;  // BNN_ENGINE_*
    bool fusable = false;
    std::string unfusable_why;
    std::vector<std::unique_ptr<bnnk::FusedStage>> stages;
    bool use_graphs = true;
    struct Graph {
        bool key_set = false;
        const float* x = nullptr;
        size_t B = 0;
        float* logits = nullptr;
        cudaStream_t s = nullptr;
        cudaGraphExec_t exec = nullptr;
        size_t launches = 0;
        int epoch = 0, arena = 0;
    };
    std::array<Graph, 8> graphs;  // >= the serving pipe's maximum depth: each buffer set keeps its graph
    size_t graph_next = 0;
    int arena_epoch = 0;  // bumped whenever an internal buffer is reallocated (graphs hold pointers)
    void drop_graphs() {
        for (auto& e : graphs)
            if (e.exec) cudaGraphExecDestroy(e.exec);
        graphs = {};
    }
    size_t bits_words_per_image = 0;
    size_t bits_batch = 0;
    bnnk::DevBuf bits[2], pix, ws, sem;
    bnnk::DevBuf lin_ws;   // split-K partial sums of the FP4 linear kernel (lin4)
    bnnk::DevBuf lin_sem;  // its per-tile counters (zeroed once; the kernel leaves them at 0)
    bnnk::DevBuf lin_x4[2];  // e2m1 images of TMA-fed lin4 stages (ping-pong: a lin4 stage writes the next one's)
    bnnk::DevBuf fcols;  // float im2col matrix (control-group engine)
};

namespace bnnk {
namespace {

int fill(float* dst, size_t n, uint64_t seed, cudaStream_t s) {
    return launch_fill_random(seed, 0, n, dst, s);
}

int build(bnn_net* net, const bnn_layer_spec* specs, size_t n, uint64_t seed, cudaStream_t s) {
    size_t ch = net->in_c, hh = net->in_h, ww = net->in_w;
    bool flat = false;
    net->max_act_per_image = ch * hh * ww;
    DevBuf tmp;
    for (size_t i = 0; i < n; ++i) {
        auto L = std::make_unique<Layer>();
        L->spec = specs[i];
        L->in_c = ch, L->in_h = hh, L->in_w = ww, L->in_flat = flat;
        const uint64_t base = specs[i].has_seed ? specs[i].seed : mix64(seed, i);
        auto chain_error = [&](const std::string& msg) {  // network.cpp:190-193
            return fail(BNN_E_SHAPE, "layer " + std::to_string(i) + " (" + kind_name(specs[i].kind) +
                                         "): " + msg);
        };
        switch (specs[i].kind) {
            case BNN_LAYER_CONV: {
                if (flat) return chain_error("input is already flattened");
                const bnn_layer_spec& ls = specs[i];
                if (ls.out_channels == 0 || ls.kernel_h == 0 || ls.kernel_w == 0)
                    return chain_error("out_channels and kernel size are required");
                L->geom = bnn_conv_geom{ls.kernel_h, ls.kernel_w, ls.stride_h, ls.stride_w,
                                        ls.pad_h,    ls.pad_w,    ch,          ls.out_channels};
                size_t oh, ow;
                if (bnn_output_dims(&L->geom, hh, ww, &oh, &ow) != BNN_OK)
                    return chain_error(bnn_last_error());
                L->rows = ls.out_channels;
                L->cols = ch * ls.kernel_h * ls.kernel_w;
                net->max_lines_words_per_image =
                    std::max(net->max_lines_words_per_image, oh * ow * wpl_of(L->cols));
                ch = ls.out_channels, hh = oh, ww = ow;
                break;
            }
            case BNN_LAYER_LINEAR: {
                if (specs[i].out_features == 0) return chain_error("out_features is required");
                L->rows = specs[i].out_features;
                L->cols = flat ? ch : ch * hh * ww;
                net->max_lines_words_per_image =
                    std::max(net->max_lines_words_per_image, wpl_of(L->cols));
                ch = specs[i].out_features, hh = ww = 0;
                flat = true;
                break;
            }
            case BNN_LAYER_MAXPOOL:
                if (flat) return chain_error("input is already flattened");
                if (hh % 2 || ww % 2)
                    return chain_error("spatial extents must be even, got " + std::to_string(hh) +
                                       "x" + std::to_string(ww));
                hh /= 2, ww /= 2;
                break;
            case BNN_LAYER_AFFINE: {
                L->n_affine = ch;  // channel count, or feature count once flat
                BNN_TRY(L->scale.alloc(ch * 4));
                BNN_TRY(L->shift.alloc(ch * 4));
                BNN_TRY(fill(L->scale.as<float>(), ch, mix64(base, 3), s));
                BNN_TRY(launch_affine_scale(L->scale.as<float>(), ch, s));
                BNN_TRY(fill(L->shift.as<float>(), ch, mix64(base, 4), s));
                net->weight_bytes += 8 * ch;
                break;
            }
            case BNN_LAYER_SIGN:
            case BNN_LAYER_HTANH:
                break;
            default:
                return fail(BNN_E_CONFIG, "unknown layer kind " + std::to_string(specs[i].kind));
        }
        if (L->rows) {  // weighted layer: generate (or load), binarize, pack once
            L->wpl = wpl_of(L->cols);
            const size_t nw = L->rows * L->cols;
            if (tmp.bytes < nw * 4) BNN_TRY(tmp.alloc(nw * 4));
            if (specs[i].weights_blob) {  // network.cpp:233-241 / 258-266
                uint64_t shp[4];
                BNN_TRY(bnn_load_tensor_blob(specs[i].weights_blob, shp, nullptr, 0));
                const bool conv = specs[i].kind == BNN_LAYER_CONV;
                const bool ok = conv ? (shp[0] == L->rows && shp[1] == L->in_c && shp[2] == specs[i].kernel_h &&
                                        shp[3] == specs[i].kernel_w)
                                     : (shp[0] == L->rows && shp[1] == L->cols && shp[2] == 1 && shp[3] == 1);
                if (!ok)
                    return chain_error(conv ? "weights blob shape does not match [D, C, kH, kW]"
                                            : "weights blob shape does not match [out, in, 1, 1]");
                std::vector<float> hw(nw);
                BNN_TRY(bnn_load_tensor_blob(specs[i].weights_blob, shp, hw.data(), nw));
                // flatten_weights is the identity on [D, C, kH, kW] memory (lowering.cpp:97-102)
                BNN_CUDA(cudaMemcpyAsync(tmp.p, hw.data(), nw * 4, cudaMemcpyHostToDevice, s));
                BNN_CUDA(cudaStreamSynchronize(s));  // hw is released on scope exit
            } else {
                BNN_TRY(fill(tmp.as<float>(), nw, mix64(base, 1), s));
            }
            // network.cpp:245,268: binarize_weights applies sign to the generated (or loaded) weights
            if (net->binarize) BNN_TRY(launch_unary(0, tmp.as<float>(), nw, tmp.as<float>(), s));
            BNN_TRY(L->wf.alloc(nw * 4));  // network.cpp:246,269: layer.weights, kept for ExecKernel::Float
            BNN_CUDA(cudaMemcpyAsync(L->wf.p, tmp.p, nw * 4, cudaMemcpyDeviceToDevice, s));
            BNN_TRY(L->packed.alloc(L->rows * L->wpl * 4));
            BNN_TRY(launch_pack_rows(tmp.as<float>(), L->rows, L->cols, L->packed.as<uint32_t>(),
                                     L->wpl, nullptr, s));
            BNN_TRY(L->bias.alloc(L->rows * 4));
            BNN_TRY(fill(L->bias.as<float>(), L->rows, mix64(base, 2), s));
            net->weight_bytes += L->rows * L->wpl * 4 + L->rows * 4;
            // tmp is reused by the next layer: order the reuse on the stream
        }
        L->out_c = ch, L->out_h = hh, L->out_w = ww, L->out_flat = flat;
        net->max_act_per_image = std::max(net->max_act_per_image, flat ? ch : ch * hh * ww);
        net->layers.push_back(std::move(L));
    }
    net->logits = flat ? ch : ch * hh * ww;
    BNN_CUDA(cudaStreamSynchronize(s));  // tmp is freed on return
    return BNN_OK;
}

size_t round_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

// Recognise the fusable pattern (network.cpp:330-420 semantics preserved exactly, see fused.cu):
//   conv (float input) -> { [maxpool] [affine_norm] [htanh] [sign] -> conv|linear }* -> linear (logits)
// Every weighted layer after the first reads packed bits; every glue run ends in a weighted layer
// (whose pack_cols(sign(.)) makes a trailing htanh/sign redundant). Anything else -> generic engine.
int plan_fused(bnn_net* net, cudaStream_t s) {
    auto& Ls = net->layers;
    const size_t n = Ls.size();
    auto no = [&](const std::string& why) {
        net->fusable = false;
        net->unfusable_why = why;
        net->stages.clear();
        return BNN_OK;
    };
    net->stages.clear();
    net->fusable = false;
    size_t i = 0;
    size_t max_words = 0;
    DevBuf bad;
    BNN_TRY(bad.alloc(sizeof(int)));
    BNN_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    while (i < n) {
        Layer& L = *Ls[i];
        const uint32_t kind = L.spec.kind;
        if (kind != BNN_LAYER_CONV && kind != BNN_LAYER_LINEAR)
            return no("layer " + std::to_string(i) + " is glue without a preceding weighted layer");
        const bool first = i == 0;
        auto st = std::make_unique<FusedStage>();
        st->layer = i;
        st->in_mode = FIN_BITS;
        FusedGeom& g = st->g;
        int T = 1, Cperm = 1;
        if (kind == BNN_LAYER_CONV) {
            g.C = int(L.in_c), g.H = int(L.in_h), g.W = int(L.in_w);
            g.KH = int(L.geom.kernel_h), g.KW = int(L.geom.kernel_w);
            g.SH = int(L.geom.stride_h), g.SW = int(L.geom.stride_w);
            g.PH = int(L.geom.pad_h), g.PW = int(L.geom.pad_w);
            g.OH = int(L.out_h), g.OW = int(L.out_w);
            T = g.KH * g.KW, Cperm = int(L.in_c);
            if (first) {
                st->in_mode = (g.C <= 32 && T <= 16 && T * g.C <= 64) ? FIN_PIX : FIN_F32;
                if (st->in_mode == FIN_F32) T = 1, Cperm = 1;  // reference im2col order
            } else if (L.in_c % 32) {
                return no("conv input channels not a multiple of 32");
            }
        } else {
            g.C = int(L.cols), g.H = g.W = 1, g.KH = g.KW = g.SH = g.SW = 1, g.PH = g.PW = 0;
            g.OH = g.OW = 1;
            if (first) {
                // float input: flatten_to_columns order (network.cpp:177-184) is each image's
                // memory order, so K1 pack_rows over [B, F] yields the stage's input bits in the
                // reference K order (T = 1, no weight permutation); pad bits are 0 on both sides
                st->pre_encode = true;
            } else {
                if (L.cols % 32) return no("linear input features not a multiple of 32");
                if (!L.in_flat) T = int(L.in_h * L.in_w), Cperm = int(L.in_c);  // NHWC flatten order
            }
        }
        g.Cw = int((size_t(g.C) + 31) / 32);
        g.K = int(L.cols);
        g.D = int(L.rows);
        size_t j = i + 1;
        bool pool = false;
        Layer* aff = nullptr;
        if (j < n && Ls[j]->spec.kind == BNN_LAYER_MAXPOOL) {
            if (kind != BNN_LAYER_CONV) return no("maxpool after a linear layer");
            pool = true, ++j;
        }
        if (j < n && Ls[j]->spec.kind == BNN_LAYER_AFFINE) aff = Ls[j].get(), ++j;
        if (j < n && Ls[j]->spec.kind == BNN_LAYER_HTANH) ++j;
        if (j < n && Ls[j]->spec.kind == BNN_LAYER_SIGN) ++j;
        if (j == n) {
            if (j != i + 1 || kind != BNN_LAYER_LINEAR)
                return no("the network does not end in a bare linear layer");
            st->epi = FEPI_LOGITS;
        } else {
            const uint32_t nk = Ls[j]->spec.kind;
            if (nk != BNN_LAYER_CONV && nk != BNN_LAYER_LINEAR)
                return no("unsupported glue sequence after layer " + std::to_string(i));
            if (L.rows % 32) return no("output channels not a multiple of 32");
            st->epi = FEPI_BITS;
            if (round_up(L.rows, 256) > 4096) return no("more than 4096 output channels");
        }
        g.pool = pool ? 1 : 0;
        g.Dw = g.D / 32;
        st->last = j - 1;
        st->Kpad = int(round_up(size_t(g.K), 128));
        st->Dpad = int(round_up(size_t(g.D), 32));
        g.KB = st->Kpad / 128;
        g.kq_last = (g.K - 128 * (g.KB - 1) + 31) / 32;
        g.dv0 = FastDiv::make(uint32_t(pool ? g.OW / 2 : g.OH * g.OW));
        g.dv1 = FastDiv::make(uint32_t(pool ? g.OH / 2 : g.OW));
        if (st->in_mode == FIN_F32 && g.K > 1024) return no("first conv reduction length > 1024");
        if (st->in_mode == FIN_BITS && st->Kpad / 32 > 1024) return no("reduction length > 32768");
        const size_t prm_n = round_up(size_t(g.D), 256);
        BNN_TRY(st->w8.alloc(size_t(st->Dpad) * st->Kpad));
        BNN_TRY(st->prm.alloc(prm_n * sizeof(int4)));
        BNN_TRY(fused_prep_weights(L.packed.as<uint32_t>(), L.wpl, g.D, g.K, Cperm, T, st->in_mode == FIN_F32 ? 0 : 1, st->Dpad,
                                   st->Kpad, st->w8.as<int8_t>(), s));
        BNN_TRY(fused_prep_params(st->w8.as<int8_t>(), st->Kpad, g.D, int(prm_n), g.K, L.bias.as<float>(),
                                  aff ? aff->scale.as<float>() : nullptr, aff ? aff->shift.as<float>() : nullptr,
                                  st->prm.as<int4>(), bad.as<int>(), s));
        g.prm = st->prm.as<int4>();
        const int bns[5] = {16, 32, 64, 128, 256};
        for (int b = 0; b < 5; ++b)
            BNN_TRY(fused_make_tmap(&st->tm[b], st->w8.as<int8_t>(), st->Dpad, st->Kpad, bns[b]));
        if ((kind == BNN_LAYER_CONV && st->epi == FEPI_BITS && st->in_mode != FIN_F32) ||
            kind == BNN_LAYER_LINEAR) {  // FP4 operands (conv: swap4 / halo4; linear: lin4)
            const int Kpad4 = int(round_up(size_t(g.K), 256));
            g.kb4 = Kpad4 / 256;
            g.kq4 = (g.K - 256 * (g.kb4 - 1) + 63) / 64;
            BNN_TRY(st->w4.alloc(size_t(st->Dpad) * (Kpad4 / 2)));
            BNN_TRY(prep_weights4(st->w8.as<int8_t>(), st->Kpad, g.K, st->Dpad, Kpad4, st->w4.as<uint8_t>(), s));
            BNN_TRY(make_tmap_2d_s8(&st->tm4, st->w4.p, size_t(st->Dpad), size_t(Kpad4 / 2), size_t(Kpad4 / 2), 128));
            st->fp4_ok = true;
        }
        if (st->epi == FEPI_LOGITS && kind == BNN_LAYER_LINEAR && g.D <= 64) {
            st->small_logits = true;
            BNN_TRY(st->wbits.alloc(size_t(g.D) * g.Cw * sizeof(uint32_t)));
            BNN_TRY(prep_logit_bits(st->w8.as<int8_t>(), st->Kpad, g.K, g.D, g.Cw, st->wbits.as<uint32_t>(), s));
        }
        if (st->in_mode == FIN_PIX && st->epi == FEPI_BITS && g.C <= 32 && g.SH == 1 && g.SW == 1 &&
            g.KH == 2 * g.PH + 1 && g.KW == 2 * g.PW + 1 && g.PH <= 1 && g.PW <= 1 && g.OH == g.H && g.OW == g.W &&
            g.D % 32 == 0) {  // halo0: the first conv on the FP4 tensor cores, channels padded to 64
            const int Kp4 = int(round_up(size_t(g.KH * g.KW * 64), 256));
            BNN_TRY(st->w4h.alloc(size_t(st->Dpad) * (Kp4 / 2)));
            BNN_TRY(prep_w4_pix(L.packed.as<uint32_t>(), L.wpl, g.D, g.C, g.KH, g.KW, st->Dpad, Kp4,
                                st->w4h.as<uint8_t>(), s));
            BNN_TRY(make_tmap_2d_s8(&st->tm4h, st->w4h.p, size_t(st->Dpad), size_t(Kp4 / 2), size_t(Kp4 / 2), 128));
            st->halo0 = true;
        }
        if (st->in_mode == FIN_PIX && st->epi == FEPI_BITS && pix_popc_ok(g)) {
            st->pix_popc = true;
            BNN_TRY(st->wbits.alloc(size_t(g.D) * sizeof(uint32_t)));
            BNN_TRY(prep_logit_bits(st->w8.as<int8_t>(), st->Kpad, g.K, g.D, 1, st->wbits.as<uint32_t>(), s));
            std::vector<uint32_t> wb(g.D);
            std::vector<int4> pr(g.D);
            BNN_CUDA(cudaMemcpyAsync(wb.data(), st->wbits.p, wb.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
            BNN_CUDA(cudaMemcpyAsync(pr.data(), st->prm.p, pr.size() * sizeof(int4), cudaMemcpyDeviceToHost, s));
            BNN_CUDA(cudaStreamSynchronize(s));
            BNN_TRY(make_pix_params(wb.data(), pr.data(), g.D, g.K, &st->pix));
        }
        if (st->epi == FEPI_BITS) {
            const size_t pos = kind == BNN_LAYER_CONV ? size_t(g.OH) * g.OW / (pool ? 4 : 1) : 1;
            st->out_words_per_image = pos * g.Dw;
            max_words = std::max(max_words, st->out_words_per_image);
        }
        net->stages.push_back(std::move(st));
        i = j;
    }
    int bad_h = 0;
    BNN_CUDA(cudaMemcpyAsync(&bad_h, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    if (bad_h) return no("a channel's binarization is not a step function of the accumulator");
    net->bits_words_per_image = max_words;
    net->fusable = true;
    return BNN_OK;
}

// Tile shape for a launch: cta_group (1: M=128 per CTA, 2: M=256 per CTA pair) and BN (the
// MMA N, weight rows per tile): the widest BN that still gives every CTA (pair) a tile.
int g_forced_cg = -1, g_forced_bn = -1;  // bnn_set_fused_tiling (tests, experiments); -1: from env
int g_tiling_epoch = 0;                   // bumped by bnn_set_fused_tiling: invalidates captured graphs

int g_forced_split = -1;  // BNN_FUSED_SPLIT / bnn_set_fused_split: 0 auto, 1 never, S forced

void choose_tile(int D, size_t rows, int KB, bool pool, int& cg, int& bn, int& ks) {
    if (g_forced_cg < 0) g_forced_cg = getenv("BNN_FUSED_CG") ? atoi(getenv("BNN_FUSED_CG")) : 0;
    if (g_forced_bn < 0) g_forced_bn = getenv("BNN_FUSED_BN") ? atoi(getenv("BNN_FUSED_BN")) : 0;
    if (g_forced_split < 0) g_forced_split = getenv("BNN_FUSED_SPLIT") ? atoi(getenv("BNN_FUSED_SPLIT")) : 0;
    const int forced_cg = g_forced_cg, forced_bn = g_forced_bn;
    // CTA pairs measured no faster than single CTAs here (the i8 MMA runs ~128 cycles per
    // instruction for any N <= 256 in both modes), so pairs are opt-in.
    cg = forced_cg == 1 || forced_cg == 2 ? forced_cg : 1;
    const size_t m_tiles = ceil_div(rows, size_t(128 * cg)), units = size_t(num_sms()) / cg;
    bn = 32;
    while (bn < 256 && bn < D) bn *= 2;
    const bool bn_forced = forced_bn == 32 || forced_bn == 64 || forced_bn == 128 || forced_bn == 256;
    if (bn_forced) bn = forced_bn;
    ks = 1;
    const size_t out_tiles = m_tiles * ceil_div(size_t(D), size_t(bn));
    // Few, K-deep output tiles (the linear layers at small batch): an MMA costs the same for
    // any N <= 256, so keep BN wide and split K across CTAs instead of narrowing BN.
    const bool can_split = cg == 1 && !pool && g_forced_split != 1;
    // The split completion (partials out, a counter, a reduction) costs ~10 us, so only deep
    // reductions split (measured at batch 256: fc 8192->1024 gains, 1024->1024 loses).
    if (can_split && (g_forced_split > 1 || (out_tiles * 2 <= units && KB >= 32))) {
        const int cap = g_forced_split > 1 ? g_forced_split : 16;
        const int kmin = g_forced_split > 1 ? 1 : 4;  // auto: at least 4 K-blocks per slice
        // every split tile needs its own co-resident CTA (fused.cu split-K completion)
        while (ks < cap && out_tiles * size_t(ks * 2) <= units && ks * 2 * kmin <= KB) ks *= 2;
        // Half-width tiles with half the slices keep the same CTA count and halve the partial
        // sums written and re-read (fc 8192->1024 at batch 256: 28 -> 24 us per layer event).
        if (ks > 1 && bn == 256 && !bn_forced && g_forced_split <= 1) {
            const size_t out2 = m_tiles * ceil_div(size_t(D), size_t(128));
            int ks2 = 1;
            while (ks2 < cap && out2 * size_t(ks2 * 2) <= units && ks2 * 2 * kmin <= KB) ks2 *= 2;
            if (ks2 > 1 && out2 * size_t(ks2) >= out_tiles * size_t(ks)) bn = 128, ks = ks2;
        }
    }
    if (ks == 1 && !bn_forced)
        while (bn > 32 && m_tiles * ceil_div(size_t(D), size_t(bn)) < units) bn /= 2;
}

int box_index(int box) { return box == 16 ? 0 : box == 32 ? 1 : box == 64 ? 2 : box == 128 ? 3 : 4; }

int ensure_arena(bnn_net* net, size_t batch) {
    if (net->arena_batch >= batch) return BNN_OK;
    BNN_TRY(net->act[0].alloc(net->max_act_per_image * batch * 4));
    BNN_TRY(net->act[1].alloc(net->max_act_per_image * batch * 4));
    BNN_TRY(net->lines.alloc(std::max<size_t>(net->max_lines_words_per_image, 1) * batch * 4));
    net->arena_batch = batch;
    return BNN_OK;
}

cudaEvent_t take_event(bnn_net* net) {
    if (!net->pool.empty()) {
        cudaEvent_t e = net->pool.back();
        net->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct EventPair {
    bnn_net* net;
    size_t layer;
    int what;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    EventPair(bnn_net* n, size_t l, int w, cudaStream_t st) : net(n), layer(l), what(w), s(st) {
        if (net->timing) {
            a = take_event(net);
            cudaEventRecord(a, s);
        }
    }
    void close() {
        if (!a) return;
        cudaEvent_t b = take_event(net);
        cudaEventRecord(b, s);
        net->pending.push_back({layer, what, a, b});
        a = nullptr;
    }
};

// Per-layer execution of a weighted layer in the layer-by-layer engine (ExecKernel,
// network.hpp:89-91, resolved as resolve_exec does at network.cpp:318-327).
enum LayerExec { EXEC_BINARY = 0, EXEC_FLOAT = 1, EXEC_BINREF = 2, EXEC_NAIVE = 3 };

int layer_exec(const bnn_net* net, const Layer& L) {
    switch (net->engine_policy) {
        case BNN_ENGINE_FLOAT: return EXEC_FLOAT;
        case BNN_ENGINE_BINARY_REFERENCE: return EXEC_BINREF;
        case BNN_ENGINE_NAIVE: return EXEC_NAIVE;
        case BNN_ENGINE_PER_LAYER:  // the layer's own KernelChoice (network.cpp:318-325)
            return L.spec.kernel == BNN_KERNEL_BINARY ? EXEC_BINARY
                   : L.spec.kernel == BNN_KERNEL_NAIVE ? EXEC_NAIVE
                                                       : EXEC_FLOAT;
        default: return EXEC_BINARY;
    }
}

// sign(layer.weights) for the BinaryReference graph (network.cpp:357,380), made once per layer.
int ensure_wpm1(Layer& L, cudaStream_t s) {
    if (L.wpm1.p) return BNN_OK;
    BNN_TRY(L.wpm1.alloc(L.rows * L.cols * 4));
    return launch_unary(0, L.wf.as<float>(), L.rows * L.cols, L.wpm1.as<float>(), s);
}

// network_forward (network.cpp:330-420), one reference operator (or fused pair) per kernel,
// float activations ping-ponging between two arena buffers. Weighted layers run as
//   binary: K2 binary im2col / K1 pack_cols(sign) + K3 xnor GEMM with the bias epilogue
//           (conv_forward_binary, linear_forward_packed: network.cpp:65-79, 121-126)
//   float : float im2col + float_gemm on the float weights (conv_forward_float,
//           linear_forward Float: network.cpp:50-63, 113-120; control.cu)
//   binref: sign(im2col) / sign(x) + float_gemm on sign(weights) (conv_forward_binary_reference,
//           linear_forward_binary_reference: network.cpp:81-94, 128-131) -- the verify oracle
//   naive : direct convolution (conv_forward_naive, network.cpp:96-111); linear as float
int forward_layerwise(bnn_net* net, const float* x, size_t B, float* logits, cudaStream_t s) {
    BNN_TRY(ensure_arena(net, B));
    size_t launches = 0;
    const float* cur = x;
    int which = 0;
    auto next = [&]() { float* o = net->act[which].as<float>(); which ^= 1; return o; };
    for (size_t li = 0; li < net->layers.size(); ++li) {
        Layer& L = *net->layers[li];
        EventPair layer_ev(net, li, 0, s);
        const int ex = layer_exec(net, L);
        switch (L.spec.kind) {
            case BNN_LAYER_CONV: {
                float* out = next();
                const size_t N = B * L.out_h * L.out_w, P = L.out_h * L.out_w;
                if (ex == EXEC_BINARY) {
                    BNN_TRY(launch_im2col_sign_pack(cur, B, L.in_c, L.in_h, L.in_w, &L.geom,
                                                    net->lines.as<uint32_t>(), L.wpl, s));
                    EventPair gemm_ev(net, li, 1, s);
                    BNN_TRY(gemm_f32(L.packed.as<uint32_t>(), L.wpl, net->lines.as<uint32_t>(), L.wpl, L.rows, N,
                                     L.cols, L.bias.as<float>(), P, out, s));
                    gemm_ev.close();
                    launches += 2;
                } else if (ex == EXEC_NAIVE) {
                    EventPair gemm_ev(net, li, 1, s);
                    BNN_TRY(launch_naive_conv(cur, B, L.in_c, L.in_h, L.in_w, L.wf.as<float>(), L.bias.as<float>(),
                                              &L.geom, out, s));
                    gemm_ev.close();
                    ++launches;
                } else {
                    if (net->fcols.bytes < L.cols * N * 4) BNN_TRY(net->fcols.alloc(L.cols * N * 4));
                    float* cols = net->fcols.as<float>();
                    BNN_TRY(launch_im2col_f32(cur, B, L.in_c, L.in_h, L.in_w, &L.geom, cols, s));
                    ++launches;
                    const float* w = L.wf.as<float>();
                    if (ex == EXEC_BINREF) {
                        BNN_TRY(launch_unary(0, cols, L.cols * N, cols, s));  // sign(im2col(x))
                        BNN_TRY(ensure_wpm1(L, s));
                        w = L.wpm1.as<float>();
                        ++launches;
                    }
                    EventPair gemm_ev(net, li, 1, s);
                    BNN_TRY(launch_float_gemm(w, cols, L.rows, N, L.cols, L.bias.as<float>(), P, out, s));
                    gemm_ev.close();
                    ++launches;
                }
                cur = out;
                break;
            }
            case BNN_LAYER_LINEAR: {
                if (!L.in_flat) {  // flatten_to_columns: [B, F] -> [F, B]
                    float* t = next();
                    BNN_TRY(launch_transpose(cur, B, L.cols, t, s));
                    ++launches;
                    cur = t;
                }
                if (ex == EXEC_BINARY) {
                    float* out = next();
                    BNN_TRY(launch_pack_cols(cur, L.cols, B, net->lines.as<uint32_t>(), L.wpl, nullptr, s));
                    EventPair gemm_ev(net, li, 1, s);
                    BNN_TRY(gemm_f32(L.packed.as<uint32_t>(), L.wpl, net->lines.as<uint32_t>(), L.wpl, L.rows, B,
                                     L.cols, L.bias.as<float>(), B, out, s));
                    gemm_ev.close();
                    launches += 2;
                    cur = out;
                } else {
                    const float* w = L.wf.as<float>();
                    if (ex == EXEC_BINREF) {
                        float* t = next();
                        BNN_TRY(launch_unary(0, cur, L.cols * B, t, s));  // sign(x)
                        BNN_TRY(ensure_wpm1(L, s));
                        w = L.wpm1.as<float>();
                        ++launches;
                        cur = t;
                    }
                    float* out = next();
                    EventPair gemm_ev(net, li, 1, s);
                    BNN_TRY(launch_float_gemm(w, cur, L.rows, B, L.cols, L.bias.as<float>(), B, out, s));
                    gemm_ev.close();
                    ++launches;
                    cur = out;
                }
                break;
            }
            case BNN_LAYER_MAXPOOL: {
                float* out = next();
                BNN_TRY(launch_maxpool2(cur, B, L.in_c, L.in_h, L.in_w, out, s));
                ++launches;
                cur = out;
                break;
            }
            case BNN_LAYER_AFFINE: {
                float* out = next();
                const size_t n = L.in_flat ? L.in_c * B : B * L.in_c * L.in_h * L.in_w;
                const size_t plane = L.in_flat ? B : L.in_h * L.in_w;
                BNN_TRY(launch_affine(cur, n, L.in_c, plane, L.scale.as<float>(), L.shift.as<float>(), out, s));
                ++launches;
                cur = out;
                break;
            }
            case BNN_LAYER_SIGN:
            case BNN_LAYER_HTANH: {
                float* out = next();
                const size_t n = L.in_flat ? L.in_c * B : B * L.in_c * L.in_h * L.in_w;
                BNN_TRY(launch_unary(L.spec.kind == BNN_LAYER_SIGN ? 0 : 1, cur, n, out, s));
                ++launches;
                cur = out;
                break;
            }
        }
        layer_ev.close();
    }
    const Layer& last = *net->layers.back();
    if (last.out_flat) {
        BNN_CUDA(cudaMemcpyAsync(logits, cur, net->logits * B * 4, cudaMemcpyDeviceToDevice, s));
    } else {
        BNN_TRY(launch_transpose(cur, B, net->logits, logits, s));
        ++launches;
    }
    net->last_launches = launches;
    return BNN_OK;
}



// Swapped-operand conv kernel (fused_swap_kernel: channels on the MMA's M, positions on N)
// for conv layers with a packed-bit epilogue. BNN_FUSED_SWAP / bnn_set_fused_swap: 1 (default)
// for layers of <= 128 output channels, where the position-major kernel runs the MMA at half
// rate (measured at batch 256: conv 128->128 70.5 -> 58.7 us); 2 for every such conv layer
// (wider layers measured slower: the swapped stage is shared-memory-bandwidth bound); 0 off.
// Forced tilings (bnn_set_fused_tiling) keep the position-major kernel.
int g_swap = -1;
int g_small_logits = 1;  // bnn_set_fused_small_logits: tiny final layers on the CUDA cores
int g_pix_popc = -1;     // bnn_set_fused_pix_popc / BNN_PIX_POPC (default 3): K <= 32 pixel-input convs on the CUDA cores

bool use_swap(const bnn_net* net, const FusedStage& st, int cg) {
    if (g_swap < 0) g_swap = getenv("BNN_FUSED_SWAP") ? atoi(getenv("BNN_FUSED_SWAP")) : 1;
    return g_swap != 0 && g_forced_cg <= 0 && g_forced_bn <= 0 && cg == 1 &&
           net->layers[st.layer]->spec.kind == BNN_LAYER_CONV && st.epi == FEPI_BITS && st.in_mode != FIN_F32 &&
           (g_swap == 2 || st.g.D <= 128);
}

// FP4 operands (fused_swap4_kernel, kind::mxf4): BNN_FUSED_FP4 / bnn_set_fused_fp4: 0 off,
// 1 (default) every conv layer with a packed-bit input and output (conv 128->128: 1.26 -> 0.94 M
// cycles per CTA at B=4096; the wider layers about even with the position-major int8 kernel at
// large batch and faster at 256, profiles/r01_fp4_*), 2 also the pixel-input first layer
// (measured slower there: its one K step leaves the epilogue the bound).
int g_fp4 = -1;

bool use_fp4(const bnn_net* net, const FusedStage& st, int cg) {
    if (g_fp4 < 0) g_fp4 = getenv("BNN_FUSED_FP4") ? atoi(getenv("BNN_FUSED_FP4")) : 1;
    if (!st.fp4_ok || g_fp4 == 0 || g_forced_cg > 0 || g_forced_bn > 0 || cg != 1) return false;
    return g_fp4 == 2 || st.in_mode == FIN_BITS;
}

// Halo-tile FP4 conv (halo.cu, halo4_kernel): BNN_FUSED_HALO / bnn_set_fused_halo: 0 off, 1
// (default) every "same" conv with a packed-bit input whose weight slice fits in shared memory;
// 2 also the others with the weights streamed through a ring (measured slower than
// fused_swap4_kernel for VGG-small's conv 512 -> 512: 40 vs 32 us per layer at batch 256).
int g_halo = -1;

bool use_halo(const bnn_net* net, const FusedStage& st, int cg) {
    if (g_halo < 0) g_halo = getenv("BNN_FUSED_HALO") ? atoi(getenv("BNN_FUSED_HALO")) : 1;
    return g_halo != 0 && use_fp4(net, st, cg) && st.in_mode == FIN_BITS;
}

// FP4 linear layers (linear.cu, lin4_kernel + lin_finish_kernel): BNN_FUSED_LIN4 /
// bnn_set_fused_lin4: 0 off (int8 fused_layer_kernel), 1 (default) every linear stage except the
// CUDA-core logits layer.
int g_lin4 = -1;

bool use_lin4(const bnn_net* net, const FusedStage& st) {
    if (g_lin4 < 0) g_lin4 = getenv("BNN_FUSED_LIN4") ? atoi(getenv("BNN_FUSED_LIN4")) : 1;
    return g_lin4 != 0 && st.fp4_ok && g_forced_cg <= 0 && g_forced_bn <= 0 &&
           net->layers[st.layer]->spec.kind == BNN_LAYER_LINEAR && st.in_mode == FIN_BITS;
}

// First conv through halo4 (halo0): BNN_FUSED_HALO0 / bnn_set_fused_halo0: 1 on, 0 (default) the
// CUDA-core pix_tile / pix_popc kernels (or the int8 tensor-core path). Measured slower for
// VGG-small's conv 3 -> 128 (41 vs 24 us per layer at batch 256): with K = 9 x 64 a tile is only 9
// MMAs, so its epilogue (128 channels x 240 positions) bounds the kernel.
int g_halo0 = -1;

// The halo0 plan for a pixel-input stage: the first conv seen as a 64-channel conv (2 packed
// words per pixel, K' = taps * 64) whose producers sign the float input themselves.
bool halo0_plan(const FusedStage& st, const FusedGeom& g, const float* x, HaloGeom& hg) {
    FusedGeom g0 = g;
    g0.C = 64, g0.Cw = 2, g0.K = g.KH * g.KW * 64;
    g0.kb4 = (g0.K + 255) / 256;
    g0.kq4 = (g0.K - 256 * (g0.kb4 - 1) + 63) / 64;
    if (!halo4_plan(g0, hg) || hg.wst) return false;
    hg.in_f32 = x;
    hg.creal = g.C;
    return true;
}

int forward_fused(bnn_net* net, const float* x, size_t B, float* logits, cudaStream_t s) {
    if (net->bits_batch < B) {
        const size_t bytes = std::max<size_t>(net->bits_words_per_image, 1) * B * 4;
        BNN_TRY(net->bits[0].alloc(bytes));
        BNN_TRY(net->bits[1].alloc(bytes));
        const size_t pre_words = net->stages.front()->pre_encode ? wpl_of(net->in_c * net->in_h * net->in_w) : 0;
        BNN_TRY(net->pix.alloc(B * std::max(net->in_h * net->in_w, pre_words) * 4));
        net->bits_batch = B;
        ++net->arena_epoch;
    }
    static const bool prof = getenv("BNN_FUSED_PROFILE") != nullptr;
    // per-stage launch geometry (batch-dependent fields, tiling, buffers)
    struct Plan {
        FusedGeom g;
        int cg, bn;
        bool lin4 = false;
        LinGeom lg{};
        CUtensorMap tmx;  // the e2m1 images of a TMA-fed lin4 stage
        bool in4_ready = false;  // ... written by the previous lin4 stage's epilogue
    };
    std::vector<Plan> plans;
    size_t ws_need = 0, sem_need = 0;  // the largest split-K workspace of any stage
    size_t lin_ws_need = 0, lin_sem_need = 0;  // the largest lin4 workspace and counter array
    size_t lin_x4_need = 0;                    // the largest expanded image block of a TMA-fed lin4
    const void* in = x;
    int which = 0;
    (void)prof;
    for (auto& stp : net->stages) {
        FusedStage& st = *stp;
        FusedGeom g = st.g;
        const bool conv = net->layers[st.layer]->spec.kind == BNN_LAYER_CONV;
        const size_t rows = conv ? B * size_t(g.OH) * g.OW : B;
        if (rows > size_t(0x7fffffff) / 2) return fail(BNN_E_CONFIG, "fused engine: batch too large");
        g.B = int(B);
        g.in = in;
        g.rows = int(rows);
        int cg = 1, bn = 32, ks = 1;
        choose_tile(g.D, rows, g.KB, g.pool != 0, cg, bn, ks);
        g.n_tiles = int(ceil_div(size_t(g.D), size_t(bn)));
        g.ksplit = ks;
        if (ks > 1) {  // split-K workspace and per-output-tile counters (pointers set below)
            const size_t m_tiles = ceil_div(rows, size_t(128));
            g.ws_rows = int(m_tiles * 128), g.ws_ld = g.n_tiles * bn;
            ws_need = std::max(ws_need, size_t(ks) * g.ws_rows * g.ws_ld * 4);
            sem_need = std::max(sem_need, m_tiles * g.n_tiles * 2 * sizeof(unsigned));
        }
        if (st.epi == FEPI_BITS) {
            g.out_bits = net->bits[which].as<uint32_t>();
            which ^= 1;
        } else {
            g.out_f32 = logits;
            g.ldo = int(B);
        }
        if (st.in_mode == FIN_PIX || st.pre_encode) g.in = net->pix.as<uint32_t>();
        Plan pl{g, cg, bn};
        if (use_lin4(net, st) && !(st.small_logits && g_small_logits) && lin4_plan(g, st.epi, pl.lg)) {
            pl.lin4 = true;
            lin_ws_need = std::max(lin_ws_need, lin4_ws_bytes(pl.lg));
            lin_sem_need = std::max(lin_sem_need, lin4_sem_count(pl.lg) * sizeof(unsigned));
            if (pl.lg.tmab) lin_x4_need = std::max(lin_x4_need, size_t(pl.lg.B) * pl.lg.Kw * 16);
        }
        plans.push_back(pl);
        in = g.out_bits;
    }
    // one split-K workspace shared by the stages (they run one after another), sized for the
    // largest before any pointer is handed out: growing it between stages would leave the
    // earlier stages' plans pointing at freed memory
    if (net->ws.bytes < ws_need) {
        BNN_TRY(net->ws.alloc(ws_need));
        ++net->arena_epoch;
    }
    if (net->sem.bytes < sem_need) {
        ++net->arena_epoch;
        BNN_TRY(net->sem.alloc(sem_need));
        BNN_CUDA(cudaMemsetAsync(net->sem.p, 0, sem_need, s));  // kernels leave them at 0
    }
    if (net->lin_ws.bytes < lin_ws_need) {
        BNN_TRY(net->lin_ws.alloc(lin_ws_need));
        ++net->arena_epoch;
    }
    if (net->lin_sem.bytes < lin_sem_need) {
        BNN_TRY(net->lin_sem.alloc(lin_sem_need));
        BNN_CUDA(cudaMemsetAsync(net->lin_sem.p, 0, lin_sem_need, s));
        ++net->arena_epoch;
    }
    for (auto& b4 : net->lin_x4)
        if (b4.bytes < lin_x4_need) {
            BNN_TRY(b4.alloc(lin_x4_need));
            ++net->arena_epoch;
        }
    for (auto& pl : plans) {
        if (pl.g.ksplit > 1) pl.g.ws = net->ws.as<int>(), pl.g.sem = net->sem.as<unsigned>();
        if (pl.lin4) pl.lg.ws = net->lin_ws.as<int>(), pl.lg.sem = net->lin_sem.as<unsigned>();
    }
    // TMA-fed lin4 stages read e2m1 images from lin_x4[k]; a preceding lin4 stage with a bits
    // epilogue writes them there directly (no expand_act4 launch), the buffers alternating
    for (size_t i = 0, k = 0; i < plans.size(); ++i) {
        Plan& pl = plans[i];
        if (!(pl.lin4 && pl.lg.tmab)) continue;
        pl.lg.in4 = net->lin_x4[k].as<uint8_t>();
        k ^= 1;
        const size_t lb = size_t(pl.lg.Kw) * 16;
        BNN_TRY(make_tmap_2d_s8(&pl.tmx, pl.lg.in4, size_t(pl.lg.B), lb, lb, uint32_t(pl.lg.NB)));
        if (i > 0 && plans[i - 1].lin4 && plans[i - 1].lg.epi == FEPI_BITS && plans[i - 1].lg.Dw == pl.lg.Kw) {
            plans[i - 1].lg.out4 = pl.lg.in4;
            pl.in4_ready = true;
        }
    }
    size_t launches = 0;
    for (size_t i = 0; i < plans.size(); ++i) {
        FusedStage& st = *net->stages[i];
        const FusedGeom& g = plans[i].g;
        EventPair layer_ev(net, st.layer, 0, s);
        if (g_pix_popc < 0) {
            g_pix_popc = getenv("BNN_PIX_POPC") ? atoi(getenv("BNN_PIX_POPC")) : 3;
            if (g_pix_popc < 0 || g_pix_popc > 3) g_pix_popc = 3;  // the range bnn_set_fused_pix_popc accepts
        }
        // pix_popc 1: the CUDA-core first conv reads the float input itself (no pack_pixels;
        // pix_tile_kernel stages packed input rows in shared memory when the layer allows);
        // 2: after pack_pixels; 3 (default): 1 up to batch 512 (B=256: 1.754 vs 1.731 M img/s),
        // 2 above (B=4096: 2.70 vs 2.66 M, the packer's one pass beats the per-tile halo rows)
        if (g_halo0 < 0) g_halo0 = getenv("BNN_FUSED_HALO0") ? atoi(getenv("BNN_FUSED_HALO0")) : 0;
        HaloGeom hg0;
        const bool use_h0 = st.halo0 && g_halo0 && g_halo != 0 && halo0_plan(st, g, x, hg0);
        const bool pix_f32 = st.pix_popc && (g_pix_popc == 1 || (g_pix_popc == 3 && B <= 512));
        if (st.in_mode == FIN_PIX && !pix_f32 && !use_h0) {  // first-layer sign bits, one word per pixel
            BNN_TRY(launch_pack_pixels(x, B, g.C, size_t(g.H) * g.W, net->pix.as<uint32_t>(), s));
            ++launches;
        }
        const bool pre4 = st.pre_encode && plans[i].lin4 && plans[i].lg.tmab &&
                          size_t(g.Cw) == wpl_of(size_t(g.C));  // straight to e2m1 images
        if (pre4) {
            BNN_TRY(launch_pack_rows_e2m1(x, B, size_t(g.C), plans[i].lg.in4, s));
            ++launches;
        } else if (st.pre_encode) {  // K1: pack_rows(sign(x)) over [B, F]
            BNN_TRY(launch_pack_rows(x, B, size_t(g.C), net->pix.as<uint32_t>(), size_t(g.Cw), nullptr, s));
            ++launches;
        }
        EventPair gemm_ev(net, st.layer, 1, s);
        if (st.small_logits && g_small_logits) {
            BNN_TRY(launch_logits_popc(g, st.wbits.as<uint32_t>(), s));
        } else if (use_h0) {
            HaloGeom h = hg0;
            h.out = g.out_bits;
            BNN_TRY(launch_halo4(st.tm4h, h, s));
        } else if (st.pix_popc && g_pix_popc) {
            FusedGeom gp = g;
            if (pix_f32) gp.in = x;
            BNN_TRY(launch_pix_popc(gp, st.pix, pix_f32, s));
        }
        else if (plans[i].lin4) {
            if (plans[i].lg.tmab && !pre4 && !plans[i].in4_ready) {
                BNN_TRY(launch_expand_act4(plans[i].lg, s));
                ++launches;
            }
            BNN_TRY(launch_lin4(st.tm4, plans[i].lg.tmab ? plans[i].tmx : st.tm4, plans[i].lg, s));
        }
        else if (HaloGeom hg; use_halo(net, st, plans[i].cg) && halo4_plan(g, hg) && (!hg.wst || g_halo == 2))
            BNN_TRY(launch_halo4(st.tm4, hg, s));
        else if (use_fp4(net, st, plans[i].cg))
            BNN_TRY(launch_swap4(st.in_mode, st.tm4, g, s));
        else if (use_swap(net, st, plans[i].cg))
            BNN_TRY(launch_swap(st.in_mode, st.tm[box_index(128)], g, s));
        else
            BNN_TRY(launch_fused(plans[i].cg, plans[i].bn, st.in_mode, st.epi, st.tm[box_index(plans[i].bn / plans[i].cg)], g, s));
        st.kname = bnn_last_gemm_kernel();
        gemm_ev.close();
        layer_ev.close();
        ++launches;
    }

    net->last_launches = launches;
    return BNN_OK;
}

// The fused engine serves ExecKernel::Binary: engine AUTO / FUSED, or PER_LAYER with every
// weighted layer's KernelChoice Binary.
bool use_fused(const bnn_net* net) {
    if (!net->fusable) return false;
    if (net->engine_policy == BNN_ENGINE_AUTO || net->engine_policy == BNN_ENGINE_FUSED) return true;
    if (net->engine_policy != BNN_ENGINE_PER_LAYER) return false;
    for (const auto& L : net->layers)
        if ((L->spec.kind == BNN_LAYER_CONV || L->spec.kind == BNN_LAYER_LINEAR) && L->spec.kernel != BNN_KERNEL_BINARY)
            return false;
    return true;
}

// The fused forward is a fixed sequence of ~10 launches; for a repeated (x, B, logits, stream)
// it is captured once into a CUDA graph and replayed (one launch from the host). Not used
// with per-layer timing (events), the profiling mode, or the legacy default stream (which
// cannot be captured).
int forward_graphed(bnn_net* net, const float* x, size_t B, float* logits, cudaStream_t s) {
    static const bool prof = getenv("BNN_FUSED_PROFILE") != nullptr || getenv("BNN_HALO_PROFILE") != nullptr ||
                             getenv("BNN_LIN4_PROFILE") != nullptr;
    const bool graphable = net->use_graphs && !net->timing && !prof && s != nullptr;
    if (!graphable) return forward_fused(net, x, B, logits, s);
    // small cache: a pipelined caller alternates input/output buffers
    bnn_net::Graph* gc = nullptr;
    for (auto& e : net->graphs) {
        if (e.exec && (e.epoch != g_tiling_epoch || e.arena != net->arena_epoch)) {  // stale kernels / buffers
            cudaGraphExecDestroy(e.exec);
            e = bnn_net::Graph{};
        }
        if (e.key_set && e.x == x && e.B == B && e.logits == logits && e.s == s) gc = &e;
    }
    if (gc && gc->exec) {
        BNN_CUDA(cudaGraphLaunch(gc->exec, s));
        net->last_launches = gc->launches;
        return BNN_OK;
    }
    if (!gc) {
        // first sighting: run eagerly (sizes the arena, sets kernel attributes), remember the key
        bnn_net::Graph& e = net->graphs[net->graph_next++ % net->graphs.size()];
        if (e.exec) cudaGraphExecDestroy(e.exec);
        e = bnn_net::Graph{};
        const int rc = forward_fused(net, x, B, logits, s);
        e.key_set = true, e.x = x, e.B = B, e.logits = logits, e.s = s;
        e.epoch = g_tiling_epoch, e.arena = net->arena_epoch;
        return rc;
    }
    cudaGraph_t graph = nullptr;
    BNN_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    const int rc = forward_fused(net, x, B, logits, s);
    const cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (rc != BNN_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    BNN_CUDA(ce);
    const cudaError_t ie = cudaGraphInstantiate(&gc->exec, graph, 0);
    cudaGraphDestroy(graph);
    BNN_CUDA(ie);
    gc->launches = net->last_launches;
    gc->epoch = g_tiling_epoch, gc->arena = net->arena_epoch;
    BNN_CUDA(cudaGraphLaunch(gc->exec, s));
    return BNN_OK;
}

int forward(bnn_net* net, const float* x, size_t B, float* logits, cudaStream_t s) {
    if (B == 0) return fail(BNN_E_CONFIG, "batch must be >= 1");
    if (use_fused(net)) return forward_graphed(net, x, B, logits, s);
    return forward_layerwise(net, x, B, logits, s);
}
}  // namespace
}  // namespace bnnk

using namespace bnnk;

extern "C" {

size_t bnn_default_spec(bnn_layer_spec* out, size_t cap) {  // network.cpp:422-465
    std::vector<bnn_layer_spec> l;
    auto conv = [&](uint64_t d) {
        bnn_layer_spec s{};
        s.kind = BNN_LAYER_CONV;
        s.kernel = BNN_KERNEL_BINARY;
        s.out_channels = d;
        s.kernel_h = s.kernel_w = 3;
        s.stride_h = s.stride_w = 1;
        s.pad_h = s.pad_w = 1;
        l.push_back(s);
    };
    auto push = [&](uint32_t k) {
        bnn_layer_spec s{};
        s.kind = k;
        s.stride_h = s.stride_w = 1;
        l.push_back(s);
    };
    auto linear = [&](uint64_t f) {
        bnn_layer_spec s{};
        s.kind = BNN_LAYER_LINEAR;
        s.kernel = BNN_KERNEL_BINARY;
        s.out_features = f;
        s.stride_h = s.stride_w = 1;
        l.push_back(s);
    };
    auto norm_act = [&] {
        push(BNN_LAYER_AFFINE);
        push(BNN_LAYER_HTANH);
        push(BNN_LAYER_SIGN);
    };
    conv(128); norm_act();
    conv(128); push(BNN_LAYER_MAXPOOL); norm_act();
    conv(256); norm_act();
    conv(256); push(BNN_LAYER_MAXPOOL); norm_act();
    conv(512); norm_act();
    conv(512); push(BNN_LAYER_MAXPOOL); norm_act();
    linear(1024); norm_act();
    linear(1024); norm_act();
    linear(10);
    for (size_t i = 0; i < l.size() && i < cap; ++i) out[i] = l[i];
    return l.size();
}

int bnn_net_create(const bnn_layer_spec* layers, size_t n_layers, size_t in_c, size_t in_h,
                   size_t in_w, uint64_t seed, int binarize_weights, bnn_net** out) {
    BNN_TRY(require_sm100());
    if (n_layers == 0) return fail(BNN_E_SHAPE, "network has no layers");
    if (in_c == 0 || in_h == 0 || in_w == 0) return fail(BNN_E_SHAPE, "input extents must be >= 1");
    auto net = std::make_unique<bnn_net>();
    net->in_c = in_c, net->in_h = in_h, net->in_w = in_w;
    net->binarize = binarize_weights != 0;  // float weights sign()ed; packed bits are the same either way
    cudaStream_t s;
    BNN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int rc = build(net.get(), layers, n_layers, seed, s);
    if (rc == BNN_OK) rc = plan_fused(net.get(), s);
    cudaStreamDestroy(s);
    if (rc != BNN_OK) return rc;
    *out = net.release();
    return BNN_OK;
}

void bnn_net_destroy(bnn_net* net) {
    if (!net) return;
    for (auto& p : net->pending) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto e : net->pool) cudaEventDestroy(e);
    net->drop_graphs();
    delete net;
}
size_t bnn_net_logits(const bnn_net* net) { return net->logits; }

int bnn_net_set_engine(bnn_net* net, int policy) {
    if (policy < BNN_ENGINE_AUTO || policy > BNN_ENGINE_PER_LAYER)
        return fail(BNN_E_CONFIG, "bad engine policy");
    if (policy == BNN_ENGINE_FUSED && !net->fusable)
        return fail(BNN_E_CONFIG, "network is not fusable: " + net->unfusable_why);
    net->engine_policy = policy;
    net->drop_graphs();
    return BNN_OK;
}

int bnn_set_fused_tiling(int cta_group, int bn) {
    if ((cta_group != 0 && cta_group != 1) || (bn != 0 && bn != 32 && bn != 64 && bn != 128 && bn != 256))
        return fail(BNN_E_CONFIG, "fused tiling: cta_group in {0,1}, bn in {0,32,64,128,256}");
    g_forced_cg = cta_group, g_forced_bn = bn;
    ++g_tiling_epoch;
    return BNN_OK;
}

int bnn_net_set_graphs(bnn_net* net, int enabled) {
    net->use_graphs = enabled != 0;
    net->drop_graphs();
    return BNN_OK;
}

int bnn_set_fused_split(int split) {
    if (split < 0 || split > 16 || (split > 1 && (split & (split - 1))))
        return fail(BNN_E_CONFIG, "fused split: 0 (auto), 1 (off) or a power of two <= 16");
    g_forced_split = split;
    ++g_tiling_epoch;
    return BNN_OK;
}

int bnn_debug_timeline(int op) { return fused_timeline(op); }

const char* bnn_net_layer_kernel(const bnn_net* net, size_t layer) {
    if (use_fused(net))
        for (const auto& st : net->stages)
            if (st->layer == layer) return st->kname;
    return "";
}

int bnn_set_fused_small_logits(int enabled) {
    g_small_logits = enabled ? 1 : 0;
    ++g_tiling_epoch;
    return BNN_OK;
}

int bnn_set_fused_pix_popc(int mode) {
    if (mode < 0 || mode > 3) return fail(BNN_E_CONFIG, "fused pix_popc: 0 (off), 1 (float input), 2 (packed pixels) or 3 (auto)");
    g_pix_popc = mode;
    ++g_tiling_epoch;
    return BNN_OK;
}

int bnn_set_fused_fp4(int mode) {
    if (mode < 0 || mode > 2) return fail(BNN_E_CONFIG, "fused fp4: 0 (off), 1 (swapped layers) or 2 (all convs)");
    g_fp4 = mode;
    ++g_tiling_epoch;
    return BNN_OK;
}

int bnn_set_fused_lin4(int enabled) {
    if (enabled < 0 || enabled > 3)
        return fail(BNN_E_CONFIG, "fused lin4: 0 (off), 1 (on), 2 (on, TMA-loaded images), 3 (on, producer-expanded images)");
    g_lin4 = enabled != 0;
    set_lin4_tma(enabled == 2 ? 1 : enabled == 3 ? 0 : -1);
    ++g_tiling_epoch;  // captured graphs hold the other kernels
    return BNN_OK;
}

int bnn_set_fused_halo0(int enabled) {
    if (enabled < 0 || enabled > 1) return fail(BNN_E_CONFIG, "fused halo0: 0 (off) or 1 (on)");
    g_halo0 = enabled;
    ++g_tiling_epoch;  // captured graphs hold the other kernels
    return BNN_OK;
}

int bnn_set_fused_halo(int enabled) {
    if (enabled < 0 || enabled > 2)
        return fail(BNN_E_CONFIG, "fused halo: 0 (off), 1 (resident weights only) or 2 (also streamed weights)");
    g_halo = enabled;
    ++g_tiling_epoch;  // captured graphs hold the other kernels
    return BNN_OK;
}

int bnn_set_fused_swap(int enabled) {
    if (enabled < 0 || enabled > 2) return fail(BNN_E_CONFIG, "fused swap: 0 (off), 1 (<= 128 channels) or 2 (all)");
    g_swap = enabled;
    ++g_tiling_epoch;  // captured graphs hold the other kernels
    return BNN_OK;
}


int bnn_set_fused_fp4_pair(int mode) {
    ++g_tiling_epoch;  // captured graphs hold the old kernels
    return fused_set_fp4_pair(mode);
}


int bnn_net_engine(const bnn_net* net) {
    if (use_fused(net)) return BNN_ENGINE_FUSED;
    switch (net->engine_policy) {
        case BNN_ENGINE_FLOAT:
        case BNN_ENGINE_BINARY_REFERENCE:
        case BNN_ENGINE_NAIVE:
        case BNN_ENGINE_PER_LAYER: return net->engine_policy;
        default: return BNN_ENGINE_GENERIC;
    }
}
size_t bnn_net_num_layers(const bnn_net* net) { return net->layers.size(); }
size_t bnn_net_last_launches(const bnn_net* net) { return net->last_launches; }

size_t bnn_net_device_bytes(const bnn_net* net) {
    return net->weight_bytes + net->act[0].bytes + net->act[1].bytes + net->lines.bytes;
}

int bnn_net_layer_params(const bnn_net* net, size_t i, uint32_t* packed, size_t* rows, size_t* cols,
                         float* bias, float* scale, float* shift) {
    if (i >= net->layers.size()) return fail(BNN_E_CONFIG, "layer index out of range");
    const Layer& L = *net->layers[i];
    if (rows) *rows = L.rows;
    if (cols) *cols = L.cols;
    if (packed && L.rows) BNN_CUDA(cudaMemcpy(packed, L.packed.p, L.rows * L.wpl * 4, cudaMemcpyDeviceToHost));
    if (bias && L.rows) BNN_CUDA(cudaMemcpy(bias, L.bias.p, L.rows * 4, cudaMemcpyDeviceToHost));
    if (scale && L.n_affine) BNN_CUDA(cudaMemcpy(scale, L.scale.p, L.n_affine * 4, cudaMemcpyDeviceToHost));
    if (shift && L.n_affine) BNN_CUDA(cudaMemcpy(shift, L.shift.p, L.n_affine * 4, cudaMemcpyDeviceToHost));
    return BNN_OK;
}

int bnn_net_layer_data(const bnn_net* net, size_t i, uint32_t* packed, float* weights, float* bias, float* scale,
                       float* shift) {
    if (i >= net->layers.size()) return fail(BNN_E_CONFIG, "layer index out of range");
    const Layer& L = *net->layers[i];
    if (weights && L.rows) BNN_CUDA(cudaMemcpy(weights, L.wf.p, L.rows * L.cols * 4, cudaMemcpyDeviceToHost));
    return bnn_net_layer_params(net, i, packed, nullptr, nullptr, bias, scale, shift);
}

int bnn_net_set_layer_data(bnn_net* net, size_t i, const uint32_t* packed, const float* weights, const float* bias,
                           const float* scale, const float* shift) {
    if (i >= net->layers.size()) return fail(BNN_E_CONFIG, "layer index out of range");
    Layer& L = *net->layers[i];
    BNN_CUDA(cudaDeviceSynchronize());  // no forward in flight reads the old parameters
    if (L.rows) {
        if (packed) BNN_CUDA(cudaMemcpy(L.packed.p, packed, L.rows * L.wpl * 4, cudaMemcpyHostToDevice));
        if (weights) {
            BNN_CUDA(cudaMemcpy(L.wf.p, weights, L.rows * L.cols * 4, cudaMemcpyHostToDevice));
            if (L.wpm1.p) {  // re-derived on next use
                cudaFree(L.wpm1.p);
                L.wpm1.p = nullptr, L.wpm1.bytes = 0;
            }
        }
        if (bias) BNN_CUDA(cudaMemcpy(L.bias.p, bias, L.rows * 4, cudaMemcpyHostToDevice));
    }
    if (L.n_affine) {
        if (scale) BNN_CUDA(cudaMemcpy(L.scale.p, scale, L.n_affine * 4, cudaMemcpyHostToDevice));
        if (shift) BNN_CUDA(cudaMemcpy(L.shift.p, shift, L.n_affine * 4, cudaMemcpyHostToDevice));
    }
    if (packed || bias || scale || shift) {  // the fused engine's prepared operands derive from these
        net->drop_graphs();
        cudaStream_t s;
        BNN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        const int rc = plan_fused(net, s);
        cudaStreamDestroy(s);
        BNN_TRY(rc);
        if (net->engine_policy == BNN_ENGINE_FUSED && !net->fusable) net->engine_policy = BNN_ENGINE_AUTO;
    }
    return BNN_OK;
}

int bnn_net_set_layer_kernel(bnn_net* net, size_t i, int kernel) {
    if (i >= net->layers.size()) return fail(BNN_E_CONFIG, "layer index out of range");
    if (kernel < BNN_KERNEL_FLOAT || kernel > BNN_KERNEL_NAIVE) return fail(BNN_E_CONFIG, "bad kernel choice");
    if (net->layers[i]->spec.kernel != uint32_t(kernel)) {
        net->layers[i]->spec.kernel = uint32_t(kernel);
        net->drop_graphs();
    }
    return BNN_OK;
}

int bnn_net_set_timing(bnn_net* net, int enabled) {
    net->timing = enabled != 0;
    return BNN_OK;
}

int bnn_net_timing(bnn_net* net, double* layer_ms, double* gemm_ms, size_t* gemm_launches) {
    const size_t n = net->layers.size();
    if (net->layer_ms.size() != n) {
        net->layer_ms.assign(n, 0.0);
        net->gemm_ms.assign(n, 0.0);
        net->gemm_launches.assign(n, 0);
    }
    for (auto& p : net->pending) {
        BNN_CUDA(cudaEventSynchronize(p.b));
        float ms = 0.f;
        BNN_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        if (p.what == 0) {
            net->layer_ms[p.layer] += ms;
        } else {
            net->gemm_ms[p.layer] += ms;
            net->gemm_launches[p.layer] += 1;
        }
        net->pool.push_back(p.a);
        net->pool.push_back(p.b);
    }
    net->pending.clear();
    for (size_t i = 0; i < n; ++i) {
        if (layer_ms) layer_ms[i] = net->layer_ms[i];
        if (gemm_ms) gemm_ms[i] = net->gemm_ms[i];
        if (gemm_launches) gemm_launches[i] = net->gemm_launches[i];
    }
    return BNN_OK;
}

int bnn_net_reset_timing(bnn_net* net) {
    BNN_TRY(bnn_net_timing(net, nullptr, nullptr, nullptr));
    std::fill(net->layer_ms.begin(), net->layer_ms.end(), 0.0);
    std::fill(net->gemm_ms.begin(), net->gemm_ms.end(), 0.0);
    std::fill(net->gemm_launches.begin(), net->gemm_launches.end(), 0);
    return BNN_OK;
}

int bnn_net_layer_shape(const bnn_net* net, size_t i, size_t out[8]) {
    if (i >= net->layers.size()) return fail(BNN_E_CONFIG, "layer index out of range");
    const Layer& L = *net->layers[i];
    out[0] = L.spec.kind;
    out[1] = L.rows;  // GEMM M
    out[2] = L.cols;  // GEMM K (= L)
    out[3] = L.spec.kind == BNN_LAYER_CONV ? L.out_h * L.out_w : (L.spec.kind == BNN_LAYER_LINEAR ? 1 : 0);
    out[4] = L.out_c;
    out[5] = L.out_h;
    out[6] = L.out_w;
    out[7] = L.out_flat ? 1 : 0;
    return BNN_OK;
}

int bnn_net_forward(bnn_net* net, const float* x, size_t batch, float* logits, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return forward(net, x, batch, logits, S(s));
}

int bnn_host_net_forward(bnn_net* net, const float* x, size_t batch, float* logits) {
    BNN_TRY(require_sm100());
    cudaStream_t s = nullptr;
    BNN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const size_t nx = batch * net->in_c * net->in_h * net->in_w, ny = batch * net->logits;
    int rc = BNN_OK;
    void *dx = nullptr, *dy = nullptr;
    if (cudaMalloc(&dx, nx * 4) != cudaSuccess || cudaMalloc(&dy, ny * 4) != cudaSuccess)
        rc = fail(BNN_E_CUDA, "cudaMalloc failed");
    if (rc == BNN_OK && cudaMemcpyAsync(dx, x, nx * 4, cudaMemcpyHostToDevice, s) != cudaSuccess)
        rc = fail(BNN_E_CUDA, "H2D copy failed");
    if (rc == BNN_OK) rc = forward(net, static_cast<float*>(dx), batch, static_cast<float*>(dy), s);
    if (rc == BNN_OK && cudaMemcpyAsync(logits, dy, ny * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        rc = fail(BNN_E_CUDA, "D2H copy failed");
    if (cudaStreamSynchronize(s) != cudaSuccess && rc == BNN_OK) rc = fail(BNN_E_CUDA, "sync failed");
    cudaFree(dx);
    cudaFree(dy);
    cudaStreamDestroy(s);
    return rc;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// Serving pipeline over host buffers: each submitted batch is copied in from (pinned) host
// memory, run through the network and its logits copied back, on three streams so that batch
// i+1's H2D and batch i-1's D2H overlap batch i's forward. `depth` device buffer sets; the
// forward of each set replays its own captured graph (bnn_net_forward's cache).
struct bnn_pipe {
    bnn_net* net = nullptr;
    size_t batch = 0, nx = 0, ny = 0;
    int depth = 0;
    uint64_t submitted = 0;
    cudaStream_t s_in = nullptr, s_run = nullptr, s_out = nullptr;
    std::vector<float*> dx, dy;
    std::vector<cudaEvent_t> ev_in, ev_run, ev_out;
};

extern "C" {

int bnn_pipe_create(bnn_net* net, size_t batch, int depth, bnn_pipe** out) {
    BNN_TRY(require_sm100());
    if (!net || !out || batch == 0 || depth < 2 || depth > 8)
        return fail(BNN_E_CONFIG, "pipe: need a network, batch > 0 and 2 <= depth <= 8");
    auto p = std::make_unique<bnn_pipe>();
    p->net = net, p->batch = batch, p->depth = depth;
    p->nx = batch * net->in_c * net->in_h * net->in_w, p->ny = batch * net->logits;
    auto build = [&]() -> int {
        BNN_CUDA(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
        BNN_CUDA(cudaStreamCreateWithFlags(&p->s_run, cudaStreamNonBlocking));
        BNN_CUDA(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
        for (int k = 0; k < depth; ++k) {
            float *x = nullptr, *y = nullptr;
            BNN_CUDA(cudaMalloc(&x, p->nx * 4));
            p->dx.push_back(x);
            BNN_CUDA(cudaMalloc(&y, p->ny * 4));
            p->dy.push_back(y);
            for (auto* evs : {&p->ev_in, &p->ev_run, &p->ev_out}) {
                cudaEvent_t e = nullptr;
                BNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                evs->push_back(e);
            }
        }
        return BNN_OK;
    };
    if (int rc = build()) {  // release whatever was created before the failure
        bnn_pipe_destroy(p.release());
        return rc;
    }
    *out = p.release();
    return BNN_OK;
}

// Enqueue one batch: x [batch, C, H, W] and logits [features, batch] are host buffers (pinned
// for asynchronous copies). Returns its sequence number in *seq. The H2D copy of `x` and the D2H
// copy into `logits` are asynchronous: the caller must not modify `x` nor read or reuse `logits`
// before bnn_pipe_wait(seq) returns, nor have more than `depth` batches outstanding.
int bnn_pipe_submit(bnn_pipe* p, const float* x, float* logits, uint64_t* seq) {
    if (!p) return fail(BNN_E_CONFIG, "pipe: null");
    const int k = int(p->submitted % uint64_t(p->depth));
    BNN_CUDA(cudaStreamWaitEvent(p->s_in, p->ev_run[k], 0));  // set k's previous forward read dx[k]
    BNN_CUDA(cudaMemcpyAsync(p->dx[k], x, p->nx * 4, cudaMemcpyHostToDevice, p->s_in));
    BNN_CUDA(cudaEventRecord(p->ev_in[k], p->s_in));
    BNN_CUDA(cudaStreamWaitEvent(p->s_run, p->ev_in[k], 0));
    BNN_CUDA(cudaStreamWaitEvent(p->s_run, p->ev_out[k], 0));  // set k's previous D2H read dy[k]
    BNN_TRY(forward(p->net, p->dx[k], p->batch, p->dy[k], p->s_run));
    BNN_CUDA(cudaEventRecord(p->ev_run[k], p->s_run));
    BNN_CUDA(cudaStreamWaitEvent(p->s_out, p->ev_run[k], 0));
    BNN_CUDA(cudaMemcpyAsync(logits, p->dy[k], p->ny * 4, cudaMemcpyDeviceToHost, p->s_out));
    BNN_CUDA(cudaEventRecord(p->ev_out[k], p->s_out));
    if (seq) *seq = p->submitted;
    ++p->submitted;
    return BNN_OK;
}

// Block until batch `seq`'s logits are in its host buffer (seq within the last `depth`).
int bnn_pipe_wait(bnn_pipe* p, uint64_t seq) {
    if (!p) return fail(BNN_E_CONFIG, "pipe: null");
    if (seq >= p->submitted || seq + uint64_t(p->depth) < p->submitted)
        return fail(BNN_E_CONFIG, "pipe: batch " + std::to_string(seq) + " is not among the last " +
                                      std::to_string(p->depth) + " submitted");
    BNN_CUDA(cudaEventSynchronize(p->ev_out[seq % uint64_t(p->depth)]));
    return BNN_OK;
}

int bnn_pipe_destroy(bnn_pipe* p) {
    if (!p) return BNN_OK;
    if (p->s_out) cudaStreamSynchronize(p->s_out);
    if (p->s_run) cudaStreamSynchronize(p->s_run);
    if (p->s_in) cudaStreamSynchronize(p->s_in);
    for (auto v : p->dx) cudaFree(v);
    for (auto v : p->dy) cudaFree(v);
    for (auto* evs : {&p->ev_in, &p->ev_run, &p->ev_out})
        for (auto e : *evs) cudaEventDestroy(e);
    for (auto s : {p->s_in, p->s_run, p->s_out})
        if (s) cudaStreamDestroy(s);
    delete p;
    return BNN_OK;
}

}  // extern "C"
