/* TEST INFRASTRUCTURE ONLY — the CPU oracle (plain-C restatement of the
 * reference hot path). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker. See bnn_oracle.h.
 *
 * Compiled with -ffp-contract=off: the one place the reference relies on a
 * fused multiply-add (affine_norm, contracted by GCC under -march=native,
 * network.cpp:160,172) is written as an explicit fmaf() here.
 */
#include "bnn_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- tensor.cpp */

/* tensor.cpp:65-71 — counter-based splitmix64 */
uint64_t orc_mix64(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* tensor.cpp:73-77 — top 24 bits scaled to [0,2) then shifted to [-1,1); exact in f32 */
float orc_unit_random(uint64_t seed, uint64_t index) {
    const uint32_t top = (uint32_t)(orc_mix64(seed, index) >> 40);
    return (float)top * 0x1.0p-23f - 1.0f;
}

/* tensor.cpp:79-96 — fill_random* are unit_random over the flat index; offset lets a
 * shard generate its slice of a larger tensor */
void orc_fill_random(size_t n, uint64_t seed, uint64_t offset, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_unit_random(seed, offset + i);
}

/* tensor.cpp:46-63 */
int orc_output_dims(const uint64_t g[8], size_t in_h, size_t in_w, size_t* out_h, size_t* out_w) {
    const size_t in[2] = {in_h, in_w};
    const char* axis[2] = {"height", "width"};
    size_t out[2];
    for (int a = 0; a < 2; ++a) {
        const size_t k = g[a], s = g[2 + a], p = g[4 + a];
        const size_t padded = in[a] + 2 * p;
        if (padded < k) {
            snprintf(g_err, sizeof g_err, "kernel larger than padded input along %s", axis[a]);
            return 1;
        }
        if ((padded - k) % s != 0) {
            snprintf(g_err, sizeof g_err, "output %s is not integral", axis[a]);
            return 1;
        }
        out[a] = (padded - k) / s + 1;
    }
    *out_h = out[0];
    *out_w = out[1];
    return 0;
}

/* -------------------------------------------------------------- binarize.cpp */

/* binarize.cpp:9,19-27 — v >= 0 -> +1 (so -0.0 -> +1, NaN -> -1) */
static inline float sign1(float v) { return v >= 0.0f ? 1.0f : -1.0f; }
/* binarize.cpp:10,29-37 */
static inline float clamp1(float v) { return v > 1.0f ? 1.0f : (v < -1.0f ? -1.0f : v); }

void orc_sign(const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = sign1(x[i]);
}

void orc_htanh(const float* x, size_t n, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = clamp1(x[i]);
}

/* tensor.cpp:32-44 — words per line = ceil(extent / 32) */
size_t orc_words_per_line(size_t extent) { return (extent + 31) / 32; }

/* binarize.cpp:39-73 — pack_rows: line i = row i, bit j; pack_cols: line j = column j,
 * bit r. Bit 1 = +1, LSB-first, pad bits stay 0. The first non-±1 entry in row-major
 * order raises EncodingError (binarize.cpp:12-15). */
int orc_pack(const float* x, size_t rows, size_t cols, int orientation, int apply_sign,
             uint32_t* out, size_t* bad_r, size_t* bad_c) {
    const size_t extent = orientation == 0 ? cols : rows;
    const size_t lines = orientation == 0 ? rows : cols;
    const size_t wpl = orc_words_per_line(extent);
    memset(out, 0, lines * wpl * sizeof(uint32_t));
    for (size_t r = 0; r < rows; ++r) {
        for (size_t c = 0; c < cols; ++c) {
            float v = x[r * cols + c];
            if (apply_sign) v = sign1(v);
            if (v == 1.0f) {
                const size_t line = orientation == 0 ? r : c;
                const size_t bit = orientation == 0 ? c : r;
                out[line * wpl + (bit >> 5)] |= 1u << (bit & 31u);
            } else if (v != -1.0f) {
                if (bad_r) *bad_r = r;
                if (bad_c) *bad_c = c;
                snprintf(g_err, sizeof g_err, "pack: entry at (%zu,%zu) is %f, expected -1 or +1",
                         r, c, (double)v);
                return 2;
            }
        }
    }
    return 0;
}

/* binarize.cpp:75-90 */
void orc_unpack(const uint32_t* words, size_t rows, size_t cols, int orientation, float* out) {
    const size_t extent = orientation == 0 ? cols : rows;
    const size_t wpl = orc_words_per_line(extent);
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) {
            const size_t line = orientation == 0 ? r : c;
            const size_t bit = orientation == 0 ? c : r;
            out[r * cols + c] = ((words[line * wpl + (bit >> 5)] >> (bit & 31u)) & 1u) ? 1.0f : -1.0f;
        }
}

/* --------------------------------------------------------------- kernels.cpp */

static inline int popc32(uint32_t v) { return __builtin_popcount(v); }

/* kernels.cpp:53-88 — out[i,j] = 2*sum_k popc(~(w_ik ^ x_jk)) - (32*wpl + pad) */
int orc_xnor_gemm(const uint32_t* w, size_t m, const uint32_t* x, size_t n, size_t inner_len,
                  int32_t* out) {
    const size_t wpl = orc_words_per_line(inner_len);
    if (wpl * 32 > (1u << 26)) {
        snprintf(g_err, sizeof g_err, "xnor_gemm: reduction length exceeds the accumulator guard");
        return 1;
    }
    const int32_t correction = (int32_t)(wpl * 32) + (int32_t)(wpl * 32 - inner_len);
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            uint32_t agree = 0;
            for (size_t k = 0; k < wpl; ++k) agree += (uint32_t)popc32(~(w[i * wpl + k] ^ x[j * wpl + k]));
            out[i * n + j] = (int32_t)(2 * agree) - correction;
        }
    return 0;
}

/* -------------------------------------------------------------- lowering.cpp */

/* lowering.cpp:7-43 — [C*kH*kW, oh*ow]; row r = (c*kH+kh)*kW+kw, col j = oh*outW+ow,
 * 0.0 outside the input */
int orc_im2col(const float* x, size_t b, size_t c, size_t h, size_t w, size_t bi,
               const uint64_t g[8], float* out) {
    size_t oh, ow;
    if (g[6] != c) {
        snprintf(g_err, sizeof g_err, "im2col: input has %zu channels, geometry expects %zu", c,
                 (size_t)g[6]);
        return 1;
    }
    if (bi >= b) {
        snprintf(g_err, sizeof g_err, "im2col: batch index out of range");
        return 1;
    }
    if (orc_output_dims(g, h, w, &oh, &ow)) return 1;
    const size_t kh_n = g[0], kw_n = g[1], sh = g[2], sw = g[3], ph = g[4], pw = g[5];
    const size_t ncol = oh * ow;
    for (size_t ci = 0; ci < c; ++ci)
        for (size_t kh = 0; kh < kh_n; ++kh)
            for (size_t kw = 0; kw < kw_n; ++kw) {
                const size_t r = (ci * kh_n + kh) * kw_n + kw;
                for (size_t oy = 0; oy < oh; ++oy) {
                    const long iy = (long)(oy * sh + kh) - (long)ph;
                    for (size_t ox = 0; ox < ow; ++ox) {
                        const long ix = (long)(ox * sw + kw) - (long)pw;
                        const int inside = iy >= 0 && iy < (long)h && ix >= 0 && ix < (long)w;
                        out[r * ncol + oy * ow + ox] =
                            inside ? x[((bi * c + ci) * h + (size_t)iy) * w + (size_t)ix] : 0.0f;
                    }
                }
            }
    return 0;
}

/* --------------------------------------------------------------- network.cpp */

/* network.cpp:65-79 — per image: pack_cols(sign(im2col)) -> xnor_gemm -> to_float ->
 * bias_add -> reshape_output into slot b (kernels.cpp:90-107, lowering.cpp:87-95) */
int orc_conv_forward_binary(const float* x, size_t b, size_t c, size_t h, size_t w,
                            const uint32_t* packed_w, const float* bias, const uint64_t g[8],
                            float* out) {
    size_t oh, ow;
    if (orc_output_dims(g, h, w, &oh, &ow)) return 1;
    const size_t kk = g[0] * g[1] * g[6], d = g[7], ncol = oh * ow;
    const size_t wpl = orc_words_per_line(kk);
    float* col = malloc(kk * ncol * sizeof(float));
    uint32_t* packed = malloc(ncol * wpl * sizeof(uint32_t));
    int32_t* acc = malloc(d * ncol * sizeof(int32_t));
    int rc = 0;
    for (size_t bi = 0; bi < b && rc == 0; ++bi) {
        rc = orc_im2col(x, b, c, h, w, bi, g, col);
        if (rc) break;
        orc_pack(col, kk, ncol, 1, 1, packed, NULL, NULL);
        rc = orc_xnor_gemm(packed_w, d, packed, ncol, kk, acc);
        for (size_t di = 0; di < d; ++di)
            for (size_t j = 0; j < ncol; ++j)
                out[(bi * d + di) * ncol + j] = (float)acc[di * ncol + j] + bias[di];
    }
    free(col);
    free(packed);
    free(acc);
    return rc;
}

/* network.cpp:121-126 — x [K, N] -> pack_cols(sign(x)) -> xnor_gemm -> +bias -> [M, N] */
int orc_linear_forward_packed(const float* x, size_t k, size_t n, const uint32_t* packed_w,
                              size_t m, const float* bias, float* out) {
    const size_t wpl = orc_words_per_line(k);
    uint32_t* px = malloc(n * wpl * sizeof(uint32_t));
    int32_t* acc = malloc(m * n * sizeof(int32_t));
    orc_pack(x, k, n, 1, 1, px, NULL, NULL);
    int rc = orc_xnor_gemm(packed_w, m, px, n, k, acc);
    for (size_t i = 0; i < m * n && rc == 0; ++i) out[i] = (float)acc[i] + bias[i / n];
    free(px);
    free(acc);
    return rc;
}

/* network.cpp:133-149 — 2x2 stride-2, max(max(a,b), max(c,d)) */
static inline float fmax_ref(float a, float b) { return a < b ? b : a; } /* std::max */
int orc_maxpool2(const float* x, size_t b, size_t c, size_t h, size_t w, float* out) {
    if (h % 2 || w % 2) {
        snprintf(g_err, sizeof g_err, "maxpool2: spatial extents must be even, got %zux%zu", h, w);
        return 1;
    }
    const size_t oh = h / 2, ow = w / 2;
    for (size_t p = 0; p < b * c; ++p)
        for (size_t y = 0; y < oh; ++y)
            for (size_t xx = 0; xx < ow; ++xx) {
                const float* s = x + p * h * w;
                const float a = s[(2 * y) * w + 2 * xx], bb = s[(2 * y) * w + 2 * xx + 1];
                const float cc = s[(2 * y + 1) * w + 2 * xx], dd = s[(2 * y + 1) * w + 2 * xx + 1];
                out[p * oh * ow + y * ow + xx] = fmax_ref(fmax_ref(a, bb), fmax_ref(cc, dd));
            }
    return 0;
}

/* network.cpp:151-165 — y = s*x + t per channel; GCC contracts to one FMA */
void orc_affine_tensor(const float* x, size_t b, size_t c, size_t plane, const float* scale,
                       const float* shift, float* out) {
    for (size_t bi = 0; bi < b; ++bi)
        for (size_t ci = 0; ci < c; ++ci)
            for (size_t i = 0; i < plane; ++i) {
                const size_t at = (bi * c + ci) * plane + i;
                out[at] = fmaf(scale[ci], x[at], shift[ci]);
            }
}

/* network.cpp:167-175 — per row feature */
void orc_affine_matrix(const float* x, size_t rows, size_t cols, const float* scale,
                       const float* shift, float* out) {
    for (size_t r = 0; r < rows; ++r)
        for (size_t j = 0; j < cols; ++j) out[r * cols + j] = fmaf(scale[r], x[r * cols + j], shift[r]);
}

/* bench.cpp:23-33 — FNV-1a over the little-endian bytes of each float */
uint64_t orc_fnv1a(const float* x, size_t n) {
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < n; ++i) {
        uint32_t bits;
        memcpy(&bits, &x[i], 4);
        for (int k = 0; k < 4; ++k) {
            h ^= (bits >> (8 * k)) & 0xFF;
            h *= 1099511628211ull;
        }
    }
    return h;
}

/* ------------------------------------------------------------------ networks */

/* network.cpp:422-465 — VGG-small: conv128, conv128+pool, conv256, conv256+pool,
 * conv512, conv512+pool, fc1024, fc1024, fc10; affine -> htanh -> sign between */
size_t orc_default_spec(orc_layer_spec* out, size_t cap) {
    orc_layer_spec l[64];
    size_t n = 0;
    const uint64_t convs[6] = {128, 128, 256, 256, 512, 512};
    memset(l, 0, sizeof l);
    for (int i = 0; i < 6; ++i) {
        l[n].kind = ORC_CONV;
        l[n].out_channels = convs[i];
        l[n].kernel_h = l[n].kernel_w = 3;
        l[n].stride_h = l[n].stride_w = 1;
        l[n].pad_h = l[n].pad_w = 1;
        ++n;
        if (i % 2 == 1) l[n++].kind = ORC_MAXPOOL;
        l[n++].kind = ORC_AFFINE;
        l[n++].kind = ORC_HTANH;
        l[n++].kind = ORC_SIGN;
    }
    const uint64_t fcs[3] = {1024, 1024, 10};
    for (int i = 0; i < 3; ++i) {
        l[n].kind = ORC_LINEAR;
        l[n].out_features = fcs[i];
        ++n;
        if (i < 2) {
            l[n++].kind = ORC_AFFINE;
            l[n++].kind = ORC_HTANH;
            l[n++].kind = ORC_SIGN;
        }
    }
    for (size_t i = 0; i < n && i < cap; ++i) {
        out[i] = l[i];
        if (out[i].stride_h == 0) out[i].stride_h = out[i].stride_w = 1;
    }
    return n;
}

typedef struct {
    orc_layer_spec spec;
    uint64_t geom[8];
    size_t in_features, out_features;
    size_t rows, cols, wpl; /* packed weights */
    uint32_t* packed;
    float *bias, *scale, *shift;
    size_t n_affine;
    size_t out_c, out_h, out_w;
    int out_flat;
} orc_layer;

typedef struct {
    size_t n;
    orc_layer* layers;
    size_t in_c, in_h, in_w, logits;
} orc_net;

static float* rand_vec(size_t n, uint64_t seed) {
    float* v = malloc(n * sizeof(float));
    orc_fill_random(n, seed, 0, v);
    return v;
}

/* network.cpp:203-306 — shape chain and deterministic parameters. base =
 * spec.seed ? *seed : mix64(net seed, layer index); weights mix64(base,1) (then
 * sign if binarize_weights), packed = pack_rows(sign(weights)); bias mix64(base,2);
 * affine scale 1 + 0.5*u with mix64(base,3), shift mix64(base,4). */
void* orc_net_build(const orc_layer_spec* specs, size_t n_layers, size_t in_c, size_t in_h,
                    size_t in_w, uint64_t seed, int binarize) {
    orc_net* net = calloc(1, sizeof(orc_net));
    net->n = n_layers;
    net->layers = calloc(n_layers, sizeof(orc_layer));
    net->in_c = in_c;
    net->in_h = in_h;
    net->in_w = in_w;
    size_t ch = in_c, hh = in_h, ww = in_w;
    int flat = 0;
    for (size_t i = 0; i < n_layers; ++i) {
        orc_layer* L = &net->layers[i];
        L->spec = specs[i];
        const uint64_t base = specs[i].has_seed ? specs[i].seed : orc_mix64(seed, i);
        switch (specs[i].kind) {
            case ORC_CONV: {
                const uint64_t g[8] = {specs[i].kernel_h, specs[i].kernel_w, specs[i].stride_h,
                                       specs[i].stride_w, specs[i].pad_h,    specs[i].pad_w,
                                       ch,                specs[i].out_channels};
                memcpy(L->geom, g, sizeof g);
                size_t oh, ow;
                if (flat || orc_output_dims(g, hh, ww, &oh, &ow)) {
                    snprintf(g_err, sizeof g_err, "layer %zu (conv): bad shape chain", i);
                    orc_net_free(net);
                    return NULL;
                }
                L->rows = specs[i].out_channels;
                L->cols = ch * g[0] * g[1];
                float* w = rand_vec(L->rows * L->cols, orc_mix64(base, 1));
                /* flatten_weights is the identity on [D, C, kH, kW] storage (lowering.cpp:97-102) */
                L->wpl = orc_words_per_line(L->cols);
                L->packed = malloc(L->rows * L->wpl * sizeof(uint32_t));
                orc_pack(w, L->rows, L->cols, 0, 1, L->packed, NULL, NULL);
                free(w);
                L->bias = rand_vec(L->rows, orc_mix64(base, 2));
                ch = specs[i].out_channels;
                hh = oh;
                ww = ow;
                break;
            }
            case ORC_LINEAR: {
                L->in_features = flat ? ch : ch * hh * ww;
                L->out_features = specs[i].out_features;
                L->rows = L->out_features;
                L->cols = L->in_features;
                float* w = rand_vec(L->rows * L->cols, orc_mix64(base, 1));
                L->wpl = orc_words_per_line(L->cols);
                L->packed = malloc(L->rows * L->wpl * sizeof(uint32_t));
                orc_pack(w, L->rows, L->cols, 0, 1, L->packed, NULL, NULL);
                free(w);
                L->bias = rand_vec(L->rows, orc_mix64(base, 2));
                ch = L->out_features;
                hh = ww = 0;
                flat = 1;
                break;
            }
            case ORC_MAXPOOL:
                if (flat || hh % 2 || ww % 2) {
                    snprintf(g_err, sizeof g_err, "layer %zu (maxpool): bad shape chain", i);
                    orc_net_free(net);
                    return NULL;
                }
                hh /= 2;
                ww /= 2;
                break;
            case ORC_AFFINE: {
                L->n_affine = ch;
                L->scale = rand_vec(ch, orc_mix64(base, 3));
                for (size_t k = 0; k < ch; ++k) L->scale[k] = 1.0f + 0.5f * L->scale[k];
                L->shift = rand_vec(ch, orc_mix64(base, 4));
                break;
            }
            default:
                break;
        }
        (void)binarize; /* sign(sign(w)) == sign(w): binarize_weights leaves packed bits unchanged */
        L->out_c = ch;
        L->out_h = hh;
        L->out_w = ww;
        L->out_flat = flat;
    }
    net->logits = flat ? ch : ch * hh * ww;
    return net;
}

void orc_net_free(void* h) {
    orc_net* net = h;
    if (!net) return;
    for (size_t i = 0; i < net->n; ++i) {
        free(net->layers[i].packed);
        free(net->layers[i].bias);
        free(net->layers[i].scale);
        free(net->layers[i].shift);
    }
    free(net->layers);
    free(net);
}

size_t orc_net_logits(void* h) { return ((orc_net*)h)->logits; }

size_t orc_net_layer_params(void* h, size_t i, uint32_t* packed, float* bias, float* scale,
                            float* shift) {
    orc_layer* L = &((orc_net*)h)->layers[i];
    if (packed && L->packed) memcpy(packed, L->packed, L->rows * L->wpl * sizeof(uint32_t));
    if (bias && L->bias) memcpy(bias, L->bias, L->rows * sizeof(float));
    if (scale && L->scale) memcpy(scale, L->scale, L->n_affine * sizeof(float));
    if (shift && L->shift) memcpy(shift, L->shift, L->n_affine * sizeof(float));
    return L->packed ? L->rows * L->wpl : 0;
}

/* network.cpp:330-420, ExecKernel::Binary. Tensor values are NCHW; once flat the value
 * is a [features, batch] matrix (flatten_to_columns, network.cpp:177-184). */
int orc_net_forward(void* h, const float* x, size_t batch, float* logits) {
    orc_net* net = h;
    size_t c = net->in_c, hh = net->in_h, ww = net->in_w;
    int flat = 0;
    size_t cur_n = batch * c * hh * ww;
    float* cur = malloc(cur_n * sizeof(float));
    memcpy(cur, x, cur_n * sizeof(float));
    int rc = 0;
    for (size_t i = 0; i < net->n && rc == 0; ++i) {
        orc_layer* L = &net->layers[i];
        switch (L->spec.kind) {
            case ORC_CONV: {
                const size_t n_out = batch * L->out_c * L->out_h * L->out_w;
                float* y = malloc(n_out * sizeof(float));
                rc = orc_conv_forward_binary(cur, batch, c, hh, ww, L->packed, L->bias, L->geom, y);
                free(cur);
                cur = y;
                cur_n = n_out;
                break;
            }
            case ORC_LINEAR: {
                if (!flat) { /* [B, F] -> [F, B] */
                    const size_t f = c * hh * ww;
                    float* m = malloc(cur_n * sizeof(float));
                    for (size_t b = 0; b < batch; ++b)
                        for (size_t k = 0; k < f; ++k) m[k * batch + b] = cur[b * f + k];
                    free(cur);
                    cur = m;
                    flat = 1;
                }
                float* y = malloc(L->rows * batch * sizeof(float));
                rc = orc_linear_forward_packed(cur, L->cols, batch, L->packed, L->rows, L->bias, y);
                free(cur);
                cur = y;
                cur_n = L->rows * batch;
                break;
            }
            case ORC_MAXPOOL: {
                float* y = malloc(cur_n / 4 * sizeof(float));
                rc = orc_maxpool2(cur, batch, c, hh, ww, y);
                free(cur);
                cur = y;
                cur_n /= 4;
                break;
            }
            case ORC_AFFINE:
                if (flat)
                    orc_affine_matrix(cur, c, batch, L->scale, L->shift, cur);
                else
                    orc_affine_tensor(cur, batch, c, hh * ww, L->scale, L->shift, cur);
                break;
            case ORC_SIGN:
                orc_sign(cur, cur_n, cur);
                break;
            case ORC_HTANH:
                orc_htanh(cur, cur_n, cur);
                break;
        }
        c = L->out_c;
        hh = L->out_h;
        ww = L->out_w;
    }
    if (rc == 0) {
        if (!flat) { /* flatten_to_columns of the final tensor */
            const size_t f = c * hh * ww;
            for (size_t b = 0; b < batch; ++b)
                for (size_t k = 0; k < f; ++k) logits[k * batch + b] = cur[b * f + k];
        } else {
            memcpy(logits, cur, cur_n * sizeof(float));
        }
    }
    free(cur);
    return rc;
}
