/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product.
 *
 * Plain-C restatement of the reference's binarized-layer hot path
 * (/root/reference/proj, C++20 "bnncore"). Each function cites the reference
 * file:line it restates. Pinned against the compiled reference (oracle/_ref)
 * and the reference's own known-answer tests in tests/test_oracle.py.
 *
 * Layouts are the reference's: row-major float matrices, NCHW tensors, packed
 * lines of ceil(extent/32) LSB-first 32-bit words with zero pad bits
 * (tensor.hpp:63-98).
 */
#ifndef BNN_ORACLE_H
#define BNN_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* layer kinds, network.hpp:15 order */
enum { ORC_CONV = 0, ORC_LINEAR = 1, ORC_MAXPOOL = 2, ORC_AFFINE = 3, ORC_SIGN = 4, ORC_HTANH = 5 };

typedef struct {
    uint32_t kind;
    uint32_t has_seed;
    uint64_t seed;
    uint64_t out_channels, kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w;
    uint64_t out_features;
} orc_layer_spec;

const char* orc_last_error(void);

uint64_t orc_mix64(uint64_t seed, uint64_t counter);
float orc_unit_random(uint64_t seed, uint64_t index);
void orc_fill_random(size_t n, uint64_t seed, uint64_t offset, float* out);

void orc_sign(const float* x, size_t n, float* out);
void orc_htanh(const float* x, size_t n, float* out);
size_t orc_words_per_line(size_t extent);
/* orientation 0 = pack_rows ([rows, cols] -> rows lines), 1 = pack_cols (cols lines).
 * Returns 0, or 2 (EncodingError) with *bad_r/*bad_c = first offending entry. */
int orc_pack(const float* x, size_t rows, size_t cols, int orientation, int apply_sign,
             uint32_t* out, size_t* bad_r, size_t* bad_c);
void orc_unpack(const uint32_t* words, size_t rows, size_t cols, int orientation, float* out);
int orc_xnor_gemm(const uint32_t* w, size_t m, const uint32_t* x, size_t n, size_t inner_len,
                  int32_t* out);

/* geom = {kH, kW, sH, sW, pH, pW, C, D} (ConvGeometry field order, tensor.hpp:101-111) */
int orc_output_dims(const uint64_t geom[8], size_t in_h, size_t in_w, size_t* out_h, size_t* out_w);
int orc_im2col(const float* x, size_t b, size_t c, size_t h, size_t w, size_t batch_index,
               const uint64_t geom[8], float* out);
int orc_conv_forward_binary(const float* x, size_t b, size_t c, size_t h, size_t w,
                            const uint32_t* packed_w, const float* bias, const uint64_t geom[8],
                            float* out);
int orc_linear_forward_packed(const float* x, size_t k, size_t n, const uint32_t* packed_w,
                              size_t m, const float* bias, float* out);
int orc_maxpool2(const float* x, size_t b, size_t c, size_t h, size_t w, float* out);
void orc_affine_tensor(const float* x, size_t b, size_t c, size_t plane, const float* scale,
                       const float* shift, float* out);
void orc_affine_matrix(const float* x, size_t rows, size_t cols, const float* scale,
                       const float* shift, float* out);
uint64_t orc_fnv1a(const float* x, size_t n);

/* networks (network.cpp:203-420, Binary execution only) */
size_t orc_default_spec(orc_layer_spec* out, size_t cap); /* build_default_network */
void* orc_net_build(const orc_layer_spec* layers, size_t n_layers, size_t in_c, size_t in_h,
                    size_t in_w, uint64_t seed, int binarize_weights);
void orc_net_free(void* net);
size_t orc_net_logits(void* net);
/* packed words / bias / scale / shift of layer i (NULL to skip); returns words count */
size_t orc_net_layer_params(void* net, size_t i, uint32_t* packed, float* bias, float* scale,
                            float* shift);
/* x: [batch, C, H, W] -> logits [features, batch] */
int orc_net_forward(void* net, const float* x, size_t batch, float* logits);

#ifdef __cplusplus
}
#endif
#endif
