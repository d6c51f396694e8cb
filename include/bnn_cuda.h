/* bnn_cuda.h — C ABI of the B200 (sm_100a) binarized-layer hot path.
 *
 * This is the drop-in boundary for the reference's operator API (namespace bnn,
 * static lib bnncore, /root/reference/proj). Every entry point names the reference
 * declaration it replaces. Two families:
 *
 *   bnn_*        device pointers, stream-ordered (enqueue only; no host sync unless
 *                the function says so). Used by the network engine and the benchmark.
 *   bnn_host_*   host pointers with the reference's exact semantics: H2D copy, kernel,
 *                D2H copy, synchronous. include/bnn_b200.hpp re-exposes these under the
 *                reference C++ signatures.
 *
 * Conventions
 *   - Packed bit matrices are the reference layout (tensor.hpp:63-98): `lines` lines of
 *     `ld_words` uint32 words; logical index 32k+b of a line is bit b (LSB first) of word
 *     k; bit 1 = +1, bit 0 = -1; pad bits past the logical extent are 0. The reference
 *     stores lines densely (ld_words == ceil(extent/32)); the device entry points accept
 *     any ld_words >= ceil(extent/32).
 *   - Return value: BNN_OK (0) or a bnn_status code; bnn_last_error() returns the
 *     thread-local message, which reproduces the reference exception text where the
 *     reference throws (ShapeError / EncodingError / ConfigError).
 *   - The library never frees caller memory. Scratch space is taken from the CUDA
 *     stream-ordered allocator on the caller's stream.
 *   - There is no CPU fallback: every compute entry point runs on the GPU or fails with
 *     BNN_E_CUDA.
 */
#ifndef BNN_CUDA_H
#define BNN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the C ABI is the library's export surface */
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* bnn_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    BNN_OK = 0,
    BNN_E_SHAPE = 1,    /* reference ShapeError   (tensor.hpp:11-13) */
    BNN_E_ENCODING = 2, /* reference EncodingError (tensor.hpp:15-17) */
    BNN_E_CONFIG = 3,   /* reference ConfigError  (tensor.hpp:19-21) */
    BNN_E_CUDA = 4,     /* CUDA runtime / launch failure, or no sm_100 device */
    BNN_E_IO = 5        /* reference IoError      (tensor.hpp:23-25) */
} bnn_status;

const char* bnn_last_error(void);
int bnn_version(void);
/* Name of the kernel variant the last GEMM call on this thread dispatched to
 * ("popc", "xnor4_kernel", ...); for tests and the benchmark. */
const char* bnn_last_gemm_kernel(void);
/* K3 kernel selection (process-wide). AUTO picks the integer-pipe kernel below ~2^26
 * bit-MACs, the tcgen05 FP4 tensor-core kernel with operands expanded from the packed bits in
 * shared memory up to ~2^32, and above that the FP4 kernel fed by TMA from operands expanded
 * once to e2m1 in HBM scratch ("K3 candidates"); POPC / UMMA / UMMA_TMA force one of
 * them (used by the parity tests to cover all three). */
enum { BNN_GEMM_AUTO = 0, BNN_GEMM_POPC = 1, BNN_GEMM_UMMA = 2, BNN_GEMM_UMMA_TMA = 3 };
int bnn_set_gemm_policy(int policy);

/* ConvGeometry (tensor.hpp:101-111), same field order. */
typedef struct {
    uint64_t kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w, in_channels, out_channels;
} bnn_conv_geom;

/* PackedBitMatrix::make (tensor.cpp:32-44): words per line for a packed extent. */
size_t bnn_words_per_line(size_t extent);
/* output_dims (tensor.cpp:46-63). BNN_E_SHAPE names the failing axis ("height"/"width"). */
int bnn_output_dims(const bnn_conv_geom* g, size_t in_h, size_t in_w, size_t* out_h, size_t* out_w);

/* ------------------------------------------------------------------ K1: encoder
 * pack_cols(sign(x)) (binarize.cpp:55-73 after binarize.cpp:24-27): x is row-major [L, N];
 * line j (column j) gets bit r = (x[r, j] >= 0). words: N lines x ld_words. */
int bnn_sign_pack_cols_f32(const float* x, size_t L, size_t N, uint32_t* words, size_t ld_words,
                           bnn_stream_t s);
/* pack_rows(sign(x)) (binarize.cpp:39-53): x is row-major [D, L]; line i = row i. */
int bnn_sign_pack_rows_f32(const float* x, size_t D, size_t L, uint32_t* words, size_t ld_words,
                           bnn_stream_t s);
/* Strict pack_cols / pack_rows of an already-binarized matrix: entries must be exactly
 * +-1. *first_bad_dev (device int64, caller-initialised to INT64_MAX) receives the smallest
 * row-major index r*cols+c of a non-+-1 entry (atomicMin), which is the entry the reference
 * reports first (binarize.cpp:12-15). Stream-ordered; the caller checks the flag. */
int bnn_pack_cols_f32(const float* x, size_t L, size_t N, uint32_t* words, size_t ld_words,
                      int64_t* first_bad_dev, bnn_stream_t s);
int bnn_pack_rows_f32(const float* x, size_t D, size_t L, uint32_t* words, size_t ld_words,
                      int64_t* first_bad_dev, bnn_stream_t s);
/* unpack (binarize.cpp:75-90); orientation 0 = row-packed [rows, cols], 1 = col-packed. */
int bnn_unpack_f32(const uint32_t* words, size_t ld_words, size_t rows, size_t cols,
                   int orientation, float* out, bnn_stream_t s);

/* --------------------------------------------------------------- K2: binary im2col
 * pack_cols(sign(im2col(x, b, g))) for every image b at once (network.cpp:72,
 * lowering.cpp:7-43): x is [B, C, H, W]; line n = b*oh*ow + oy*ow + ox, bit
 * r = (c*kH + kh)*kW + kw. Spatial zero padding encodes as bit 1 (sign(0) = +1). */
int bnn_im2col_sign_pack_f32(const float* x, size_t B, size_t C, size_t H, size_t W,
                             const bnn_conv_geom* g, uint32_t* words, size_t ld_words,
                             bnn_stream_t s);

/* ------------------------------------------------------------ K3: xnor-popcount GEMM
 * xnor_gemm (kernels.cpp:53-88): w row-packed M lines, x col-packed N lines, both with
 * ceil(L/32) significant words and zero pad bits. out[i*ldo + j] = L - 2*sum_k popc(w^x),
 * identical to the reference's 2*sum popc(~(w^x)) - 32*wpl - pad. Rejects 32*wpl > 2^26
 * like the reference (kernels.cpp:66-68). */
int bnn_xnor_gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M,
                      size_t N, size_t L, int32_t* out, size_t ldo, bnn_stream_t s);
/* Fused epilogue: to_float + bias_add (kernels.cpp:90-107) + reshape_output
 * (lowering.cpp:87-95). Column j = (img, p) with img = j / P, p = j % P is written to
 * out[img*M*P + i*P + p]; P = N gives the row-major [M, N] linear layout, P = oh*ow the
 * [B, D, oh, ow] conv layout. bias may be NULL (zero). */
int bnn_xnor_gemm_bias_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx,
                           size_t M, size_t N, size_t L, const float* bias, size_t P, float* out,
                           bnn_stream_t s);

/* -------------------------------------------------------------- layer forwards
 * conv_forward_binary (network.cpp:65-79): x [B, C, H, W] -> out [B, D, oh, ow].
 * packed_w: D lines x ldw words of pack_rows(sign(flatten_weights(W))). */
int bnn_conv_forward_binary_f32(const float* x, size_t B, size_t C, size_t H, size_t W,
                                const uint32_t* packed_w, size_t ldw, const float* bias,
                                const bnn_conv_geom* g, float* out, bnn_stream_t s);
/* linear_forward_packed (network.cpp:121-126): x [K, N] (features x batch) -> out [M, N]. */
int bnn_linear_forward_packed_f32(const float* x, size_t K, size_t N, const uint32_t* packed_w,
                                  size_t ldw, size_t M, const float* bias, float* out,
                                  bnn_stream_t s);

/* -------------------------------------------------------------- K4: glue ops */
int bnn_sign_f32(const float* x, size_t n, float* out, bnn_stream_t s);  /* binarize.cpp:24 */
int bnn_htanh_f32(const float* x, size_t n, float* out, bnn_stream_t s); /* binarize.cpp:34 */
/* maxpool2 (network.cpp:133-149), x [B, C, H, W] with even H, W. */
int bnn_maxpool2_f32(const float* x, size_t B, size_t C, size_t H, size_t W, float* out,
                     bnn_stream_t s);
/* affine_norm (network.cpp:151-175): out = fmaf(scale[ch], x, shift[ch]) where
 * ch = (i / plane) % channels. Tensor form: plane = H*W, channels = C. Matrix form
 * ([features, batch]): plane = batch, channels = features. */
int bnn_affine_f32(const float* x, size_t n, size_t channels, size_t plane, const float* scale,
                   const float* shift, float* out, bnn_stream_t s);
/* to_float (kernels.cpp:90-95): out[i] = (float)a[i]. */
int bnn_to_float_s32(const int32_t* a, size_t n, float* out, bnn_stream_t s);
/* bias_add (kernels.cpp:97-107), in place: a[d*cols + j] += bias[d]. */
int bnn_bias_add_f32(float* a, size_t rows, size_t cols, const float* bias, bnn_stream_t s);
/* flatten_to_columns (network.cpp:177-184): [B, F] -> [F, B]. */
int bnn_flatten_to_columns_f32(const float* x, size_t B, size_t F, float* out, bnn_stream_t s);
/* fill_random (tensor.cpp:65-96): out[i] = unit_random(seed, offset + i). Bit-identical to
 * the CPU generator, so each shard generates its slice of a global tensor. */
int bnn_fill_random_f32(uint64_t seed, uint64_t offset, size_t n, float* out, bnn_stream_t s);
uint64_t bnn_mix64(uint64_t seed, uint64_t counter); /* tensor.cpp:65-71 (host) */
/* fnv1a_hash (bench.cpp:23-33) of a device float buffer; synchronous. */
int bnn_fnv1a_f32(const float* x, size_t n, uint64_t* hash, bnn_stream_t s);
/* max_i |a[i] - b[i]| of two device arrays (verify_network's deviation, bench.cpp:178-181),
 * computed on the device; synchronous. */
int bnn_max_abs_diff_f32(const float* a, const float* b, size_t n, double* out, bnn_stream_t s);

/* ------------------------------------------------------------- network engine
 * build_network + network_forward, ExecKernel::Binary (network.cpp:203-420). Weights are
 * generated on the device with fill_random from the reference seeds and packed once at
 * build time; forward runs the whole graph on one stream. */
enum { BNN_LAYER_CONV = 0, BNN_LAYER_LINEAR = 1, BNN_LAYER_MAXPOOL = 2, BNN_LAYER_AFFINE = 3,
       BNN_LAYER_SIGN = 4, BNN_LAYER_HTANH = 5 }; /* LayerKind order, network.hpp:15 */

/* KernelChoice (network.hpp:16), a weighted layer's own kernel under BNN_ENGINE_PER_LAYER */
enum { BNN_KERNEL_FLOAT = 0, BNN_KERNEL_BINARY = 1, BNN_KERNEL_NAIVE = 2 };

typedef struct { /* LayerSpec (network.hpp:23-39) */
    uint32_t kind;
    uint32_t has_seed;
    uint64_t seed;
    uint64_t out_channels, kernel_h, kernel_w, stride_h, stride_w, pad_h, pad_w;
    uint64_t out_features;
    const char* weights_blob; /* tensor blob path of the float weights; NULL -> seeded weights */
    uint32_t kernel;          /* BNN_KERNEL_* (LayerSpec::kernel) */
    uint32_t reserved;
} bnn_layer_spec;

typedef struct bnn_net bnn_net;

/* build_default_network (network.cpp:422-465) into caller storage; returns layer count. */
size_t bnn_default_spec(bnn_layer_spec* out, size_t cap);
/* build_network (network.cpp:203-306) on the current CUDA device. ShapeError messages name
 * the layer ("layer N (kind): ..."). */
int bnn_net_create(const bnn_layer_spec* layers, size_t n_layers, size_t in_c, size_t in_h,
                   size_t in_w, uint64_t seed, int binarize_weights, bnn_net** out);
void bnn_net_destroy(bnn_net* net);
size_t bnn_net_logits(const bnn_net* net);
size_t bnn_net_num_layers(const bnn_net* net);
/* Copy layer i's row-packed weights (dense reference layout, rows x ceil(cols/32)) and
 * bias / affine parameters to host buffers (NULL to skip). */
int bnn_net_layer_params(const bnn_net* net, size_t i, uint32_t* packed, size_t* rows,
                         size_t* cols, float* bias, float* scale, float* shift);
/* BuiltLayer's parameters (network.hpp:57-77) to / from host buffers, NULL to skip: packed
 * [rows, ceil(cols/32)] words, float weights [rows, cols] (after binarize_weights), bias
 * [rows], affine scale / shift [channels]. Setting replaces the device copies the engines
 * use (Binary / fused: packed, bias, scale, shift; Float / BinaryReference / Naive: weights,
 * bias, scale, shift) and re-prepares the fused engine, as if the network had been built
 * with them -- the reference's test hook of perturbing net.layers[i] (test_bench.cpp:159-173).
 * Synchronous. */
int bnn_net_layer_data(const bnn_net* net, size_t i, uint32_t* packed, float* weights, float* bias,
                       float* scale, float* shift);
int bnn_net_set_layer_data(bnn_net* net, size_t i, const uint32_t* packed, const float* weights,
                           const float* bias, const float* scale, const float* shift);
/* network_forward (network.cpp:330-420): x device [B, C, H, W] -> logits device
 * [features, B] (the reference layout, network.hpp:104-105). Stream-ordered. */
int bnn_net_forward(bnn_net* net, const float* x, size_t batch, float* logits, bnn_stream_t s);
/* Per-layer CUDA-event timing, the device analogue of ForwardOptions::layer_seconds
 * (network.hpp:93-97). When enabled, bnn_net_forward records events around every layer and
 * around every GEMM launch on its stream. bnn_net_timing synchronizes on the recorded events
 * and returns the totals (ms) accumulated since the last reset; arrays have one entry per
 * layer (NULL to skip). */
int bnn_net_set_timing(bnn_net* net, int enabled);
int bnn_net_timing(bnn_net* net, double* layer_ms, double* gemm_ms, size_t* gemm_launches);
int bnn_net_reset_timing(bnn_net* net);
/* Layer i: out[0] kind, [1] GEMM M (rows of packed weights), [2] GEMM K, [3] GEMM columns per
 * image (oh*ow for conv, 1 for linear, 0 otherwise), [4..6] output C, H, W, [7] output flat. */
int bnn_net_layer_shape(const bnn_net* net, size_t i, size_t out[8]);
/* Engine selection. FUSED (fused.cu): one tcgen05 launch per weighted layer with the glue
 * (bias, maxpool, affine_norm, htanh, sign) folded into its epilogue and packed-bit NHWC
 * activations; available when the topology matches conv {[maxpool][affine][htanh][sign]
 * conv|linear}* linear (the default network does). GENERIC: one kernel per reference op.
 * AUTO (default) = FUSED when available. Both are bit-exact with the reference. */
/* BNN_ENGINE_FLOAT: the paper's float control group (ExecKernel::Float: conv_forward_float /
 * linear_forward Float on the float weights, control.cu), bit-exact with the reference's
 * FMA-contracted float_gemm. */
/* BNN_ENGINE_BINARY_REFERENCE: ExecKernel::BinaryReference, the graph verify_network checks the
 * xnor path against (sign(im2col) / sign(x) then float_gemm on sign(weights), network.cpp:81-94,
 * 128-131). BNN_ENGINE_NAIVE: ExecKernel::Naive (direct convolution, network.cpp:96-111; linear
 * layers as Float). BNN_ENGINE_PER_LAYER: ExecKernel::PerLayer, each weighted layer runs its
 * spec's KernelChoice (bnn_layer_spec.kernel); all-Binary networks use the fused engine. All of
 * them are bit-exact with the reference's network_forward under the same ExecKernel. */
enum { BNN_ENGINE_AUTO = 0, BNN_ENGINE_GENERIC = 1, BNN_ENGINE_FUSED = 2, BNN_ENGINE_FLOAT = 3,
       BNN_ENGINE_BINARY_REFERENCE = 4, BNN_ENGINE_NAIVE = 5, BNN_ENGINE_PER_LAYER = 6 };
int bnn_net_set_engine(bnn_net* net, int policy);
/* Layer i's KernelChoice (BNN_KERNEL_*) for BNN_ENGINE_PER_LAYER (LayerSpec::kernel). */
int bnn_net_set_layer_kernel(bnn_net* net, size_t i, int kernel);
/* Fused-engine tile shape override, process-wide (tests / experiments): cta_group 1 (M=128
 * per CTA) or 2 (CTA pairs, M=256, tcgen05 cta_group::2), bn = MMA N in {32,64,128,256};
 * 0 = automatic (the default). */
int bnn_set_fused_tiling(int cta_group, int bn);
/* CUDA-graph replay of the fused forward for a repeated (x, batch, logits, stream) on a
 * non-default stream (default on). The first call runs eagerly, the second captures, later
 * calls replay the graph. */
int bnn_net_set_graphs(bnn_net* net, int enabled);
/* Fused engine split-K for few, K-deep output tiles (the linear layers at small batch): 0 auto
 * (default), 1 off, or a forced power of two <= 16. Process-wide; bit-exact either way. */
int bnn_set_fused_split(int split);
/* Fused engine: conv layers with a packed-bit output use the swapped-operand kernel (output
 * channels on the tensor-core M, positions on N: full rate for 128-channel layers): 1 (default)
 * for layers of <= 128 channels, 2 for all, 0 never. Process-wide; all are bit-exact. */
int bnn_set_fused_swap(int enabled);
/* Fused engine: a final layer of <= 64 logits runs as a CUDA-core xnor-popcount kernel (1,
 * default) or on the tensor cores like the other layers (0). Bit-exact either way. */
int bnn_set_fused_small_logits(int enabled);
/* Fused engine: a pixel-input first conv whose patch fits one word (K = kh*kw*C <= 32, e.g. the
 * 3x3 RGB layer) with 32..256 output channels runs as a CUDA-core XOR-popcount kernel reading
 * the float input itself (1), after the pixel packer (2), 1 up to batch 512 and 2 above (3,
 * default), or on the tensor cores (0). Process-wide; bit-exact in every mode. */
int bnn_set_fused_pix_popc(int mode);
/* ------------------------------------------------- the float control group (control.cu)
 * float_gemm (kernels.cpp:33-51): w [M, K] x [K, N], k-ascending FMA chain per output, then
 * + bias (may be NULL) with the reshape epilogue of bnn_xnor_gemm_bias_f32 (P = 0: P = N). */
int bnn_float_gemm_f32(const float* w, size_t M, size_t K, const float* x, size_t N, const float* bias,
                       size_t P, float* out, bnn_stream_t s);
/* im2col (lowering.cpp:7-43, float, zero padding) of batch slices [b0, b0 + nb): cols
 * [C*kH*kW, nb*oh*ow]; nb = 1 is the reference's im2col(x, b0, geom). */
int bnn_im2col_f32(const float* x, size_t B, size_t C, size_t H, size_t W, size_t b0, size_t nb,
                   const bnn_conv_geom* g, float* cols, bnn_stream_t s);
/* col2im (lowering.cpp:45-84), the adjoint: m [C*kH*kW, oh*ow] -> x [1, C, in_h, in_w], with
 * the input extents recovered from the geometry (returned in *in_h / *in_w; x == NULL queries
 * them only). Bit-identical (same additions in the same order). */
int bnn_col2im_f32(const float* m, size_t rows, size_t cols, const bnn_conv_geom* g, size_t oh, size_t ow,
                   float* x, size_t* in_h, size_t* in_w, bnn_stream_t s);
/* conv_forward_naive (network.cpp:96-111, naive_conv kernels.cpp:109-147): w [D, C, kH, kW]. */
int bnn_conv_forward_naive_f32(const float* x, size_t B, size_t C, size_t H, size_t W, const float* w,
                               const float* bias, const bnn_conv_geom* g, float* out, bnn_stream_t s);
/* conv_forward_float (network.cpp:50-63). */
int bnn_conv_forward_float_f32(const float* x, size_t B, size_t C, size_t H, size_t W, const float* w_flat,
                               const float* bias, const bnn_conv_geom* g, float* out, bnn_stream_t s);

/* ------------------------------------------------------- on-disk formats (host side)
 * packed blob (binarize.cpp:116-148): orientation byte, rows and cols (u64 LE), words (u32 LE).
 * tensor blob (tensor.cpp:123-150): batch, channels, height, width (u64 LE), floats (f32 LE).
 * Loaders with a NULL output pointer return the header only. Errors: BNN_E_IO with the
 * reference's IoError messages ("packed blob size mismatch: <path>", ...). */
int bnn_save_packed_blob(const char* path, int orientation, uint64_t rows, uint64_t cols,
                         const uint32_t* words);
int bnn_load_packed_blob(const char* path, int* orientation, uint64_t* rows, uint64_t* cols,
                         uint32_t* words, size_t cap_words);
int bnn_save_tensor_blob(const char* path, const uint64_t shape[4], const float* data);
int bnn_load_tensor_blob(const char* path, uint64_t shape[4], float* data, size_t cap);
/* load_network_spec (network.cpp:487-536) + build_network: a NetworkSpec JSON file (layers
 * may name a weights_blob tensor blob). binarize_override -1 keeps the spec's flag. */
int bnn_net_create_from_spec(const char* path, int binarize_override, bnn_net** out);
int bnn_spec_info(const char* path, uint64_t input_shape[4], size_t* n_layers);

/* ------------------------------------------------------ bench / verify harness (bench.cpp)
 * run_verify (bench.cpp:193-199): the default network (spec_path NULL) or a NetworkSpec file
 * with binarize_weights forced on, input from input_blob or fill_random(batch, ...,
 * mix64(seed, "input")); Binary vs BinaryReference on the device.
 * run_benchmark (bench.cpp:102-170) + emit_report (bench.cpp:219-257): kernels_mask bit 0
 * Binary, bit 1 Float, bit 2 Naive (in that order); the report JSON is written to out_path in
 * the reference's schema. */
int bnn_run_verify(const char* spec_path, size_t batch, uint64_t seed, const char* input_blob, double* max_dev,
                   size_t* compared, int* pass, int* pad_exercised);
int bnn_run_benchmark(const char* spec_path, size_t batch, size_t iterations, size_t warmup, uint64_t seed,
                      int kernels_mask, int layer_times, const char* out_path);

/* Kernel the last fused forward ran for weighted layer `layer` ("" if none / not fused). */
const char* bnn_net_layer_kernel(const bnn_net* net, size_t layer);
/* Fused engine: FP4 operands (kind::mxf4 block-scaled e2m1, exact for +-1 x {0,1}) in the
 * swapped-operand conv kernel: 0 off, 1 (default) every conv with a packed-bit input, 2 also
 * the pixel-input first conv. Bit-exact in every mode. */
int bnn_set_fused_fp4(int mode);
/* Fused engine: the halo-tile FP4 conv (halo4_kernel) for "same" convs (3x3 pad 1, 1x1, ...,
 * stride 1) with a packed-bit input whose weights fit in shared memory: each input pixel is
 * expanded to e2m1 once per tile instead of once per tap. 0 off (fused_swap4_kernel), 1
 * (default) on, 2 also for convs whose weights do not fit (streamed through a ring of shared-
 * memory slots; slower than fused_swap4_kernel for VGG-small). Bit-exact in every mode. */
int bnn_set_fused_halo(int enabled);
/* Fused engine: the pixel-input first conv ("same" geometry, C <= 32) on the halo-tile FP4 kernel
 * with the float input signed by its producers and the channels padded to 64 (zero weights): 1
 * on, 0 (default: measured faster) the CUDA-core pix_tile / pix_popc kernels. Bit-exact either
 * way. */
int bnn_set_fused_halo0(int enabled);
/* Fused engine: linear layers on the FP4 tensor-core kernel (lin4_kernel: e2m1 weights by TMA,
 * packed input bits expanded in shared memory, K split over CTAs with an exact integer
 * reduction in lin_finish_kernel) instead of the int8 fused_layer_kernel. 0 off, 1 (default)
 * on; the images are TMA-loaded from an e2m1 copy expanded once per layer (expand_act4_kernel)
 * when many feature tiles share them (>= 4 tiles, batch >= 512), else expanded by the producer
 * warps of every CTA; 2 / 3 force one of the two. Bit-exact either way. */
int bnn_set_fused_lin4(int enabled);
/* Fused engine: FP4 swapped conv on CTA pairs (cta_group::2, 256 channels per pair: each SM
 * expands half the activation rows) for layers with >= 256 channels: 0 off, 1 (default) on.
 * Positions per tile (pairs and the 128-channel kernel): 192 or 224, whichever needs fewer
 * rounds over the SMs; modes 2 / 3 force 192 / 224 (mode 0: 192). */
int bnn_set_fused_fp4_pair(int mode);
/* Debug timeline of the fused engine's launches (globaltimer stamps per CTA; stderr):
 * op 1 = start recording, op 2 = print the recorded launches and stop. */
int bnn_debug_timeline(int op);
/* Engine the next bnn_net_forward uses (FUSED, GENERIC, FLOAT, BINARY_REFERENCE, NAIVE or
 * PER_LAYER when that mixes kernels). */
int bnn_net_engine(const bnn_net* net);
/* Number of kernels the last bnn_net_forward enqueued (the benchmark's gpu_launches). */
size_t bnn_net_last_launches(const bnn_net* net);
/* Bytes of device memory held by the engine (weights + activation arena). */
size_t bnn_net_device_bytes(const bnn_net* net);

/* ------------------------------------------------------------- pipe-peak probes
 * Microbenchmarks behind the K3 candidate choice (bops = 2 per bit-MAC), timed with CUDA
 * events on stream s at the clocks of the moment; synchronous.
 *   popc: LOP3 + POPC + IADD register tile (candidate A's inner loop without smem traffic)
 *   bmma: mma.sync m16n8k256 b1 xor.popc (candidate B; software-emulated on sm_100a) */
int bnn_probe_popc_peak(double* bops_per_s, double* ms, bnn_stream_t s);
int bnn_probe_bmma_peak(double* bops_per_s, double* ms, bnn_stream_t s);
/*   umma: tcgen05.mma dispatch rate (candidate C), kind 0 = kind::i8 (+-1 bytes), 1 = kind::mxf4
 *         (block-scaled e2m1, the fused conv kernels' operands), M = 128, N in [64, 256]; ops = 2
 *         per MAC; *cycles_per_mma = cycles per instruction on one SM. */
int bnn_probe_umma_peak(int kind, int N, double* ops_per_s, double* cycles_per_mma, bnn_stream_t s);

/* ------------------------------------------------- host-buffer (reference-exact) API
 * Same semantics as the reference functions; synchronous; internal stream. */
int bnn_host_sign_pack(const float* x, size_t rows, size_t cols, int orientation,
                       int apply_sign, uint32_t* words);
int bnn_host_xnor_gemm(const uint32_t* w, size_t M, const uint32_t* x, size_t N, size_t L,
                       int32_t* out);
int bnn_host_conv_forward_binary(const float* x, size_t B, size_t C, size_t H, size_t W,
                                 const uint32_t* packed_w, const float* bias,
                                 const bnn_conv_geom* g, float* out);
int bnn_host_linear_forward_packed(const float* x, size_t K, size_t N, const uint32_t* packed_w,
                                   size_t M, const float* bias, float* out);
int bnn_host_net_forward(bnn_net* net, const float* x, size_t batch, float* logits);

/* Serving pipeline over host buffers (the reference's network_forward per batch, run as a
 * stream of batches): each submitted batch is copied in from host memory, run through the
 * network and its logits [features, batch] copied back, on separate copy / compute streams so
 * that batch i+1's H2D and batch i-1's D2H overlap batch i's forward. Host buffers should be
 * pinned (cudaHostAlloc / torch pin_memory) for the copies to be asynchronous. At most `depth`
 * (2..8) batches may be outstanding; bnn_pipe_wait(seq) blocks until batch seq's logits are in
 * its host buffer. Both copies are asynchronous: a submitted batch's `x` must stay unchanged and
 * its `logits` untouched until bnn_pipe_wait(seq) returns. Each buffer set replays its own
 * captured CUDA graph of the forward after its first two batches. */
typedef struct bnn_pipe bnn_pipe;
int bnn_pipe_create(bnn_net* net, size_t batch, int depth, bnn_pipe** out);
int bnn_pipe_submit(bnn_pipe* p, const float* x, float* logits, uint64_t* seq);
int bnn_pipe_wait(bnn_pipe* p, uint64_t seq);
int bnn_pipe_destroy(bnn_pipe* p);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* BNN_CUDA_H */
