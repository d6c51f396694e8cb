// Fused binary layer (fused.cu): geometry block and launch entry points.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bnnk {

// activation producer input: packed NHWC bits, float NCHW (im2col in the producer), or the
// pixel-packed sign bits of a first layer with few channels (pack_pixels_kernel)
enum { FIN_BITS = 0, FIN_F32 = 1, FIN_PIX = 2 };
enum { FEPI_BITS = 0, FEPI_LOGITS = 1, FEPI_NCHW = 2 };  // epilogue output

// Division by a launch constant without the ~20-instruction integer divide: for n < 2^31,
// n / d = (umulhi(n, mul) + n) >> shift (Granlund-Montgomery, round-up multiplier).
struct FastDiv {
    uint32_t d, mul, shift;
    static FastDiv make(uint32_t d) {
        if (d == 0) d = 1;  // unused divisor
        uint32_t l = 0;
        while ((uint64_t(1) << l) < d) ++l;
        const uint64_t m = ((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1;
        return FastDiv{d, uint32_t(m), l};
    }
#ifdef __CUDACC__
    __device__ __forceinline__ int div(int n) const {
        return int((__umulhi(uint32_t(n), mul) + uint32_t(n)) >> shift);
    }
#endif
};

struct FusedGeom {
    const void* in;  // FIN_BITS: u32 [B, H, W, Cw] packed NHWC; FIN_F32: float [B, C, H, W]
    int B, H, W, C, Cw;
    int KH, KW, SH, SW, PH, PW;
    int OH, OW;
    int K;        // logical reduction length (KH*KW*C)
    int KB;       // 128-element K blocks (Kpad / 128)
    int D;        // output channels / features
    int rows;     // GEMM rows: B*OH*OW (conv) or B (linear)
    int pool;     // rows are pool-major and the epilogue takes the 2x2 max
    int n_tiles;  // ceil(D / BN)
    const int4* prm;    // [>= n_tiles*BN] (Tu, flip, S_d, bias bits): prep_params_kernel
    uint32_t* out_bits; // FEPI_BITS: [rows / (pool ? 4 : 1), Dw]
    int Dw;             // D / 32
    float* out_f32;     // FEPI_LOGITS: [D, ldo] (features x batch); FEPI_NCHW: [B, D, OH*OW]
    int ldo;
    int ksplit;               // split-K factor (1: none); S > 1 needs ws/sem, CTA-local tiles, no pool
    int* ws;                  // split-K partial sums [ksplit][ws_rows][ws_ld]
    unsigned* sem;            // split-K counters, 2 per output tile, zero between launches
    int ws_rows, ws_ld;
    unsigned long long* dbg;  // profiling counters (BNN_FUSED_PROFILE=1), else null
    int dbg_mode;             // profiling experiments (results invalid): 1 no A stores, 2 no epilogue math, 8 no wait::st
    unsigned long long* tl;   // timeline stamps (bnn_debug_timeline), [grid][4], else null
    int pdl_late;             // trigger dependent launch at the end of the CTA (else at entry)
    int kq_last;              // 32-byte K steps that carry data in the last K block (1..4)
    FastDiv dv0, dv1;         // decode_row divisors: pool (OW/2, OH/2) or (OH*OW, OW)
    int kb4, kq4;             // FP4 path: 256-element K blocks, 64-element K steps in the last
};

// Halo-tile FP4 conv (halo.cu): "same" convs with packed-bit input, weights resident in shared
// memory, activations expanded once per pixel into a padded-canvas halo tile.
constexpr int kHaloMaxSteps = 128;  // K / 64 (K <= 8192)
struct HaloGeom {
    const uint32_t* in;  // packed NHWC bits [B, H, W, Cw]
    uint32_t* out;       // packed NHWC bits [B, OH', OW', Dw] (pooled or not)
    const int4* prm;     // per-channel (Tu, flip, ...) from prep_params_kernel
    int B, H, W, Cw, D, Dw, pool;
    int G, S, Q, P;      // canvas: images per canvas row, rows per image, columns per image, pitch
    int TR, N, NH, nst;  // canvas rows per tile, MMA N, halo rows, halo stages
    int n_tiles, m_tiles, total_rows, grid;
    int steps, KB4;      // K / 64 MMA steps, 256-element weight blocks
    int wst;             // 0: weights resident in shared memory; else ring slots of streamed blocks
    size_t smem;
    FastDiv dP, dS, dQ, dNw, dG;  // dNw: pooled epilogue units (<= 32 columns) per row pair and image
    unsigned long long* tl;   // timeline stamps (bnn_debug_timeline), [grid][4], else null
    const float* in_f32;      // first layer (halo0): float NCHW input, creal channels -> bit words
    int creal;
    unsigned long long* dbg;  // BNN_HALO_PROFILE counters, else null
    int dbg_mode;             // profiling experiments (results invalid): 1 no epilogue, 2 no halo fill, 4 no MMA
    int taps, cpt;            // taps (<= 9), K64 steps per tap (C / 64)
    int toff[9];              // canvas shift of tap t, in pixels (= 16-byte halo rows)
};
bool halo4_plan(const FusedGeom& g, HaloGeom& h);
// First conv through halo4 (halo0): the float input signed per pixel by the producers, C <= 32
// channels padded to 64 per tap (zero weights). prep_w4_pix builds its e2m1 weights from the
// reference's packed rows: [Dpad, Kpad4/2], K' = KH*KW*64 tap-major.
int prep_w4_pix(const uint32_t* packed, size_t wpl, int D, int C, int KH, int KW, int Dpad, int Kpad4, uint8_t* w4,
                cudaStream_t s);
int launch_halo4(const CUtensorMap& tm4, const HaloGeom& h, cudaStream_t s);

// FP4 linear layer with split-K (linear.cu): weights [Dpad, Kpad4/2] e2m1 via tm4, input bits
// [B, Kw]; ksplit > 1 writes partial sums to ws [ksplit][B][Dpad] and the tile's slices reduce
// them in the same launch (counters sem, 2 per tile, zero between launches).
struct LinGeom {
    const uint32_t* in;
    int B, K, Kw, D, Dw, Dpad;
    int KB4, kq_last;          // 256-element K blocks, 64-element steps in the last one
    int m_tiles, n_tiles, NB;  // 128-feature tiles, image tiles of NB (UMMA N)
    int ksplit, kbs;           // K slices, K blocks per slice
    int nst;                   // smem ring stages (weights 16 KB + images NB x 128 B each)
    const int4* prm;
    int epi;                   // FEPI_BITS or FEPI_LOGITS
    uint32_t* out_bits;        // [B, Dw]
    float* out_f32;            // [D, ldo]
    int ldo;
    int* ws;
    unsigned* sem;
    unsigned long long* dbg;  // BNN_LIN4_PROFILE phase stamps, else null
    unsigned long long* tl;   // timeline stamps (bnn_debug_timeline), [grid][4], else null
    int tmab;                 // 1: images TMA-loaded from in4 (expanded once by expand_act4), no producers
    uint8_t* in4;             // [B, Kw * 16] e2m1 images when tmab
    uint8_t* out4;            // FEPI_BITS: write [B, Dw * 16] e2m1 (the next layer's in4) instead of out_bits
};
bool lin4_plan(const FusedGeom& g, int epi, LinGeom& l);
// Images [B, Kw] packed bits -> e2m1 {0, 1.0} lines [B, Kw * 16 bytes] in put_word4's order.
int launch_expand_act4(const LinGeom& l, cudaStream_t s);
// -1 auto (by size), 0 producer-expanded images, 1 TMA-loaded images (bnn_set_fused_lin4 1 / 3 / 2)
void set_lin4_tma(int mode);
size_t lin4_ws_bytes(const LinGeom& l);
size_t lin4_sem_count(const LinGeom& l);
int launch_lin4(const CUtensorMap& tm4, const CUtensorMap& tmx, const LinGeom& l, cudaStream_t s);

// Debug timeline (globaltimer stamps per CTA and launch): op 1 enable + reset, 2 print + disable.
int fused_timeline(int op);
unsigned long long* fused_timeline_slot(int slots);
void fused_timeline_name(const char* name);
// Swapped-operand conv (fused_swap_kernel): 128 channels x 256 positions per tile, bits
// epilogue, CTA-local; tm must be the weight map with box rows 128.
int launch_swap(int in_mode, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s);
// FP4 (kind::mxf4) swapped-operand conv; tm4 maps the e2m1 weights [Dpad, Kpad4/2] bytes, box
// rows 128 x 128 bytes.
int prep_weights4(const int8_t* w8, int Kpad, int K, int Dpad, int Kpad4, uint8_t* w4, cudaStream_t s);
int launch_swap4(int in_mode, const CUtensorMap& tm4, const FusedGeom& g, cudaStream_t s);
// Tiny final logits layer on the CUDA cores (logits_popc_kernel); wbits from prep_logit_bits.
int prep_logit_bits(const int8_t* w8, int Kpad, int K, int D, int Kw, uint32_t* wbits, cudaStream_t s);
int launch_logits_popc(const FusedGeom& g, const uint32_t* wbits, cudaStream_t s);
// Pixel-input first conv with K <= 32 and 32..256 output channels on the CUDA cores
// (pix_popc_kernel). PixParams (a kernel parameter: constant-bank operands): channel d's weight
// bits in the engine K order (prep_logit_bits, one word per channel), its popcount threshold
// P_d and the flip bits, from make_pix_params over host copies of wbits and the stage params.
// f32_in: g.in is the float NCHW input (signs taken in the gather), else pack_pixels' words.
struct PixParams {
    uint32_t w[256];
    int p[256];
    uint32_t flip[8];
};
bool pix_popc_ok(const FusedGeom& g);
int make_pix_params(const uint32_t* wbits_host, const int4* prm_host, int D, int K, PixParams* pp);
int launch_pix_popc(const FusedGeom& g, const PixParams& pp, bool f32_in, cudaStream_t s);

int fused_prep_weights(const uint32_t* packed, size_t ldw, int D, int K, int C, int T, int perm_bits, int Dpad,
                       int Kpad, int8_t* out, cudaStream_t s);
int fused_prep_params(const int8_t* w8, int Kpad, int D, int Dp, int K, const float* bias, const float* scale,
                      const float* shift, int4* prm, int* bad_dev, cudaStream_t s);
int fused_make_tmap(CUtensorMap* map, const int8_t* w, int Dpad, int Kpad, int BN);
int fused_set_fp4_pair(int mode);
int launch_pack_pixels(const float* x, size_t B, int C, size_t HW, uint32_t* out, cudaStream_t s);
// cg = 1: CTA-local M=128 tiles; cg = 2: CTA pairs with cta_group::2 M=256 tiles. tm must be
// the weight map whose box has BN / cg rows.
int launch_fused(int cg, int BN, int in_mode, int epi, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s);

}  // namespace bnnk
