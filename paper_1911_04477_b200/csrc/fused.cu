// Fused binary layer on the 5th-generation tensor cores: implicit-GEMM binary conv / linear
// with the inter-layer glue folded into the epilogue.
//
// One launch computes, for every output position of a conv (or every image of a linear
// layer), what the reference computes as
//
//   conv_forward_binary / linear_forward_packed   (network.cpp:65-79, 121-126)
//     = xnor_gemm(pack_rows(sign W), pack_cols(sign im2col(x)))  -> to_float -> bias_add
//   [maxpool2]                                     (network.cpp:133-149)
//   affine_norm   fmaf(scale, y, shift)            (network.cpp:151-175, FMA-contracted)
//   htanh, sign                                    (binarize.cpp:24-37)
//
// and writes the result directly as the NEXT layer's packed input bits. Why this is exact:
//   * the xnor-popcount value L - 2*popc(w ^ x) is the integer dot product of the +-1
//     vectors, so it is computed as an int8 x int8 -> int32 tcgen05.mma (kind::i8) of the
//     +-1 bytes; every accumulator is the reference's exact integer.
//   * the reduction order of K is free for an exact integer sum, so weights and activations
//     use the engine's K order (tap-major, channel-minor) instead of im2col's c-major order;
//     the weights are permuted once at build time (prep kernel below).
//   * float(acc) + bias is monotone in acc, so maxpool of the four floats equals the float of
//     the max integer: the 2x2 max is taken on the accumulators.
//   * sign(htanh(z)) = sign(z) = (z >= 0) for every z (htanh keeps the sign, -0.0 >= 0).
//   * spatial zero padding reads as 0.0 in the reference's im2col and sign(0.0) = +1, so an
//     out-of-image activation word is 0xFFFFFFFF.
//
// Data layout (HBM): activations between fused layers are packed bits, NHWC:
// act[((b*H + y)*W + x)*Cw + w], bit j of word w = channel 32w + j (1 = +1). Conv layers
// whose output is max-pooled enumerate their output rows pool-major
// (row = ((b*OH/2 + py)*OW/2 + px)*4 + sub), so a pooling window is four adjacent TMEM
// lanes and the pooled row index is row/4, the NHWC order of the pooled tensor.
//
// Kernel anatomy (persistent, one CTA per SM, 320 threads):
//   warp 0      TMA producer of the weight tile B (int8 +-1, [Dpad, Kpad], K-major,
//               SWIZZLE_128B), BN rows x 128 K-bytes per stage
//   warp 1      TMEM allocator + single-thread UMMA issuer, M=128 x N=BN x K=32 per
//               instruction, 4 per stage
//   warps 2-5   epilogue: tcgen05.ld -> (2x2 max) -> +bias -> fma(scale, ., shift) -> >= 0
//               -> 32-channel words -> vector stores; or float logits / NCHW floats
//   warps 6-9   activation producers: one tile row (output position) per thread; read 4
//               packed words per stage (one 16-byte load), expand bit -> +-1 byte and store
//               them in the SWIZZLE_128B K-major layout the UMMA descriptor expects.
#include <algorithm>
#include <string>
#include <vector>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "bnn_common.cuh"
#include "fused.cuh"
#include "umma.cuh"

namespace bnnk {

// debug timeline (bnn_debug_timeline): globaltimer stamps per CTA and launch
constexpr int kTlSlots = 64;  // launches (or chain stages) per recording
constexpr int kTlCtas = 160;  // >= SMs
unsigned long long* g_tl = nullptr;
int g_tl_used = -1;  // -1: off
std::vector<std::string> g_tl_names;

using namespace umma;

namespace {

constexpr int kStages = 4;   // CG = 1: A 16 KB + B up to 32 KB per stage
constexpr int kStages2 = 6;  // CG = 2: A 16 KB + B up to 16 KB per stage (per CTA)
constexpr int kThreads = 448;  // 14 warps: TMA, MMA, 4+4 epilogue (2-5, 10-13), 4 producer (6-9)
constexpr int kRows = 128;   // UMMA M
constexpr int kKB = 128;     // K bytes per stage

constexpr int kMaxF32K = 1024;  // float-input layers: K <= this (im2col offset table in smem)
constexpr int kMaxQ = 1024;     // K words per layer (bits mode), entries of the offset table
constexpr int kMaxD = 4096;     // output channels of a bits-epilogue launch (threshold table)
constexpr int kMaxPixTaps = 16; // pixel-packed first layer: taps (and taps*C <= 64)

template <int BN, int CG, int ATM>
constexpr size_t fused_smem() {
    static_assert(kMaxF32K <= kMaxQ, "one table region");
    return 1024 + size_t(CG == 2 ? kStages2 : kStages) * ((ATM ? 0 : kRows) + BN / CG) * kKB + 256 + kMaxQ * 8 +
           kMaxD * 4 + kMaxD / 8;
}

__device__ __forceinline__ bool decode_row(const FusedGeom& g, int row, int& b, int& oy, int& ox) {
    if (row >= g.rows) return false;
    if (g.pool) {  // dv0 = OW/2, dv1 = OH/2
        const int s = row & 3, win = row >> 2;
        const int t = g.dv0.div(win), px = win - t * int(g.dv0.d);
        b = g.dv1.div(t);
        const int py = t - b * int(g.dv1.d);
        oy = 2 * py + (s >> 1);
        ox = 2 * px + (s & 1);
    } else {  // dv0 = OH*OW, dv1 = OW
        b = g.dv0.div(row);
        const int p = row - b * int(g.dv0.d);
        oy = g.dv1.div(p);
        ox = p - oy * int(g.dv1.d);
    }
    return true;
}

// Store one 16-byte chunk of row r at its SWIZZLE_128B position (chunk ^ (r % 8)).
__device__ __forceinline__ void put_chunk(uint32_t tile, int r, int chunk, uint32_t a, uint32_t b, uint32_t c,
                                          uint32_t d) {
    st_shared_v4(tile + uint32_t(r) * 128u + (uint32_t(chunk ^ (r & 7)) << 4), a, b, c, d);
}

// One packed word (32 K positions) -> 32 operand bytes in {0, 1} (the bit itself; see the
// u8 encoding note at fused_prep_weights). Byte j of output word s is bit 8j + s, so each
// output word is one shift + one AND: 15 ALU ops for 32 bytes. The weights use the same
// within-word order.
__device__ __forceinline__ void put_word(uint32_t tile, int r, int i, uint32_t w) {
    constexpr uint32_t m = 0x01010101u;
    put_chunk(tile, r, 2 * i, w & m, (w >> 1) & m, (w >> 2) & m, (w >> 3) & m);
    put_chunk(tile, r, 2 * i + 1, (w >> 4) & m, (w >> 5) & m, (w >> 6) & m, (w >> 7) & m);
}

// Per-row state of the activation producer for the current tile.
struct RowCtx {
    bool valid;
    int pix;  // b*H (bits/pixel modes)
    int y0, x0;  // oy*SH, ox*SW
};

// The 4 packed words (one 128-position K block) of one row. qtab[q] = {dy<<16 | dx&0xffff,
// cw} for K word q (cw < 0: K padding). One 16-byte load when the block is one tap of
// contiguous channels (Cw % 4 == 0), else word by word.
// Activation loads. A single-layer launch uses the read-only path (ld.global.nc), predicated.
// Coherent = true (ld.global.ca, volatile asm) is for activations written during the same launch
// by other CTAs; the per-layer kernels use the read-only path.
__device__ __forceinline__ uint4 ld_ca4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.ca.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_ca(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

template <bool Coherent = false>
__device__ __forceinline__ uint4 load_bits(const FusedGeom& g, const int2* qtab, const RowCtx& rc, int kb) {
    const uint32_t* act = static_cast<const uint32_t*>(g.in);
    if (!rc.valid) return make_uint4(0, 0, 0, 0);
    if ((g.Cw & 3) == 0) {
        const int2 e = qtab[4 * kb];
        if (e.y < 0) return make_uint4(0, 0, 0, 0);  // a block past K (FP4's 256-position blocks)
        const int iy = rc.y0 + (e.x >> 16), ix = rc.x0 + int(short(e.x & 0xffff));
        const bool inb = unsigned(iy) < unsigned(g.H) && unsigned(ix) < unsigned(g.W);
        const uint32_t* src = act + (size_t((rc.pix + iy) * g.W + ix)) * g.Cw + e.y;
        if (Coherent) {
            const uint4 v = ld_ca4(inb ? src : act);
            return inb ? v : make_uint4(~0u, ~0u, ~0u, ~0u);
        }
        if (inb) return __ldg(reinterpret_cast<const uint4*>(src));
        return make_uint4(~0u, ~0u, ~0u, ~0u);  // spatial padding: sign(0.0) = +1
    }
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int2 e = qtab[4 * kb + i];
        const int iy = rc.y0 + (e.x >> 16), ix = rc.x0 + int(short(e.x & 0xffff));
        const bool inb = unsigned(iy) < unsigned(g.H) && unsigned(ix) < unsigned(g.W);
        const uint32_t* src = act + size_t((rc.pix + iy) * g.W + ix) * g.Cw + e.y;
        if (Coherent) {
            const uint32_t v = ld_ca(e.y >= 0 && inb ? src : act);
            w[i] = e.y < 0 ? 0u : inb ? v : ~0u;
        } else {
            w[i] = e.y < 0 ? 0u  // K padding: 0 bytes, and the weights are 0 there too
                   : inb ? __ldg(src) : ~0u;
        }
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// Pixel-packed first layer (FIN_PIX): in[(b*H + y)*W + x] holds the C <= 32 sign bits of one
// input pixel (pack_pixels_kernel). The row's K = T*C bits are gathered tap by tap,
// tap-major / channel-minor (K <= 64: one K block). qtab[tap] = {dy<<16 | dx&0xffff, 0}.
// load_pix() only issues the loads (their values are consumed kPF blocks later by
// gather_pix(), so the L2 latency is hidden like the bits path's).
// NT: compile-time tap count (9 for the 3x3 first layer: no dead iterations), else kMaxPixTaps
// with the runtime T <= NT.
template <int NT = kMaxPixTaps>
struct PixRaw {
    uint32_t v[NT];
};

template <bool Coherent = false, int NT = kMaxPixTaps>
__device__ __forceinline__ PixRaw<NT> load_pix(const FusedGeom& g, const int2* qtab, const RowCtx& rc) {
    const uint32_t* pix = static_cast<const uint32_t*>(g.in);
    const int T = NT == kMaxPixTaps ? g.KH * g.KW : NT;
    const uint32_t cmask = g.C == 32 ? ~0u : ((1u << g.C) - 1u);
    PixRaw<NT> raw;
#pragma unroll
    for (int tap = 0; tap < NT; ++tap) {
        const int2 e = qtab[tap < T ? tap : 0];
        const int iy = rc.y0 + (e.x >> 16), ix = rc.x0 + int(short(e.x & 0xffff));
        const bool inb = rc.valid && tap < T && unsigned(iy) < unsigned(g.H) && unsigned(ix) < unsigned(g.W);
        const uint32_t* src = pix + size_t(rc.pix + iy) * g.W + ix;
        uint32_t v = cmask;  // padding: every channel +1
        if (Coherent) {
            if (tap < T) {  // T is uniform: no divergence
                const uint32_t u = ld_ca(inb ? src : pix);
                v = inb ? u : cmask;
            }
        } else if (inb) {
            v = __ldg(src);
        }
        raw.v[tap] = v;
    }
    return raw;
}

template <int NT>
__device__ __forceinline__ uint4 gather_pix(const FusedGeom& g, const PixRaw<NT>& raw, bool valid) {
    if (!valid) return make_uint4(0, 0, 0, 0);
    const int T = NT == kMaxPixTaps ? g.KH * g.KW : NT;
    uint64_t acc = 0;
#pragma unroll
    for (int tap = 0; tap < NT; ++tap)
        if (tap < T) acc |= uint64_t(raw.v[tap]) << (tap * g.C);
    return make_uint4(uint32_t(acc), uint32_t(acc >> 32), 0u, 0u);
}

__device__ __forceinline__ void store_bits(uint32_t tile, int r, uint4 u) {
    put_word(tile, r, 0, u.x);
    put_word(tile, r, 1, u.y);
    put_word(tile, r, 2, u.z);
    put_word(tile, r, 3, u.w);
}

// One K block of one row, float NCHW input, reference im2col order r = (c*KH + ky)*KW + kx;
// bytes in natural order, value (x >= 0) (binarize.cpp:9). tab[k] = {c*H*W + ky*W + kx, ky<<16|kx}.
__device__ __forceinline__ void produce_f32(const FusedGeom& g, const int2* tab, uint32_t tile, int r,
                                            bool valid, int b, int oy, int ox, int kb) {
    const float* x = static_cast<const float*>(g.in) + size_t(b) * g.C * g.H * g.W;
    const int y0 = oy * g.SH - g.PH, x0 = ox * g.SW - g.PW;
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const int k0 = kb * kKB + j * 16;
        uint32_t u[4] = {0, 0, 0, 0};
        if (valid && k0 < g.K) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int k = k0 + e;
                if (k < g.K) {
                    const int2 t = tab[k];
                    const int iy = y0 + (t.y >> 16), ix = x0 + (t.y & 0xffff);
                    float v = 0.0f;
                    if (iy >= 0 && iy < g.H && ix >= 0 && ix < g.W) v = __ldg(x + t.x + y0 * g.W + x0);
                    u[e >> 2] |= uint32_t(v >= 0.0f) << (8 * (e & 3));
                }
            }
        }
        put_chunk(tile, r, j, u[0], u[1], u[2], u[3]);
    }
}

// Profiling aid (FusedGeom::dbg, set by BNN_FUSED_PROFILE=1): cycles each role spends
// blocked on its barriers, accumulated over CTAs. Slots: [role*4 + 0/1] waits, [role*4 + 3]
// total cycles; roles 0 TMA, 1 MMA, 2 epilogue, 3 producer.
__device__ __forceinline__ long long dclock() {
#ifdef __CUDA_ARCH__
    return clock64();
#else
    return 0;
#endif
}

// "memory" clobber: the read must not move across the barriers it brackets (a volatile asm
// without it can be scheduled ahead of __syncthreads)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}

struct WaitClock {
    long long w[2];
    long long t_start;
    __device__ __forceinline__ WaitClock() : w{0, 0}, t_start(dclock()) {}
    __device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity, int slot) {
        const long long t0 = dclock();
        mbar_wait(bar, parity);
        w[slot] += dclock() - t0;
    }
    __device__ __forceinline__ void flush(unsigned long long* dbg, int role) {
        if (!dbg) return;
        atomicAdd(dbg + role * 4 + 0, (unsigned long long)w[0]);
        atomicAdd(dbg + role * 4 + 1, (unsigned long long)w[1]);
        atomicAdd(dbg + role * 4 + 3, (unsigned long long)(dclock() - t_start));
    }
};

// CG = 1: one CTA computes a 128-row tile with M=128 x N=BN instructions.
// CG = 2: a CTA pair (cluster of 2) computes a 256-row tile with cta_group::2 M=256 x N=BN
// instructions issued by the even CTA: each CTA produces its own 128 activation rows, TMA-loads
// half of the weight tile (BN/2 rows), and holds its 128 accumulator rows in its own TMEM. The
// i8 MMA costs the same per instruction for any N <= 256 at M=128 (measured, profiles/), so
// layers with D = 128 need the pair to reach the full tensor rate; the pair also halves each
// SM's weight traffic.
// ATM = 1: the activation operand A lives in TMEM (tcgen05.st by the producers, the MMA reads
// it with the TS form) instead of shared memory. This takes the A tile off the shared-memory
// port (its stores and the MMA's reads) and replaces the per-stage proxy fence (a MEMBAR that
// drained the producers' prefetch loads) with tcgen05.wait::st. TMEM then holds the A stages
// (32 columns each) next to the accumulators; with BN = 256 there is room for one accumulator
// only, so the epilogue of tile i no longer overlaps the MMAs of tile i+1.
template <int BN, int ATM>
struct TmemPlan {
    static constexpr int kAStage = 32;  // columns per A stage (128 K-bytes per lane)
    static constexpr int kAcc = ATM ? (2 * BN + kStages * kAStage <= 512 ? 2 : 1) : 2;
    static constexpr int kACol = kAcc * BN;  // first A-stage column
    static constexpr int kUsed = kACol + (ATM ? kStages * kAStage : 0);
    static constexpr uint32_t kCols = kUsed <= 32 ? 32 : kUsed <= 64 ? 64 : kUsed <= 128 ? 128 : kUsed <= 256 ? 256 : 512;
    static_assert(kUsed <= 512, "TMEM budget");
};

template <int BN, int IN, int EPI, int CG, int ATM, int PT = 0>
__global__ void __launch_bounds__(kThreads, 1)
    fused_layer_kernel(const __grid_constant__ CUtensorMap tmW, const FusedGeom g) {
    static_assert(!(ATM && (CG == 2 || IN == FIN_F32)), "TMEM A operand: CTA-local, bits/pixel input");
    using TP = TmemPlan<BN, ATM>;
    constexpr int kS = CG == 2 ? kStages2 : kStages;
    constexpr int BH = BN / CG;  // weight rows held by this CTA
    constexpr int kAcc = TP::kAcc;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - raw);
    uint8_t* sA = smem;                                           // [kS][128 * 128] (SS form only)
    uint8_t* sB = smem + (ATM ? 0 : size_t(kS) * kRows * kKB);    // [kS][BH * 128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(kS) * BH * kKB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kS;
    uint64_t* tfull = bars + 2 * kS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int2* ftab = reinterpret_cast<int2*>(bars + 32);  // offset table [kMaxQ]
    int* tu_s = reinterpret_cast<int*>(ftab + kMaxQ);                 // [kMaxD] thresholds Tu
    uint32_t* flip_s = reinterpret_cast<uint32_t*>(tu_s + kMaxD);     // [kMaxD / 32] flip words

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    if (!g.pdl_late) asm volatile("griddepcontrol.launch_dependents;");  // the next layer may start its prologue
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 0] = gtimer();
    const int unit = blockIdx.x / CG, units = gridDim.x / CG;
    const int m_tiles = (g.rows + kRows * CG - 1) / (kRows * CG);
    const int n_tiles = g.n_tiles;
    const int S = g.ksplit;  // split-K factor (>= 1): tile t is (output tile t / S, K slice t % S)
    const int tiles = m_tiles * n_tiles * S;
    const int KB = g.KB;
    auto kb_begin = [&](int t) { return (t % S) * KB / S; };
    auto kb_end = [&](int t) { return (t % S + 1) * KB / S; };
    auto tile_n = [&](int t) { return (t / S) % n_tiles; };
    auto tile_m = [&](int t) { return (t / S) / n_tiles; };

    if (threadIdx.x == 0) {
        tma_prefetch(&tmW);
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], 4 * CG + CG);  // one arrive per producer warp + per TMA thread
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8 * CG);  // eight epilogue warps per CTA
        }
        fence_mbar_init();
    }
    if (IN == FIN_F32) {  // im2col offset table: k -> (c*H*W + ky*W + kx, ky, kx)
        const int khw = g.KH * g.KW;
        for (int k = threadIdx.x; k < g.K; k += blockDim.x) {
            const int c = k / khw, t = k - c * khw, ky = t / g.KW, kx = t - ky * g.KW;
            ftab[k] = make_int2(c * g.H * g.W + ky * g.W + kx, (ky << 16) | kx);
        }
    } else if (IN == FIN_BITS) {  // K word q -> (tap offset, channel word); all divisions here
        const int kw_total = (g.K + 31) >> 5;  // a partial last word holds zero pad bits
        for (int q = threadIdx.x; q < 4 * KB; q += blockDim.x) {
            int2 e = make_int2(0, -1);
            if (q < kw_total) {
                const int tap = q / g.Cw, cw = q - tap * g.Cw, ky = tap / g.KW, kx = tap - ky * g.KW;
                e = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), cw);
            }
            ftab[q] = e;
        }
    } else {  // FIN_PIX: tap -> offset
        for (int tap = threadIdx.x; tap < g.KH * g.KW; tap += blockDim.x) {
            const int ky = tap / g.KW, kx = tap - ky * g.KW;
            ftab[tap] = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), 0);
        }
    }
    if (EPI == FEPI_BITS) {  // this launch's thresholds and flip bits, for every n tile
        const int dp = n_tiles * BN;
        for (int d = threadIdx.x; d < dp; d += blockDim.x) tu_s[d] = __ldg(g.prm + d).x;
        for (int d0 = warp * 32; d0 < dp; d0 += (kThreads / 32) * 32) {
            const uint32_t f = __ballot_sync(0xffffffffu, __ldg(g.prm + d0 + lane).y != 0);
            if (lane == 0) flip_s[d0 >> 5] = f;
        }
    }
    if (warp == 1) {
        if (CG == 2)
            tmem_alloc_cg2<TP::kCols>(tmem_slot);
        else
            tmem_alloc<TP::kCols>(tmem_slot);
    }
    __syncwarp();  // reconverge role-divergent lanes: bar.sync counts a partial warp as whole
    tc_fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    // (stamp 1 is written at the very end, after the TMEM dealloc)
    // Programmatic dependent launch: everything above touches only this launch's constants
    // (weights' tensor map, thresholds, tables, TMEM, barriers), so it overlaps the previous
    // layer's tail. From here on the previous layer's output is read and a buffer it may still
    // be reading is written: wait for it to complete.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 2] = gtimer();

    // barrier the producers / TMA / epilogue signal: the even CTA's (shared::cluster address)
    auto leader = [&](uint64_t* bar) { return CG == 2 ? mapa(smem_u32(bar), 0) : smem_u32(bar); };

    if (warp == 0) {
        // -------------------------------------------------------------- weight TMA
        if (lane == 0) {
            WaitClock wc;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = unit; t < tiles; t += units) {
                const int nt = tile_n(t), kb1 = kb_end(t);
                for (int kb = kb_begin(t); kb < kb1; ++kb) {
                    wc.wait(&empty[stage], phase ^ 1, 0);
                    uint8_t* dst = sB + size_t(stage) * BH * kKB;
                    if (CG == 2) {
                        const uint32_t fb = leader(&full[stage]);
                        mbar_arrive_expect_tx_cluster(fb, BH * kKB);
                        tma_load_2d_cg2(&tmW, fb, dst, kb * kKB, nt * BN + int(rank) * BH);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], BH * kKB);
                        tma_load_2d(&tmW, &full[stage], dst, kb * kKB, nt * BN);
                    }
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
            }
            wc.flush(g.dbg, 0);
        }
    } else if (warp == 1) {
        // -------------------------------------------------------------- UMMA issuer
        if (CG == 1 || rank == 0) {
            constexpr uint32_t idesc = idesc_i8(kRows * CG, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            WaitClock wc;
            for (int t = unit; t < tiles; t += units) {
                wc.wait(&tempty[acc], acc_phase ^ 1, 0);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
                const int kb0 = kb_begin(t), kb1 = kb_end(t);
                for (int kb = kb0; kb < kb1; ++kb) {
                    wc.wait(&full[stage], phase, 1);
                    tc_fence_after();
                    {  // the converged warp issues (one elected lane): see mma_i8_w
                        const uint32_t a0 = smem_u32(sA + size_t(stage) * kRows * kKB);
                        const uint32_t b0 = smem_u32(sB + size_t(stage) * BH * kKB);
                        // K steps past the layer's K in its last block multiply zeros: skip them
                        const int nk = kb == KB - 1 ? g.kq_last : kKB / 32;
#pragma unroll
                        for (int k = 0; k < kKB / 32; ++k) {
                            if (k >= nk) break;
                            if (ATM)
                                mma_i8_ts_w(d_tmem, tmem_base + uint32_t(TP::kACol + stage * TP::kAStage + 8 * k),
                                            sdesc_k_sw128(b0 + 32 * k), idesc, (kb != kb0 || k != 0));
                            else if (CG == 2)
                                mma_i8_cg2_w(d_tmem, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                             (kb != kb0 || k != 0));
                            else
                                mma_i8_w(d_tmem, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                         (kb != kb0 || k != 0));
                        }
                        if (CG == 2) {
                            mma_commit_cg2_mc_w(&empty[stage], 3);  // both CTAs' slots free
                            if (kb == kb1 - 1) mma_commit_cg2_mc_w(&tfull[acc], 3);
                        } else {
                            mma_commit_w(&empty[stage]);
                            if (kb == kb1 - 1) mma_commit_w(&tfull[acc]);
                        }
                    }
                    __syncwarp();
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
                if (++acc == kAcc) acc = 0, acc_phase ^= 1;
            }
            if (lane == 0) wc.flush(g.dbg, 1);
            if (CG == 1) {
                // Free TMEM as soon as the epilogue has read the last accumulators (wait for the
                // release of every slot, as if kAcc more tiles followed) instead of after the
                // final __syncthreads, so the dealloc overlaps the epilogue's last stores.
                for (int k = 0; k < kAcc; ++k) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    if (++acc == kAcc) acc = 0, acc_phase ^= 1;
                }
                tc_fence_after();
                tmem_dealloc<TP::kCols>(tmem_base);
            }
        }
    } else if (warp < 6 || warp >= 10) {
        // -------------------------------------------------------------- epilogue
        // Accumulator u = sum_k bit_k * w_k (bits in {0,1}, weights +-1); the reference's
        // xnor-popcount value is a = 2u - S_d with S_d = sum_k w_k (prm.z).
        // Eight warps: warps 2-5 convert the first half of the tile's 32-column chunks,
        // warps 10-13 the second half (same TMEM lane quarter = same rows), which halves the
        // time the accumulator stays busy after the last MMA.
        const int q = warp & 3;  // TMEM lane quarter of this warp
        const int r = q * 32 + lane;
        constexpr int NC = BN / 32;
        const int c_lo = warp >= 10 ? (NC + 1) / 2 : 0, c_hi = warp >= 10 ? NC : (NC + 1) / 2;
        // Split-K completion (S > 1, CTA-local tiles, no pooling): the S CTAs of an output tile
        // publish their partial sums, meet at a counter, and each reduces 128/S rows of the tile
        // (its K-slice index picks the rows); the last one out resets the counters for the
        // next launch. The S CTAs are co-resident (grid = tiles <= SMs, one CTA per SM).
        const int et = (warp < 6 ? warp - 2 : warp - 6) * 32 + lane;  // 0..255 over the 8 warps
        auto epi_bar = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };  // the 8 epilogue warps
        auto split_reduce = [&](int t, int mt, int n0) {
            const int u = t / S, ks = t % S;
            __threadfence();  // this thread's partials, device-wide
            epi_bar();
            if (warp == 2 && lane == 0) {
                atomicAdd(g.sem + 2 * u, 1u);
                unsigned seen;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(g.sem + 2 * u) : "memory");
                } while (seen < unsigned(S));
                __threadfence();
            }
            __syncwarp();  // bar.sync is .aligned: the warp must arrive converged
            epi_bar();
            // each thread sums 4 adjacent columns of one row over the S slices (independent
            // 16-byte L2 loads, all in flight); 8 adjacent lanes hold one 32-channel word
            const int rp = kRows / S;
            constexpr int C4 = BN / 4;  // 4-column groups per row (a multiple of 8)
            for (int i0 = 0; i0 < rp * C4; i0 += 256) {
                const int i = i0 + et;
                const bool live = i < rp * C4;
                const int row2 = mt * kRows + ks * rp + (live ? i / C4 : 0), c4 = i % C4;
                const int n = n0 + 4 * c4;
                int4 sum = make_int4(0, 0, 0, 0);
                if (live) {
                    const int4* src = reinterpret_cast<const int4*>(g.ws + size_t(row2) * g.ws_ld + n);
                    const size_t slice = size_t(g.ws_rows) * g.ws_ld / 4;  // int4 stride between slices
#pragma unroll 4
                    for (int s2 = 0; s2 < S; ++s2) {
                        const int4 v4 = __ldcg(src + s2 * slice);
                        sum.x += v4.x, sum.y += v4.y, sum.z += v4.z, sum.w += v4.w;
                    }
                }
                const bool out = live && row2 < g.rows && n < g.D;
                if (EPI == FEPI_BITS) {
                    uint32_t w = 0;
                    if (live) {
                        const int4 t4 = *reinterpret_cast<const int4*>(tu_s + n);
                        w = (uint32_t(sum.x >= t4.x) | (uint32_t(sum.y >= t4.y) << 1) | (uint32_t(sum.z >= t4.z) << 2) |
                             (uint32_t(sum.w >= t4.w) << 3))
                            << (4 * (c4 & 7));
                    }
                    w |= __shfl_xor_sync(0xffffffffu, w, 1);
                    w |= __shfl_xor_sync(0xffffffffu, w, 2);
                    w |= __shfl_xor_sync(0xffffffffu, w, 4);
                    if (out && (c4 & 7) == 0) g.out_bits[size_t(row2) * g.Dw + (n >> 5)] = w ^ flip_s[n >> 5];
                } else if (out) {
                    const int sv[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int d = n + j;
                        if (d >= g.D) break;
                        const int4 pd = __ldg(g.prm + d);
                        const float y = __fadd_rn(__int2float_rn(2 * sv[j] - pd.z), __int_as_float(pd.w));
                        if (EPI == FEPI_LOGITS) {
                            g.out_f32[size_t(d) * g.ldo + row2] = y;
                        } else {
                            const int P = g.OH * g.OW, b = row2 / P;
                            g.out_f32[(size_t(b) * g.D + d) * P + (row2 - b * P)] = y;
                        }
                    }
                }
            }
            epi_bar();
            if (warp == 2 && lane == 0 && atomicAdd(g.sem + 2 * u + 1, 1u) == unsigned(S - 1)) {
                g.sem[2 * u] = 0;  // every CTA of the tile is past its wait and its reads
                g.sem[2 * u + 1] = 0;
            }
        };
        int acc = 0;
        uint32_t acc_phase = 0;
        WaitClock wc;
        for (int t = unit; t < tiles; t += units) {
            const int mt = tile_m(t), nt = tile_n(t);
            const int row = mt * kRows * CG + int(rank) * kRows + r;
            const int n0 = nt * BN;
            const bool valid = row < g.rows;
            wc.wait(&tfull[acc], acc_phase, 0);
            tc_fence_after();
            uint32_t words[BN / 32];
            const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN);
            // TMEM loads double-buffered: chunk c+1 is in flight while chunk c is converted
            // (tcgen05.wait::ld waits for every outstanding load, so it comes first).
            uint32_t va[32], vb[32];
            auto convert = [&](const uint32_t(&v)[32], int c) {
                if (S > 1) {  // split-K: this slice's partial sums go to the workspace
                    int4* dst = reinterpret_cast<int4*>(g.ws + ((size_t(t % S) * g.ws_rows + row) * g.ws_ld + n0 + c * 32));
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        dst[j] = make_int4(int(v[4 * j]), int(v[4 * j + 1]), int(v[4 * j + 2]), int(v[4 * j + 3]));
                    return;
                }
                if (g.dbg_mode & 2) {
                    words[0] = v[0];
                } else if (EPI == FEPI_BITS) {
                    // bit = (u >= Tu) ^ flip: the exact float predicate of the reference
                    // (fma(scale, float(a) + bias, shift) >= 0), monotone in a, tabulated at
                    // build time (prep_params_kernel). Pooling: the predicate of the max is the
                    // OR of the (u >= Tu) terms, so the 2x2 max is a word OR over 4 lanes.
                    // Thresholds come from shared memory as broadcast 16-byte loads.
                    const int4* t4 = reinterpret_cast<const int4*>(tu_s + n0 + c * 32);
                    uint32_t w = 0;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const int4 t = t4[j >> 2];
                        w |= (uint32_t(int(v[j]) >= t.x) << j) | (uint32_t(int(v[j + 1]) >= t.y) << (j + 1)) |
                             (uint32_t(int(v[j + 2]) >= t.z) << (j + 2)) | (uint32_t(int(v[j + 3]) >= t.w) << (j + 3));
                    }
                    if (g.pool) {
                        w |= __shfl_xor_sync(0xffffffffu, w, 1);
                        w |= __shfl_xor_sync(0xffffffffu, w, 2);
                    }
                    w ^= flip_s[(n0 >> 5) + c];
#pragma unroll
                    for (int cc = 0; cc < BN / 32; ++cc)  // static register index
                        if (cc == c) words[cc] = w;
                } else {
                    // to_float(a) + bias (kernels.cpp:90-107): one rounding of an exact integer
                    const int4 pl = __ldg(g.prm + n0 + c * 32 + lane);  // this lane's channel
                    const int P = g.OH * g.OW;
                    const int b = valid ? row / P : 0, p = row - b * P;
#pragma unroll 4
                    for (int j = 0; j < 32; ++j) {
                        const int d = n0 + c * 32 + j;
                        const int sd = __shfl_sync(0xffffffffu, pl.z, j);
                        const float bias = __int_as_float(__shfl_sync(0xffffffffu, pl.w, j));
                        const float y = __fadd_rn(__int2float_rn(2 * int(v[j]) - sd), bias);
                        if (valid && d < g.D) {
                            if (EPI == FEPI_LOGITS)
                                g.out_f32[size_t(d) * g.ldo + row] = y;
                            else
                                g.out_f32[(size_t(b) * g.D + d) * P + p] = y;
                        }
                    }
                }
            };
            // TMEM loads double-buffered: chunk c+1 is in flight while chunk c is converted
            // (tcgen05.wait::ld waits for every outstanding load, so it comes first).
            if (c_lo < c_hi) tmem_ld32(tbase + uint32_t(c_lo * 32), va);
#pragma unroll 1
            for (int c = c_lo; c < c_hi; c += 2) {
                tmem_ld_wait();
                if (c + 1 < c_hi) tmem_ld32(tbase + uint32_t((c + 1) * 32), vb);
                convert(va, c);
                if (c + 1 < c_hi) {
                    tmem_ld_wait();
                    if (c + 2 < c_hi) tmem_ld32(tbase + uint32_t((c + 2) * 32), va);
                    convert(vb, c + 1);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {  // TMEM buffer free before the stores drain
                if (CG == 2)
                    mbar_arrive_cluster(leader(&tempty[acc]));
                else
                    mbar_arrive(&tempty[acc]);
            }
            if (S > 1) {
                split_reduce(t, mt, n0);
            } else if (EPI == FEPI_BITS && valid && (!g.pool || (lane & 3) == 0)) {
                const int orow = g.pool ? (row >> 2) : row;
                uint32_t* dst = g.out_bits + size_t(orow) * g.Dw + (n0 >> 5);
                constexpr int H = (NC + 1) / 2;  // chunks per half
                if (H % 4 == 0 && (g.Dw & 3) == 0 && n0 + BN <= g.D) {
#pragma unroll
                    for (int c = 0; c < NC; c += 4)
                        if (c >= c_lo && c < c_hi)
                            *reinterpret_cast<uint4*>(dst + c) =
                                make_uint4(words[c], words[c + 1], words[c + 2], words[c + 3]);
                } else {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        if (c >= c_lo && c < c_hi && n0 + 32 * c < g.D) dst[c] = words[c];
                }
            }
            if (++acc == kAcc) acc = 0, acc_phase ^= 1;
        }
        if (warp == 2 && lane == 0) wc.flush(g.dbg, 2);
    } else {
        // -------------------------------------------------------------- activation producers (warps 6-9)
        // One tile row per thread: the row's 4 packed words of the block -> 128 operand bytes
        // in the UMMA layout. The words are loaded kPF blocks ahead into registers.
        // Measured limits (profiles/): the per-stage proxy fence (fence.proxy.async =
        // MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC) drains in-flight loads, and the A-tile stores
        // compete with the UMMA operand reads and the weight TMA for shared-memory bandwidth.
        // tile row 0..127; with A in TMEM a warp may only write its lane quarter (warp % 4)
        const int r = ATM ? 32 * (warp & 3) + lane : threadIdx.x - 6 * 32;
        const int row_off = int(rank) * kRows + r;
        int stage = 0;
        uint32_t phase = 0;
        WaitClock wc;
        auto publish = [&](int st) {  // this warp's rows of stage st are written
            if (ATM) {
                if (!(g.dbg_mode & 8)) tmem_st_wait();
                tc_fence_before();
            } else {
                fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) {
                if (CG == 2)
                    mbar_arrive_cluster(leader(&full[st]));
                else
                    mbar_arrive(&full[st]);
            }
        };
        if (IN != FIN_F32) {
            constexpr int kPF = 3;
            constexpr int NT = PT ? PT : kMaxPixTaps;
            using Raw = typename std::conditional<IN == FIN_BITS, uint4, PixRaw<NT>>::type;
            int t_ld = unit, kb_ld = unit < tiles ? kb_begin(unit) : 0;  // next block to load
            int kb_ld_end = unit < tiles ? kb_end(unit) : 0;
            RowCtx rc;
            auto set_row = [&]() {
                int b = 0, oy = 0, ox = 0;
                rc.valid = t_ld < tiles && decode_row(g, tile_m(t_ld) * kRows * CG + row_off, b, oy, ox);
                rc.pix = b * g.H, rc.y0 = oy * g.SH, rc.x0 = ox * g.SW;
            };
            set_row();
            Raw pf[kPF];
            bool pv[kPF];  // row validity of each prefetched block (pixel gather)
            auto next_load = [&](Raw& dst, bool& v) {
                v = rc.valid;
                if constexpr (IN == FIN_BITS) {
                    dst = t_ld < tiles ? load_bits(g, ftab, rc, kb_ld) : make_uint4(0, 0, 0, 0);
                } else {
                    dst = load_pix<false, NT>(g, ftab, rc);
                }
                if (t_ld < tiles && ++kb_ld == kb_ld_end) {  // per-tile divisions only at tile change
                    t_ld += units;
                    kb_ld = t_ld < tiles ? kb_begin(t_ld) : 0;
                    kb_ld_end = t_ld < tiles ? kb_end(t_ld) : 0;
                    set_row();
                }
            };
#pragma unroll
            for (int i = 0; i < kPF; ++i) next_load(pf[i], pv[i]);
            for (int t = unit; t < tiles; t += units) {
                const int kb1 = kb_end(t);
                for (int kb = kb_begin(t); kb < kb1; ++kb) {
                    uint4 u;
                    if constexpr (IN == FIN_BITS)
                        u = pf[0];
                    else
                        u = gather_pix(g, pf[0], pv[0]);
#pragma unroll
                    for (int i = 0; i < kPF - 1; ++i) pf[i] = pf[i + 1], pv[i] = pv[i + 1];
                    next_load(pf[kPF - 1], pv[kPF - 1]);
                    wc.wait(&empty[stage], phase ^ 1, 0);
                    if (ATM) {
                        // bytes 4s..4s+3 of word i's 32-byte segment = column 8i + s (put_word's order)
                        const uint32_t taddr = tmem_base + (uint32_t(32 * (warp & 3)) << 16) +
                                               uint32_t(TP::kACol + stage * TP::kAStage);
                        tc_fence_after();
                        if (g.KB == 1 && g.kq_last == 1) {  // one K step (e.g. a 27-bit first layer)
                            uint32_t v[8];
#pragma unroll
                            for (int s8 = 0; s8 < 8; ++s8) v[s8] = (u.x >> s8) & 0x01010101u;
                            if (!(g.dbg_mode & 1)) tmem_st8(taddr, v);
                        } else {
                            uint32_t v[32];
                            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                            for (int i = 0; i < 4; ++i)
#pragma unroll
                                for (int s8 = 0; s8 < 8; ++s8) v[8 * i + s8] = (w4[i] >> s8) & 0x01010101u;
                            if (!(g.dbg_mode & 1)) tmem_st32(taddr, v);
                        }
                    } else if (!(g.dbg_mode & 1)) {
                        store_bits(smem_u32(sA + size_t(stage) * kRows * kKB), r, u);
                    }
                    publish(stage);
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
            }
        } else {
            for (int t = unit; t < tiles; t += units) {
                int b = 0, oy = 0, ox = 0;
                const bool valid = decode_row(g, tile_m(t) * kRows * CG + row_off, b, oy, ox);
                const int kb1 = kb_end(t);
                for (int kb = kb_begin(t); kb < kb1; ++kb) {
                    wc.wait(&empty[stage], phase ^ 1, 0);
                    produce_f32(g, ftab, smem_u32(sA + size_t(stage) * kRows * kKB), r, valid, b, oy, ox, kb);
                    publish(stage);
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
            }
        }
        if (r == 0) wc.flush(g.dbg, 3);
    }

    if (g.tl && warp == 1 && lane == 0) g.tl[blockIdx.x * 4 + 1] = gtimer();
    __syncwarp();  // reconverge role-divergent lanes before the CTA barrier
    tc_fence_before();
    __syncthreads();
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 3] = gtimer();
    if (g.pdl_late) asm volatile("griddepcontrol.launch_dependents;");
    if (CG == 2) {
        cluster_sync();  // no remote arrive / pair MMA may target a CTA that has exited
        if (warp == 1) tmem_dealloc_cg2<TP::kCols>(tmem_base);
    }  // CG == 1: the MMA warp deallocated already
}

// ---------------------------------------------------------------------------------------------
// Swapped-operand fused conv: tiles of 128 output channels (UMMA M, the weights, TMA-loaded
// into shared memory) x 256 output positions (UMMA N, the activations, expanded by the
// producer warps into shared memory).
//
// Why: a kind::i8 M=128 instruction costs the same ~128-150 cycles for any N <= 256
// (profiles/r01_fused_v3_bn_sweep.log), so the position-major tiles above (positions on M,
// channels on N) run layers with 128 output channels at half the tensor rate. Putting the
// positions on N fills the instruction for every layer. Both operands now come from shared
// memory (A may only come from TMEM, and 2 x 256 accumulator columns fill TMEM), so each
// 4-instruction stage moves 96 KB through shared memory (TMA 16 KB + producer 32 KB written,
// 48 KB read by the MMA): ~128 B/clk bounds it near the MMA rate. Two accumulator slots of
// 256 columns let the epilogue of tile i overlap the MMAs of tile i+1 at every width.
//
// Epilogue: TMEM lane = output channel, column = position. Each thread tests its channel's
// threshold (Tu, flip: prep_params_kernel) against 32 positions; __ballot_sync over the warp
// turns 32 channels into the packed output word of each position; pooled layers OR the 4
// words of a window (pool-major positions: 4 adjacent columns).
constexpr int kSwN = 256;  // positions per tile
constexpr size_t kSwSmem = 1024 + size_t(kStages) * (kRows + kSwN) * kKB + 256 + kMaxQ * 8;

template <int IN, int PT>
__global__ void __launch_bounds__(kThreads, 1)
    fused_swap_kernel(const __grid_constant__ CUtensorMap tmW, const FusedGeom g) {
    static_assert(IN == FIN_BITS || IN == FIN_PIX, "packed-bit or pixel-packed input");
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* sW = smem_raw + (base - raw);                 // [kStages][128 * 128] weights (A)
    uint8_t* sX = sW + size_t(kStages) * kRows * kKB;      // [kStages][256 * 128] activations (B)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + size_t(kStages) * kSwN * kKB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int2* ftab = reinterpret_cast<int2*>(bars + 32);

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.launch_dependents;");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 0] = gtimer();
    const int units = gridDim.x, unit = blockIdx.x;
    const int m_tiles = (g.D + kRows - 1) / kRows;
    const int n_tiles = (g.rows + kSwN - 1) / kSwN;
    const int tiles = m_tiles * n_tiles;  // t -> (channel tile t % m_tiles, position tile t / m_tiles)
    const int KB = g.KB;

    if (threadIdx.x == 0) {
        tma_prefetch(&tmW);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 4 + 1);  // four producer warps + the TMA thread
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        fence_mbar_init();
    }
    if (IN == FIN_BITS) {
        const int kw_total = (g.K + 31) >> 5;
        for (int q = threadIdx.x; q < 4 * KB; q += blockDim.x) {
            int2 e = make_int2(0, -1);
            if (q < kw_total) {
                const int tap = q / g.Cw, cw = q - tap * g.Cw, ky = tap / g.KW, kx = tap - ky * g.KW;
                e = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), cw);
            }
            ftab[q] = e;
        }
    } else {
        for (int tap = threadIdx.x; tap < g.KH * g.KW; tap += blockDim.x) {
            const int ky = tap / g.KW, kx = tap - ky * g.KW;
            ftab[tap] = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), 0);
        }
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    __syncwarp();  // reconverge role-divergent lanes: bar.sync counts a partial warp as whole
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 2] = gtimer();

    if (warp == 0) {
        // ------------------------------------------------------------ weight TMA (A)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            WaitClock wc;
            for (int t = unit; t < tiles; t += units) {
                const int mt = t % m_tiles;
                for (int kb = 0; kb < KB; ++kb) {
                    wc.wait(&empty[stage], phase ^ 1, 0);
                    mbar_arrive_expect_tx(&full[stage], kRows * kKB);
                    tma_load_2d(&tmW, &full[stage], sW + size_t(stage) * kRows * kKB, kb * kKB, mt * kRows);
                    if (++stage == kStages) stage = 0, phase ^= 1;
                }
            }
            wc.flush(g.dbg, 0);
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ UMMA issuer
        constexpr uint32_t idesc = idesc_i8(kRows, kSwN);
        int stage = 0;
        uint32_t phase = 0;
        int i = 0;
        WaitClock wc;
        for (int t = unit; t < tiles; t += units, ++i) {
            const int acc = i & 1;
            wc.wait(&tempty[acc], ((i >> 1) & 1) ^ 1, 0);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + uint32_t(acc * kSwN);
            for (int kb = 0; kb < KB; ++kb) {
                wc.wait(&full[stage], phase, 1);
                tc_fence_after();
                {  // the converged warp issues (one elected lane): see mma_i8_w
                    const uint32_t a0 = smem_u32(sW + size_t(stage) * kRows * kKB);
                    const uint32_t b0 = smem_u32(sX + size_t(stage) * kSwN * kKB);
                    const int nk = kb == KB - 1 ? g.kq_last : kKB / 32;  // K steps past K: zeros
#pragma unroll
                    for (int k = 0; k < kKB / 32; ++k) {
                        if (k >= nk) break;
                        mma_i8_w(d_tmem, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                 (kb != 0 || k != 0));
                    }
                    mma_commit_w(&empty[stage]);
                    if (kb == KB - 1) mma_commit_w(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == kStages) stage = 0, phase ^= 1;
            }
        }
        if (lane == 0) wc.flush(g.dbg, 1);
        // early TMEM release (see fused_layer_kernel): wait until both slots are read
        for (int k = 0; k < 2; ++k, ++i) mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    } else if (warp < 6 || warp >= 10) {
        // ------------------------------------------------------------ epilogue
        WaitClock wc;
        const int q = warp & 3;                       // TMEM lane quarter: channels q*32 + lane
        const int col0 = warp >= 10 ? kSwN / 2 : 0;   // this warp's half of the positions
        int i = 0;
        for (int t = unit; t < tiles; t += units, ++i) {
            const int acc = i & 1;
            const int mt = t % m_tiles, nt = t / m_tiles;
            const int c = mt * kRows + q * 32 + lane;
            const bool wvalid = mt * kRows + q * 32 < g.D;  // D % 32 == 0: whole words
            const int4 pc = wvalid ? __ldg(g.prm + c) : make_int4(0x7fffffff, 0, 0, 0);
            const int Tu = pc.x;
            const bool flip = pc.y != 0;  // folded into each compare: bit = (u >= Tu) != flip
            const int oword = mt * (kRows / 32) + q;
            wc.wait(&tfull[acc], (i >> 1) & 1, 0);
            tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kSwN + col0);
            uint32_t va[32], vb[32];
            auto emit = [&](const uint32_t(&v)[32], int cc) {
                uint32_t mine = 0;
                if (g.pool) {  // one compare per pool window, as in fused_swap4_kernel
#pragma unroll
                    for (int p = 0; p < 8; ++p) {
                        const int a = int(v[4 * p]), b = int(v[4 * p + 1]), c = int(v[4 * p + 2]), d = int(v[4 * p + 3]);
                        const int m = flip ? min(min(a, b), min(c, d)) : max(max(a, b), max(c, d));
                        const uint32_t w = __ballot_sync(0xffffffffu, (m >= Tu) != flip);
                        if (lane == p) mine = w;
                    }
                    const int pos = nt * kSwN + col0 + cc * 32 + 4 * lane;
                    if (wvalid && lane < 8 && pos < g.rows) g.out_bits[size_t(pos >> 2) * g.Dw + oword] = mine;
                } else {
                    uint32_t mk[4] = {0u, 0u, 0u, 0u};  // four independent select chains
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t w = __ballot_sync(0xffffffffu, (int(v[j]) >= Tu) != flip);
                        if (lane == j) mk[j & 3] = w;
                    }
                    mine = (mk[0] | mk[1]) | (mk[2] | mk[3]);
                    const int pos = nt * kSwN + col0 + cc * 32 + lane;
                    if (wvalid && pos < g.rows) g.out_bits[size_t(pos) * g.Dw + oword] = mine;
                }
            };
            tmem_ld32(tbase, va);
            tmem_ld_wait();
            tmem_ld32(tbase + 32, vb);
            emit(va, 0);
            tmem_ld_wait();
            tmem_ld32(tbase + 64, va);
            emit(vb, 1);
            tmem_ld_wait();
            tmem_ld32(tbase + 96, vb);
            emit(va, 2);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);  // accumulator free before the last words
            emit(vb, 3);
        }
        if (warp == 2 && lane == 0) wc.flush(g.dbg, 2);
    } else {
        // ------------------------------------------------------------ activation producers (B)
        // thread pt owns tile rows pt and pt + 128 (two positions); loads kPF blocks ahead
        const int pt = threadIdx.x - 6 * 32;
        constexpr int NT = PT ? PT : kMaxPixTaps;
        using Raw = typename std::conditional<IN == FIN_BITS, uint4, PixRaw<NT>>::type;
        constexpr int kPF = 2;
        int stage = 0;
        uint32_t phase = 0;
        int t_ld = unit, kb_ld = 0;
        RowCtx rc[2];
        auto set_rows = [&]() {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int b = 0, oy = 0, ox = 0;
                rc[h].valid = t_ld < tiles && decode_row(g, (t_ld / m_tiles) * kSwN + pt + 128 * h, b, oy, ox);
                rc[h].pix = b * g.H, rc[h].y0 = oy * g.SH, rc[h].x0 = ox * g.SW;
            }
        };
        set_rows();
        Raw pf[kPF][2];
        bool pv[kPF][2];
        auto next_load = [&](Raw (&dst)[2], bool (&v)[2]) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                v[h] = rc[h].valid;
                if constexpr (IN == FIN_BITS)
                    dst[h] = t_ld < tiles ? load_bits(g, ftab, rc[h], kb_ld) : make_uint4(0, 0, 0, 0);
                else
                    dst[h] = load_pix<false, NT>(g, ftab, rc[h]);
            }
            if (t_ld < tiles && ++kb_ld == KB) {
                t_ld += units;
                kb_ld = 0;
                set_rows();
            }
        };
#pragma unroll
        for (int i = 0; i < kPF; ++i) next_load(pf[i], pv[i]);
        const bool one_step = KB == 1 && g.kq_last == 1;  // e.g. the 27-bit first layer: 32 bytes per row
        WaitClock wc;
        for (int t = unit; t < tiles; t += units) {
            for (int kb = 0; kb < KB; ++kb) {
                uint4 u[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if constexpr (IN == FIN_BITS)
                        u[h] = pf[0][h];
                    else
                        u[h] = gather_pix(g, pf[0][h], pv[0][h]);
                }
#pragma unroll
                for (int i = 0; i < kPF - 1; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h) pf[i][h] = pf[i + 1][h], pv[i][h] = pv[i + 1][h];
                next_load(pf[kPF - 1], pv[kPF - 1]);
                wc.wait(&empty[stage], phase ^ 1, 0);
                const uint32_t tile = smem_u32(sX + size_t(stage) * kSwN * kKB);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (g.dbg_mode & 1) break;  // profiling: no stores (results invalid)
                    if (one_step)
                        put_word(tile, pt + 128 * h, 0, u[h].x);  // the MMA reads the first 32 bytes only
                    else
                        store_bits(tile, pt + 128 * h, u[h]);
                }
                if (!(g.dbg_mode & 8)) fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[stage]);
                if (++stage == kStages) stage = 0, phase ^= 1;
            }
        }
        if (pt == 0) wc.flush(g.dbg, 3);
    }

    if (g.tl && warp == 1 && lane == 0) g.tl[blockIdx.x * 4 + 1] = gtimer();
    __syncwarp();  // reconverge role-divergent lanes: bar.sync counts a partial warp as whole
    tc_fence_before();
    __syncthreads();  // (TMEM: deallocated by the MMA warp)
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 3] = gtimer();
}

template <int IN, int PT>
int launch_swap_t(const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    auto kern = fused_swap_kernel<IN, PT>;
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSwSmem)));
        attr_set = true;
    }
    const int tiles = int(ceil_div(size_t(g.D), size_t(kRows)) * ceil_div(size_t(g.rows), size_t(kSwN)));
    const int grid = std::min(tiles, num_sms());
    static const int pdl = getenv("BNN_PDL") ? atoi(getenv("BNN_PDL")) : 0;
    FusedGeom gd = g;
    gd.tl = fused_timeline_slot(1);
    if (gd.tl) g_tl_names.push_back("swap D=" + std::to_string(g.D) + " KB=" + std::to_string(g.KB));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSwSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl == 2 ? 0 : 1;
    static const int prof = getenv("BNN_FUSED_PROFILE") ? atoi(getenv("BNN_FUSED_PROFILE")) : 0;
    unsigned long long* dbg = nullptr;
    if (prof) {
        BNN_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
        BNN_CUDA(cudaMemset(dbg, 0, 16 * sizeof(unsigned long long)));
        gd.dbg = dbg;
        gd.dbg_mode = prof >> 1;
    }
    BNN_CUDA(cudaLaunchKernelEx(&cfg, kern, tm, gd));
    BNN_TRY(launch_check("fused_swap_kernel"));
    if (prof) {
        unsigned long long h[16];
        BNN_CUDA(cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost));
        cudaFree(dbg);
        const double n = double(grid);
        fprintf(stderr,
                "[swap in=%d rows=%d D=%d KB=%d grid=%d] per-CTA kcycles: total %.1f | tma wait %.1f | mma wait-acc %.1f "
                "wait-full %.1f | epi wait %.1f | prod wait %.1f\n",
                IN, g.rows, g.D, g.KB, grid, h[3] / n / 1e3, h[0] / n / 1e3, h[4] / n / 1e3, h[5] / n / 1e3,
                h[8] / n / 1e3, h[12] / n / 1e3);
    }
    return BNN_OK;
}

// ---------------------------------------------------------------------------------------------
// Pixel-input first conv with K = T*C <= 32 (the 3x3 RGB layer: K = 27) on the CUDA cores.
// One patch is one word, so the layer is one XOR + POPC per (position, channel): 33.5 M popcounts
// at batch 256, against a tensor-core launch that issues a single K=32 MMA per tile and is bound
// by its epilogue and pixel gathers. With the patch x and channel d's weights w_d as K-bit words
// (1 = +1; bits >= K are 0 in both), the reference's xnor value is a = K - 2 p, p = popc(x ^ w_d)
// (kernels.hpp:46-54), and its float decision sign(htanh(fmaf(scale, float(a) + bias, shift)))
// is (a >= T_d) ^ flip_d (prep_params_kernel). In the accumulator form a >= T_d <=> u >= Tu_d
// with a = 2u - S_d, so a >= T_d <=> p <= (K + S_d)/2 - Tu_d = P_d (K + S_d = 2 * #(+1 weights)
// is even): one compare per channel with no per-position term. A 2x2 max pool is the OR of the
// four (a >= T_d) before the flip (network.cpp:133-149: max of the floats = float of the max
// integer), i.e. min of the four popcounts <= P_d.
// One thread per output (pooled) position; the patch is gathered tap-major / channel-minor (the
// engine K order, weights_to_bits_kernel's bit order), out-of-image taps read +1 on every
// channel (sign(0.0) of im2col's zero padding). The per-channel weights and thresholds are a
// kernel parameter (PixParams): with the channel loops unrolled, every w_d / P_d is a
// constant-bank operand of the XOR / compare, so a channel costs XOR, POPC, compare, select.
template <int DW, bool F32, bool POOL>
__global__ void __launch_bounds__(256, F32 ? (DW > 6 ? 1 : 4) : (DW > 6 ? 1 : 6)) pix_popc_kernel(const FusedGeom g, const PixParams pp) {
    // PDL: the next layer may start its prologue (it waits for this grid before reading);
    // this grid waits for the pixel packer's words
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t* pix = static_cast<const uint32_t*>(g.in);
    const float* xf = static_cast<const float*>(g.in);
    const uint32_t cmask = g.C == 32 ? ~0u : ((1u << g.C) - 1u);
    const int PH2 = g.OH / 2, PW2 = g.OW / 2;
    const int np = POOL ? g.B * PH2 * PW2 : g.B * g.OH * g.OW;  // output (pooled) positions
    const size_t HW = size_t(g.H) * g.W;
    constexpr int NS = POOL ? 4 : 1;
    for (int p = int(blockIdx.x * blockDim.x + threadIdx.x); p < np; p += int(gridDim.x * blockDim.x)) {
        uint32_t xs[NS];
#pragma unroll
        for (int sub = 0; sub < NS; ++sub) {
            int b, oy, ox;
            if (POOL) {  // pooled index ((b*OH/2 + py)*OW/2 + px), window element sub
                const int t = g.dv0.div(p), px = p - t * PW2;
                b = g.dv1.div(t);
                oy = 2 * (t - b * PH2) + (sub >> 1), ox = 2 * px + (sub & 1);
            } else {
                b = g.dv0.div(p);
                const int r = p - b * g.OH * g.OW;
                oy = g.dv1.div(r), ox = r - oy * g.OW;
            }
            const int y0 = oy * g.SH - g.PH, x0 = ox * g.SW - g.PW;
            uint32_t x = 0;
            int sh = 0;
            for (int kh = 0; kh < g.KH; ++kh) {
                const int iy = y0 + kh;
                const bool yin = unsigned(iy) < unsigned(g.H);
                const size_t row = (size_t(b) * (F32 ? g.C : 1) * g.H + iy) * g.W;
                for (int kw = 0; kw < g.KW; ++kw, sh += g.C) {
                    const int ix = x0 + kw;
                    uint32_t v = cmask;
                    if (yin && unsigned(ix) < unsigned(g.W)) {
                        if constexpr (F32) {  // bit c = (x[b, c, iy, ix] >= 0) (binarize.cpp:9)
                            v = 0;
                            for (int c = 0; c < g.C; ++c) v |= uint32_t(__ldg(xf + row + c * HW + ix) >= 0.0f) << c;
                        } else {
                            v = __ldg(pix + row + ix);
                        }
                    }
                    x |= v << sh;
                }
            }
            xs[sub] = x;
        }
        uint32_t o[DW];
#pragma unroll
        for (int w = 0; w < DW; ++w) {
            // bit j of nd = (c > P_d) = the sign of P_d - c (|P_d| <= 33, make_pix_params), shifted
            // in by a funnel shift: subtract + shift per channel instead of compare + select + or
            uint32_t nd = 0;
#pragma unroll
            for (int j = 31; j >= 0; --j) {
                const int d = 32 * w + j;
                int c = __popc(xs[0] ^ pp.w[d]);
                if (POOL) c = min(min(c, __popc(xs[1] ^ pp.w[d])), min(__popc(xs[2] ^ pp.w[d]), __popc(xs[3] ^ pp.w[d])));
                nd = __funnelshift_l(uint32_t(pp.p[d] - c), nd, 1);
            }
            o[w] = ~nd ^ pp.flip[w];
        }
        uint32_t* out = g.out_bits + size_t(p) * DW;
        if constexpr (DW % 4 == 0) {
#pragma unroll
            for (int w = 0; w < DW; w += 4) *reinterpret_cast<uint4*>(out + w) = make_uint4(o[w], o[w + 1], o[w + 2], o[w + 3]);
        } else if constexpr (DW % 2 == 0) {
#pragma unroll
            for (int w = 0; w < DW; w += 2) *reinterpret_cast<uint2*>(out + w) = make_uint2(o[w], o[w + 1]);
        } else {
#pragma unroll
            for (int w = 0; w < DW; ++w) out[w] = o[w];
        }
    }
}

// Float-input variant for unpooled layers whose per-image position count is a multiple of 256
// (bnn_set_fused_pix_popc(1)): each CTA takes 256 consecutive positions of one image, signs and
// packs the input rows they touch ONCE into shared memory (one word per pixel, coalesced float
// loads; rows outside the image read +1), then gathers the patches from there. This folds the
// pixel packer into the layer without pix_popc_kernel<F32>'s 27 scattered float loads per position.
template <int DW>
__global__ void __launch_bounds__(256) pix_tile_kernel(const FusedGeom g, const PixParams pp) {
    extern __shared__ uint32_t tile[];  // [rows][W] sign words of the input rows of this tile
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const float* xf = static_cast<const float*>(g.in);
    const uint32_t cmask = g.C == 32 ? ~0u : ((1u << g.C) - 1u);
    const int OHOW = g.OH * g.OW;
    const size_t HW = size_t(g.H) * g.W;
    const int ntiles = g.B * (OHOW / 256);
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int p0 = t * 256;
        const int b = p0 / OHOW, r0 = p0 - b * OHOW;
        const int oy0 = r0 / g.OW, oy1 = (r0 + 255) / g.OW;
        const int iy0 = oy0 * g.SH - g.PH;
        const int nw = ((oy1 - oy0) * g.SH + g.KH) * g.W;
        const float* xb = xf + size_t(b) * g.C * HW;
        __syncthreads();  // the previous tile's gathers are done
        for (int i = threadIdx.x; i < nw; i += 256) {
            const int ry = i / g.W, ix = i - ry * g.W, iy = iy0 + ry;
            uint32_t v = cmask;
            if (unsigned(iy) < unsigned(g.H)) {  // bit c = (x[b, c, iy, ix] >= 0) (binarize.cpp:9)
                v = 0;
                const float* src = xb + size_t(iy) * g.W + ix;
                for (int c = 0; c < g.C; ++c) v |= uint32_t(__ldg(src + c * HW) >= 0.0f) << c;
            }
            tile[i] = v;
        }
        __syncthreads();
        const int r = r0 + int(threadIdx.x);
        const int oy = g.dv1.div(r), ox = r - oy * g.OW;
        const int ty = (oy - oy0) * g.SH, x0 = ox * g.SW - g.PW;
        uint32_t x = 0;
        int sh = 0;
        for (int kh = 0; kh < g.KH; ++kh)
            for (int kw = 0; kw < g.KW; ++kw, sh += g.C) {
                const int ix = x0 + kw;
                x |= (unsigned(ix) < unsigned(g.W) ? tile[(ty + kh) * g.W + ix] : cmask) << sh;
            }
        uint32_t o[DW];
#pragma unroll
        for (int w = 0; w < DW; ++w) {
            uint32_t nd = 0;  // bit j = (popc > P_d), as in pix_popc_kernel
#pragma unroll
            for (int j = 31; j >= 0; --j) {
                const int d = 32 * w + j;
                nd = __funnelshift_l(uint32_t(pp.p[d] - __popc(x ^ pp.w[d])), nd, 1);
            }
            o[w] = ~nd ^ pp.flip[w];
        }
        uint32_t* out = g.out_bits + size_t(p0 + int(threadIdx.x)) * DW;
#pragma unroll
        for (int w = 0; w < DW; ++w) out[w] = o[w];
    }
}

// ---------------------------------------------------------------------------------------------
// Tiny final layers (a handful of logits, e.g. 1024 -> 10): one CUDA-core thread per logit,
// xnor-popcount over the packed input row, instead of a tensor-core launch whose fixed
// pipeline latency (TMA, expansion, 8 dependent K blocks on 2 CTAs) dominates: the layer
// is ~1 M bit-MACs. a = K - 2 popc(w ^ x) (kernels.hpp:46-54: pad bits are 0 on both sides),
// logit = float(a) + bias (kernels.cpp:90-107), written [D, ldo] (features x batch).
__global__ void logits_popc_kernel(const uint32_t* __restrict__ act, int Kw, int K, const uint32_t* __restrict__ wbits,
                                   const int4* __restrict__ prm, int D, int B, float* __restrict__ out, int ldo) {
    // PDL: resident while the previous layer drains (it triggers at entry); wait for its bits
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D * B) return;
    const int d = i / B, b = i - d * B;  // consecutive threads: consecutive images (coalesced logits)
    const uint4* x4 = reinterpret_cast<const uint4*>(act + size_t(b) * Kw);
    const uint4* w4 = reinterpret_cast<const uint4*>(wbits + size_t(d) * Kw);
    int acc = 0;
    if ((Kw & 3) == 0 && Kw <= 64) {  // every word's load in flight before the first popcount
        uint4 xv[16], wv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (4 * q < Kw) xv[q] = __ldg(x4 + q), wv[q] = __ldg(w4 + q);
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (4 * q < Kw)
                acc += __popc(xv[q].x ^ wv[q].x) + __popc(xv[q].y ^ wv[q].y) + __popc(xv[q].z ^ wv[q].z) + __popc(xv[q].w ^ wv[q].w);
    } else if ((Kw & 3) == 0) {
        for (int q = 0; q < Kw / 4; ++q) {
            const uint4 x = __ldg(x4 + q), w = __ldg(w4 + q);
            acc += __popc(x.x ^ w.x) + __popc(x.y ^ w.y) + __popc(x.z ^ w.z) + __popc(x.w ^ w.w);
        }
    } else {
        for (int q = 0; q < Kw; ++q) acc += __popc(__ldg(act + size_t(b) * Kw + q) ^ __ldg(wbits + size_t(d) * Kw + q));
    }
    out[size_t(d) * ldo + b] = __fadd_rn(__int2float_rn(K - 2 * acc), __int_as_float(__ldg(&prm[d].w)));
}

// The engine's int8 weights back to sign bits in the activation bit order (word q bit j = K
// position 32q + j). prep_weights_kernel's within-word byte order: byte 4s + j holds position
// 8j + s, so position j of a 32-group sits at byte 4 (j % 8) + j / 8. Positions >= K: 0.
__global__ void weights_to_bits_kernel(const int8_t* __restrict__ w8, int Kpad, int K, int D, int Kw,
                                       uint32_t* __restrict__ wbits) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= D * Kw) return;
    const int d = i / Kw, q = i - d * Kw;
    uint32_t w = 0;
    for (int j = 0; j < 32; ++j) {
        const int k = 32 * q + j;
        if (k < K && w8[size_t(d) * Kpad + 32 * q + 4 * (j % 8) + j / 8] > 0) w |= 1u << j;
    }
    wbits[i] = w;
}

// ---------------------------------------------------------------------------------------------
// FP4 swapped-operand conv (kind::mxf4, block-scaled e2m1): the same channels x positions tiles
// as fused_swap_kernel, but each operand element is a 4-bit e2m1 value instead of an int8:
// activations {0.0, 1.0} (codes 0x0, 0x2), weights {-1.0, +1.0} (0xA, 0x2), every block scale
// 2^0 (ue8m0 0x7F). Products and sums are exact in the f32 accumulator (|sum| <= K < 2^24),
// so the accumulator is the same integer u = sum bit * w as the int8 path. Half the operand
// bytes per K element (the swapped stage is shared-memory-bandwidth bound) and twice the MMA
// K per instruction (64).
//
// Layout: a 128-byte K-major SW128 row holds 256 elements; element e of a row is nibble e % 2
// (low first) of byte e / 2. An activation word (32 K positions) expands to 16 bytes in
// put_word4's order (8 ALU ops); the FP4 weights carry the same within-word permutation.
// TMEM: accumulators 2 x 224 columns (224 positions per tile), then 32 columns of scale
// factors for A and 32 for B, filled with 0x7F7F7F7F: every layout the MMA reads sees 2^0.
// NP positions per tile: 224 (4 producer warps, 2 rows per thread, 14 warps), 192 (6 producer
// warps, 1 row per thread, 16 warps) or 240 (8 producer warps, 1 row per thread, 4 epilogue
// warps, 14 warps; the scale factors take the last 32 TMEM columns). The producers bound this
// kernel, and an MMA costs about the same for any N here, so wide tiles fed by more producer
// warps win.
// CG = 2 (layers with >= 256 channels, packed-bit input, NP = 192): a CTA pair (cluster of 2)
// computes 256 channels x 192 positions with cta_group::2 M=256 instructions issued by the
// even CTA. Each CTA TMA-loads its own 128 weight rows and expands only its half of the
// positions (96 rows, two threads per row: one per 128-position half of the K block), so the
// activation expansion that bounds the CG = 1 kernel is done once per 256 channels instead of
// once per 128, with half the rows per thread. Each CTA holds its 128 channels x 192 positions
// of the accumulator in its own TMEM and runs the same epilogue.
template <int NP, int CG = 1>
constexpr size_t sw4_smem() {
    return 1024 + size_t(CG == 2 ? kStages2 : kStages) * (kRows + NP / CG) * kKB + 256 + kMaxQ * 8;
}
// SP = 1 (CG = 1, NP = 192): 12 producer warps, two threads per tile row (one per 128-position
// half of each K block), 22 warps in all.
// CG = 2, NP = 224: 8 producer warps (2-thread rows over 112 rows per CTA), 18 warps.
template <int NP, int SP = 0, int CG = 1>
constexpr int sw4_threads() {
    return SP ? (NP == 224 ? 768 : 704) : (CG == 2 && NP == 224) ? 576 : NP == 192 ? 512 : kThreads;
}

// 32 activation bits -> 32 e2m1 nibbles (16 bytes) at 16-byte chunk `chunk` of row r. Output
// word s takes bits s, s+4, ..., s+28 (one shift and one mask: nibble value 2 = e2m1 1.0), so
// element e = 8s + n of a 32-group holds K position 4n + s; the FP4 weights are permuted to
// match (prep_weights4_kernel).
__device__ __forceinline__ void put_word4(uint32_t tile, int r, int chunk, uint32_t w) {
    put_chunk(tile, r, chunk, (w << 1) & 0x22222222u, w & 0x22222222u, (w >> 1) & 0x22222222u,
              (w >> 2) & 0x22222222u);
}

// Issued by the whole converged warp (one elected lane), see mma_i8_w in umma.cuh.
template <int CG = 1>
__device__ __forceinline__ void mma_mxf4(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
    if constexpr (CG == 2) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
                d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
                d_tmem),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
            : "memory");
    }
}

// Block-scaled instruction descriptor (CUTLASS InstrDescriptorBlockScaled): E2M1 (MXF4
// format 1) for A and B, K-major, scale format UE8M0, K = 64, scale-factor ids 0.
__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);
}

template <int IN, int PT, int NP, int CG = 1, int SP = 0>
__global__ void __launch_bounds__(sw4_threads<NP, SP, CG>(), 1)
    fused_swap4_kernel(const __grid_constant__ CUtensorMap tmW4, const FusedGeom g) {
    static_assert(IN == FIN_BITS || IN == FIN_PIX, "packed-bit or pixel-packed input");
    static_assert(NP == 192 || NP == 224 || NP == 240, "tile positions");
    static_assert(CG == 1 || (CG == 2 && IN == FIN_BITS && (NP == 192 || NP == 224)), "CTA pairs: packed bits");
    static_assert(!SP || (CG == 1 && IN == FIN_BITS && (NP == 192 || NP == 224)), "split producers: packed bits");
    constexpr bool kSplit = CG == 2 || SP;  // two producer threads per tile row
    constexpr int kSw4N = NP;
    constexpr int kBH = NP / CG;  // activation rows this CTA expands per stage
    constexpr int kS = CG == 2 ? kStages2 : kStages;
    constexpr int kSfCol = NP == 240 ? 480 : 2 * kSw4N;  // SFA, then SFB: 16 columns each at NP 240
    constexpr int kProd = SP ? (NP == 224 ? 14 : 12) : (CG == 2 && NP == 224) ? 8 : NP == 240 ? 8 : NP == 192 ? 6 : 4;  // producer warps
    constexpr int kEpi = NP == 240 ? 4 : 8;                   // epilogue warps
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* sW = smem_raw + (base - raw);           // [kS][128 * 128] weights (A)
    uint8_t* sX = sW + size_t(kS) * kRows * kKB;     // [kS][kBH * 128] activations (B)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sX + size_t(kS) * kBH * kKB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kS;
    uint64_t* tfull = bars + 2 * kS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int2* ftab = reinterpret_cast<int2*>(bars + 32);

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.launch_dependents;");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 0] = gtimer();
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
    const int units = gridDim.x / CG, unit = blockIdx.x / CG;
    const int m_tiles = (g.D + kRows * CG - 1) / (kRows * CG);
    const int n_tiles = (g.rows + kSw4N - 1) / kSw4N;
    const int tiles = m_tiles * n_tiles;
    const int KB = g.kb4;  // 256-element K blocks
    // barrier the producers / TMA / epilogue signal: the even CTA's (shared::cluster address)
    auto leader = [&](uint64_t* bar) { return CG == 2 ? mapa(smem_u32(bar), 0) : smem_u32(bar); };

    if (threadIdx.x == 0) {
        tma_prefetch(&tmW4);
        for (int s = 0; s < kS; ++s) {
            mbar_init(&full[s], CG * (kProd + 1));
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], CG * kEpi);
        }
        fence_mbar_init();
    }
    if (IN == FIN_BITS) {
        const int kw_total = (g.K + 31) >> 5;
        for (int q = threadIdx.x; q < 8 * KB; q += blockDim.x) {
            int2 e = make_int2(0, -1);
            if (q < kw_total) {
                const int tap = q / g.Cw, cw = q - tap * g.Cw, ky = tap / g.KW, kx = tap - ky * g.KW;
                e = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), cw);
            }
            ftab[q] = e;
        }
    } else {
        for (int tap = threadIdx.x; tap < g.KH * g.KW; tap += blockDim.x) {
            const int ky = tap / g.KW, kx = tap - ky * g.KW;
            ftab[tap] = make_int2(((ky - g.PH) << 16) | ((kx - g.PW) & 0xffff), 0);
        }
    }
    if (warp == 1) {
        if (CG == 2)
            tmem_alloc_cg2<512>(tmem_slot);
        else
            tmem_alloc<512>(tmem_slot);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    if (warp >= 2 && warp < 6) {  // scale factors: every byte of columns [448, 512) = 2^0
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0x7F7F7F7Fu;
        const uint32_t lane_base = tmem_base + (uint32_t(32 * (warp & 3)) << 16);
        tmem_st32(lane_base + kSfCol, v);
        if (NP != 240) tmem_st32(lane_base + kSfCol + 32, v);
        tmem_st_wait();
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    // CG = 2: the peer's barriers are initialised and its scale factors written before any
    // remote arrive or pair MMA
    if (CG == 2) cluster_sync();
    tc_fence_after();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 2] = gtimer();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            WaitClock wc;
            for (int t = unit; t < tiles; t += units) {
                const int mt = t % m_tiles;
                for (int kb = 0; kb < KB; ++kb) {
                    wc.wait(&empty[stage], phase ^ 1, 0);
                    uint8_t* dst = sW + size_t(stage) * kRows * kKB;
                    if (CG == 2) {
                        const uint32_t fb = leader(&full[stage]);
                        mbar_arrive_expect_tx_cluster(fb, kRows * kKB);
                        tma_load_2d_cg2(&tmW4, fb, dst, kb * kKB, (mt * CG + int(rank)) * kRows);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], kRows * kKB);
                        tma_load_2d(&tmW4, &full[stage], dst, kb * kKB, mt * kRows);
                    }
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
            }
            wc.flush(g.dbg, 0);
            if (CG == 2) {
                // every stage's last release (the pair MMA's multicast commit) has landed in
                // this CTA's barriers before it may exit
                for (int k = 0; k < kS; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (++stage == kS) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_mxf4(kRows * CG, kSw4N);
        int stage = 0;
        uint32_t phase = 0;
        int i = 0;
        WaitClock wc;
        for (int t = unit; t < tiles && (CG == 1 || rank == 0); t += units, ++i) {
            const int acc = i & 1;
            wc.wait(&tempty[acc], ((i >> 1) & 1) ^ 1, 0);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + uint32_t(acc * kSw4N);
            for (int kb = 0; kb < KB; ++kb) {
                wc.wait(&full[stage], phase, 1);
                tc_fence_after();
                {  // the converged warp issues (one elected lane): see mma_i8_w
                    const uint32_t a0 = smem_u32(sW + size_t(stage) * kRows * kKB);
                    const uint32_t b0 = smem_u32(sX + size_t(stage) * kBH * kKB);
                    const int nk = kb == KB - 1 ? g.kq4 : kKB / 32;  // 64-element K steps past K: zeros
#pragma unroll
                    for (int k = 0; k < kKB / 32; ++k) {
                        if (k >= nk) break;
                        mma_mxf4<CG>(d_tmem, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                     tmem_base + kSfCol, tmem_base + kSfCol + (NP == 240 ? 16 : 32),
                                     (kb != 0 || k != 0));
                    }
                    if (CG == 2) {
                        mma_commit_cg2_mc_w(&empty[stage], 3);  // both CTAs' slots free
                        if (kb == KB - 1) mma_commit_cg2_mc_w(&tfull[acc], 3);
                    } else {
                        mma_commit_w(&empty[stage]);
                        if (kb == KB - 1) mma_commit_w(&tfull[acc]);
                    }
                }
                __syncwarp();
                if (++stage == kS) stage = 0, phase ^= 1;
            }
        }
        if (lane == 0) wc.flush(g.dbg, 1);
        if (CG == 1 || rank == 0) {
            // the epilogue has read the last accumulators (CG = 2: both CTAs' epilogue warps,
            // whose remote arrives have then all landed here)
            for (int k = 0; k < 2; ++k, ++i) mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);
            tc_fence_after();
            if (CG == 1) tmem_dealloc<512>(tmem_base);
        }  // CG = 2: both CTAs deallocate after the final cluster barrier
    } else if (warp < 6 || (kEpi == 8 && warp >= 10 && warp < 14)) {
        WaitClock wc;
        // epilogue: lane = channel, ceil(NP/32) chunks of 32 positions (split over warps 2-5 /
        // 10-13 when there are 8 epilogue warps)
        const int q = warp & 3;
        constexpr int NC = (kSw4N + 31) / 32, NH = kEpi == 8 ? (NC + 1) / 2 : NC;
        const int c0 = warp >= 10 ? NH : 0, c1 = warp >= 10 ? NC : NH;
        int i = 0;
        for (int t = unit; t < tiles; t += units, ++i) {
            const int acc = i & 1;
            const int mt = t % m_tiles, nt = t / m_tiles;
            const int m0 = (mt * CG + int(rank)) * kRows;  // this CTA's first channel
            const int c = m0 + q * 32 + lane;
            const bool wvalid = m0 + q * 32 < g.D;
            const int4 pc = wvalid ? __ldg(g.prm + c) : make_int4(0x7fffffff, 0, 0, 0);
            const float Tf = float(pc.x);  // exact: |Tu| <= K < 2^24
            const bool flip = pc.y != 0;
            const int oword = m0 / 32 + q;
            wc.wait(&tfull[acc], (i >> 1) & 1, 0);
            tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * kSw4N);
            uint32_t va[32];
            for (int cc = c0; cc < c1; ++cc) {
                tmem_ld32(tbase + uint32_t(cc * 32), va);
                tmem_ld_wait();
                if (cc == c1 - 1) {  // accumulator free before the last words
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 2)
                            mbar_arrive_cluster(leader(&tempty[acc]));
                        else
                            mbar_arrive(&tempty[acc]);
                    }
                }
                uint32_t mine = 0;
                if (g.pool) {
                    // 32 columns = 8 pool windows (pool-major: 4 adjacent columns). The pooled
                    // bit OR_k((u_k >= T) ^ flip) is (max_k u_k >= T) without flip and
                    // (min_k u_k < T) with it: one compare and one ballot per window.
#pragma unroll
                    for (int p = 0; p < 8; ++p) {
                        const float a = __uint_as_float(va[4 * p]), b = __uint_as_float(va[4 * p + 1]);
                        const float c = __uint_as_float(va[4 * p + 2]), d = __uint_as_float(va[4 * p + 3]);
                        const float m = flip ? fminf(fminf(a, b), fminf(c, d)) : fmaxf(fmaxf(a, b), fmaxf(c, d));
                        const uint32_t w = __ballot_sync(0xffffffffu, (m >= Tf) != flip);
                        if (lane == p) mine = w;
                    }
                    const int q0 = cc * 32 + 4 * lane;  // lane p < 8: window p's first column
                    if (wvalid && lane < 8 && q0 < kSw4N && nt * kSw4N + q0 < g.rows)
                        g.out_bits[size_t((nt * kSw4N + q0) >> 2) * g.Dw + oword] = mine;
                } else {
                    uint32_t mk[4] = {0u, 0u, 0u, 0u};  // four independent select chains
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t w = __ballot_sync(0xffffffffu, (__uint_as_float(va[j]) >= Tf) != flip);
                        if (lane == j) mk[j & 3] = w;
                    }
                    mine = (mk[0] | mk[1]) | (mk[2] | mk[3]);
                    const int pos = (cc * 32 + lane < kSw4N) ? nt * kSw4N + cc * 32 + lane : g.rows;  // past the tile: none
                    if (wvalid && pos < g.rows) g.out_bits[size_t(pos) * g.Dw + oword] = mine;
                }
            }
        }
        if (warp == 2 && lane == 0) wc.flush(g.dbg, 2);
    } else {
        // producers: thread pt owns tile row pt (NP = 192: warps 6-9, 14-15) or rows pt and
        // pt + 128 (NP = 224: warps 6-9); blocks are loaded kPF ahead
        const int pt = NP == 240 ? (warp - 6) * 32 + lane : (warp < 10 ? warp - 6 : warp - 10) * 32 + lane;
        // CG = 2: thread pt expands row pt % 96 of this CTA's half, K words 4 * (pt / 96) .. +3
        // of each 8-word block
        const int prow = kSplit ? pt % kBH : pt, phalf = kSplit ? pt / kBH : 0;
        const bool one = kSplit ? pt < 2 * kBH : pt < kSw4N;  // NP = 240: the last warp has 16 rows
        const bool two = NP == 224 && !kSplit && pt + 128 < kSw4N;
        constexpr int NT = PT ? PT : kMaxPixTaps;
        struct Bits8 {
            uint4 lo, hi;
        };
        using Raw = typename std::conditional<IN == FIN_BITS, Bits8, PixRaw<NT>>::type;
        // kPF blocks loaded ahead. (Rotating the slots in place, the loop unrolled kPF times,
        // measured slower here: 1.38 M vs 1.14 M cycles per CTA for conv 128->128 at B=4096.)
        constexpr int kPF = 2;
        int stage = 0;
        uint32_t phase = 0;
        const bool one_step = KB == 1 && g.kq4 == 1 && IN == FIN_PIX;  // <= 64 K positions: 32 bytes per row
        WaitClock wc;
        int t_ld = unit, kb_ld = 0;
        RowCtx rc[2];
        auto set_rows = [&]() {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int b = 0, oy = 0, ox = 0;
                rc[h].valid = t_ld < tiles && (h == 0 ? one : two) &&
                              decode_row(g, (t_ld / m_tiles) * kSw4N + int(rank) * kBH + prow + 128 * h, b, oy, ox);
                rc[h].pix = b * g.H, rc[h].y0 = oy * g.SH, rc[h].x0 = ox * g.SW;
            }
        };
        set_rows();
        Raw pf[kPF][2];
        bool pv[kPF][2];
        auto next_load = [&](Raw (&dst)[2], bool (&v)[2]) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                v[h] = rc[h].valid;
                if constexpr (IN == FIN_BITS && kSplit) {
                    dst[h].lo = t_ld < tiles ? load_bits(g, ftab, rc[h], 2 * kb_ld + phalf) : make_uint4(0, 0, 0, 0);
                    dst[h].hi = make_uint4(0, 0, 0, 0);
                } else if constexpr (IN == FIN_BITS) {
                    dst[h].lo = t_ld < tiles ? load_bits(g, ftab, rc[h], 2 * kb_ld) : make_uint4(0, 0, 0, 0);
                    dst[h].hi = t_ld < tiles ? load_bits(g, ftab, rc[h], 2 * kb_ld + 1) : make_uint4(0, 0, 0, 0);
                } else {
                    dst[h] = load_pix<false, NT>(g, ftab, rc[h]);
                }
            }
            if (t_ld < tiles && ++kb_ld == KB) {
                t_ld += units;
                kb_ld = 0;
                set_rows();
            }
        };
#pragma unroll
        for (int i = 0; i < kPF; ++i) next_load(pf[i], pv[i]);
        int pending = -1;  // a filled stage whose fence + release waits for the next one
        auto release = [&](int st) {
            if (CG == 2)
                mbar_arrive_cluster(leader(&full[st]));
            else
                mbar_arrive(&full[st]);
        };
        for (int t = unit; t < tiles; t += units) {
            for (int kb = 0; kb < KB; ++kb) {
                uint4 lo[2], hi[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if constexpr (IN == FIN_BITS) {
                        lo[h] = pf[0][h].lo, hi[h] = pf[0][h].hi;
                    } else {
                        lo[h] = gather_pix(g, pf[0][h], pv[0][h]);
                        hi[h] = make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int i = 0; i < kPF - 1; ++i)
#pragma unroll
                    for (int h = 0; h < 2; ++h) pf[i][h] = pf[i + 1][h], pv[i][h] = pv[i + 1][h];
                next_load(pf[kPF - 1], pv[kPF - 1]);
                wc.wait(&empty[stage], phase ^ 1, 0);
                const uint32_t tile = smem_u32(sX + size_t(stage) * kBH * kKB);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if ((h == 1 && !two) || (h == 0 && !one)) break;  // no such tile row
                    if (g.dbg_mode & 1) break;  // profiling: no stores (results invalid)
                    if constexpr (kSplit) {
                        put_word4(tile, prow, 4 * phalf + 0, lo[0].x);
                        put_word4(tile, prow, 4 * phalf + 1, lo[0].y);
                        put_word4(tile, prow, 4 * phalf + 2, lo[0].z);
                        put_word4(tile, prow, 4 * phalf + 3, lo[0].w);
                        break;
                    }
                    const int r = pt + 128 * h;
                    put_word4(tile, r, 0, lo[h].x);
                    put_word4(tile, r, 1, lo[h].y);
                    if (one_step) continue;  // the MMA reads the first 32 bytes only
                    put_word4(tile, r, 2, lo[h].z);
                    put_word4(tile, r, 3, lo[h].w);
                    put_word4(tile, r, 4, hi[h].x);
                    put_word4(tile, r, 5, hi[h].y);
                    put_word4(tile, r, 6, hi[h].z);
                    put_word4(tile, r, 7, hi[h].w);
                }
                // one proxy fence per two stages (the fence cost ~11 % of this role's time at
                // batch 256): the even stage of a pair is released together with the odd one
                if (pending >= 0) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        release(pending);
                        release(stage);
                    }
                    pending = -1;
                } else {
                    pending = stage;
                }
                if (++stage == kS) stage = 0, phase ^= 1;
            }
        }
        if (pending >= 0) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) release(pending);
        }
        if (pt == 0) wc.flush(g.dbg, 3);
    }

    if (CG == 1 && g.tl && warp == 1 && lane == 0) g.tl[blockIdx.x * 4 + 1] = gtimer();
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 3] = gtimer();
    if (CG == 2) {
        // Every cross-CTA operation has landed (the drains above: the leader saw all remote
        // arrives, each CTA saw all multicast commits), so the teardown barrier needs no
        // release of this CTA's global stores.
        cluster_sync_relaxed();
        if (warp == 1) tmem_dealloc_cg2<512>(tmem_base);
        if (g.tl && warp == 1 && lane == 0) g.tl[blockIdx.x * 4 + 1] = gtimer();  // k1: TMEM released
    }
}

template <int IN, int PT, int NP, int CG = 1, int SP = 0>
int launch_swap4_t(const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    auto kern = fused_swap4_kernel<IN, PT, NP, CG, SP>;
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sw4_smem<NP, CG>())));
        attr_set = true;
    }
    const int tiles = int(ceil_div(size_t(g.D), size_t(kRows * CG)) * ceil_div(size_t(g.rows), size_t(NP)));
    const int grid = std::min(tiles, num_sms() / CG) * CG;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(unsigned(sw4_threads<NP, SP, CG>()));
    cfg.dynamicSmemBytes = sw4_smem<NP, CG>();
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CG;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CG == 2 ? 2 : 1;
    static const int prof = getenv("BNN_FUSED_PROFILE") ? atoi(getenv("BNN_FUSED_PROFILE")) : 0;
    FusedGeom gd = g;
    unsigned long long* dbg = nullptr;
    if (prof) {
        BNN_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
        BNN_CUDA(cudaMemset(dbg, 0, 16 * sizeof(unsigned long long)));
        gd.dbg = dbg;
        gd.dbg_mode = prof >> 1;
    }
    gd.tl = fused_timeline_slot(1);
    if (gd.tl) g_tl_names.push_back("swap4 cg=" + std::to_string(CG) + " D=" + std::to_string(g.D) + " KB4=" + std::to_string(g.kb4));
    BNN_CUDA(cudaLaunchKernelEx(&cfg, kern, tm, gd));
    BNN_TRY(launch_check("fused_swap4_kernel"));
    if (prof) {
        unsigned long long h[16];
        BNN_CUDA(cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost));
        cudaFree(dbg);
        const double n = double(grid);
        fprintf(stderr,
                "[swap4 in=%d cg=%d rows=%d D=%d KB4=%d grid=%d] per-CTA kcycles: total %.1f | tma wait %.1f | mma wait-acc %.1f "
                "wait-full %.1f | epi wait %.1f | prod wait %.1f | role totals mma %.1f epi %.1f prod %.1f\n",
                IN, CG, g.rows, g.D, g.kb4, grid, h[3] / n / 1e3, h[0] / n / 1e3, h[4] / n / 1e3, h[5] / n / 1e3,
                h[8] / n / 1e3, h[12] / n / 1e3, h[7] / n / 1e3, h[11] / n / 1e3, h[15] / n / 1e3);
    }
    return BNN_OK;
}

// Build-time FP4 weights: the int8 +-1 rows (engine K order, int8 within-word permutation:
// position b of a 32-group at byte 4 (b % 8) + b / 8) -> e2m1 nibbles in put_word4's order
// (element e of a 32-group holds position 4 (e % 8) + e / 8), [Dpad, Kpad4 / 2] bytes;
// positions >= K are 0.0.
__global__ void prep_weights4_kernel(const int8_t* __restrict__ w8, int Kpad, int K, int Dpad, int Kpad4,
                                     uint8_t* __restrict__ w4) {
    const size_t total = size_t(Dpad) * (Kpad4 / 2);
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int d = int(i / (Kpad4 / 2)), e0 = int(i % (Kpad4 / 2)) * 2;
        uint8_t v = 0;
        for (int h = 0; h < 2; ++h) {
            const int e = e0 + h, q = e >> 5, el = e & 31;
            const int bb = 4 * (el % 8) + el / 8, k = 32 * q + bb;  // the K position element e holds
            if (k >= K) continue;
            const int8_t s = w8[size_t(d) * Kpad + 32 * q + 4 * (bb % 8) + bb / 8];
            const uint8_t code = s > 0 ? 0x2 : s < 0 ? 0xA : 0x0;
            v |= uint8_t(code << (4 * h));
        }
        w4[i] = v;
    }
}

// Build-time weight preparation: reference packed rows (pack_rows(sign(flatten(W))),
// K order r) -> int8 +-1 rows [Dpad, Kpad] in the engine's K order. With T > 1 the engine
// order is tap-major (k' = tap*C + c) and the reference order is channel-major
// (r = c*T + tap): conv taps (lowering.hpp:8-10) or the spatial positions of
// flatten_to_columns (network.cpp:177-184). T == 1 is the identity. With perm_bits, byte
// position 4s + j inside every 32-position group holds logical position 8j + s, the order
// put_word() emits activation bits in. Rows >= D and columns >= K are 0.
//
// Operand encoding: activations enter the MMA as their bits {0, 1} (not +-1), so the
// accumulator is u = sum_k bit_k w_k and the reference's value is a = 2u - S_d with
// S_d = sum_k w_k (prep_params_kernel). Everything stays exact integer arithmetic.
__global__ void prep_weights_kernel(const uint32_t* __restrict__ packed, size_t ldw, int D, int K, int C,
                                    int T, int perm_bits, int Kpad, size_t total, int8_t* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int d = int(i / Kpad), kb = int(i % Kpad);
        const int k = perm_bits ? ((kb & ~31) | (8 * (kb & 3) + ((kb >> 2) & 7))) : kb;
        int8_t v = 0;
        if (d < D && k < K) {
            const int rr = T > 1 ? (k % C) * T + k / C : k;
            v = ((packed[size_t(d) * ldw + (rr >> 5)] >> (rr & 31)) & 1u) ? 1 : -1;
        }
        out[i] = v;
    }
}

// Per output channel: S_d = sum of the prepared weights, and the integer threshold that
// reproduces the reference's float decision exactly. The reference binarizes
//     z(a) = fmaf(scale, float(a) + bias, shift)        (to_float, bias_add, affine_norm)
// with sign(htanh(z)) = (z >= 0). Rounding is monotone, so P(a) = (z(a) >= 0) is monotone in
// the integer a: P(a) = (a >= T) ^ flip for a T in [-K, K+1]. T and flip are found by
// evaluating P with the same IEEE operations (__fadd_rn, __fmaf_rn) at every a in [-K, K]
// and checking the step form for all of them; a channel that fails the check is reported
// (the engine then refuses to fuse). In the accumulator domain a = 2u - S_d, so
// a >= T  <=>  u >= ceil((T + S_d) / 2) = Tu.
__global__ void prep_params_kernel(const int8_t* __restrict__ w8, int Kpad, int D, int Dp, int K,
                                   const float* bias, const float* scale, const float* shift,
                                   int4* __restrict__ prm, int* bad) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= Dp) return;
    if (d >= D) {
        prm[d] = make_int4(0, 0, 0, 0);
        return;
    }
    int S = 0;
    for (int k = 0; k < Kpad; ++k) S += w8[size_t(d) * Kpad + k];
    const float b = bias[d], sc = scale ? scale[d] : 1.0f, sh = shift ? shift[d] : 0.0f;
    auto P = [&](int a) { return __fmaf_rn(sc, __fadd_rn(__int2float_rn(a), b), sh) >= 0.0f; };
    int T = K + 1;
    const bool p_lo = P(-K);
    int flip = p_lo ? 1 : 0;  // increasing predicate starts false; decreasing starts true
    for (int a = -K; a <= K; ++a)
        if (P(a) != p_lo) {
            T = a;
            break;
        }
    // P(a) = (a >= T) ^ flip must hold at every a (one step at most)
    for (int a = -K; a <= K; ++a)
        if (P(a) != (bool((a >= T) ? 1 : 0) != bool(flip))) {
            atomicExch(bad, 1);
            break;
        }
    const int Tu = (T + S + 1) >> 1;  // ceil((T + S) / 2), arithmetic shift = floor
    prm[d] = make_int4(Tu, flip, S, __float_as_int(b));
}

// First-layer encoder for FIN_PIX: the sign bits of a pixel's C <= 32 channels in one word,
// out[(b*H + y)*W + x] bit c = (x[b, c, y, x] >= 0) (binarize.cpp:9). Reads are coalesced per
// channel plane; 4 bytes written per pixel.
__global__ void pack_pixels_kernel(const float* __restrict__ x, int C, size_t HW, size_t total,
                                   uint32_t* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t b = i / HW, p = i - b * HW;
        const float* src = x + b * C * HW + p;
        uint32_t w = 0;
        for (int c = 0; c < C; ++c) w |= uint32_t(__ldg(src + c * HW) >= 0.0f) << c;
        out[i] = w;
    }
}

template <int BN, int IN, int EPI, int CG, int ATM, int PT = 0>
int launch_fused_t(const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    auto kern = fused_layer_kernel<BN, IN, EPI, CG, ATM, PT>;
    constexpr size_t smem = fused_smem<BN, CG, ATM>();
    static bool attr_set = false;  // per instantiation; the attribute is per function
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr_set = true;
    }
    const int m_tiles = (g.rows + kRows * CG - 1) / (kRows * CG);
    const int tiles = m_tiles * g.n_tiles * g.ksplit;
    // split-K: the ksplit CTAs of an output tile wait for each other, so every tile needs its
    // own co-resident CTA (one CTA per SM, grid = tiles <= SMs)
    if (g.ksplit > 1 && tiles > num_sms() / CG)
        return fail(BNN_E_CONFIG, "fused split-K: more tiles than SMs");
    const int grid = std::min(tiles, num_sms() / CG) * CG;
    static const int prof = getenv("BNN_FUSED_PROFILE") ? atoi(getenv("BNN_FUSED_PROFILE")) : 0;
    FusedGeom gd = g;
    static const int pdl = getenv("BNN_PDL") ? atoi(getenv("BNN_PDL")) : 0;  // 0 early, 1 late, 2 off
    gd.pdl_late = pdl == 1;
    gd.tl = fused_timeline_slot(1);
    if (gd.tl) g_tl_names.push_back("layer BN=" + std::to_string(BN) + " D=" + std::to_string(g.D) + " KB=" + std::to_string(g.KB));
    unsigned long long* dbg = nullptr;
    if (prof) {
        BNN_CUDA(cudaMalloc(&dbg, 16 * sizeof(unsigned long long)));
        BNN_CUDA(cudaMemset(dbg, 0, 16 * sizeof(unsigned long long)));
        gd.dbg = dbg;
        gd.dbg_mode = prof >> 1;  // 3: producer skips its stores, 5: epilogue skips its math, 17: no wait::st
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CG;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = pdl == 2 ? attr + 1 : attr;
    cfg.numAttrs = (CG == 2 ? 2 : 1) - (pdl == 2 ? 1 : 0);
    BNN_CUDA(cudaLaunchKernelEx(&cfg, kern, tm, gd));
    BNN_TRY(launch_check("fused_layer_kernel"));
    if (prof) {
        unsigned long long h[16];
        BNN_CUDA(cudaMemcpy(h, dbg, sizeof h, cudaMemcpyDeviceToHost));
        cudaFree(dbg);
        const double n = double(grid);
        fprintf(stderr,
                "[fused CG=%d BN=%d in=%d epi=%d rows=%d D=%d KB=%d grid=%d] per-CTA kcycles: total %.1f | tma wait "
                "%.1f | mma wait-acc %.1f wait-full %.1f | epi wait %.1f | prod wait %.1f\n",
                CG, BN, IN, EPI, g.rows, g.D, g.KB, grid, h[3] / n / 1e3, h[0] / n / 1e3, h[4] / n / 1e3 * CG,
                h[5] / n / 1e3 * CG, h[8] / n / 1e3, h[12] / n / 1e3);
    }
    return BNN_OK;
}

template <int IN, int EPI, int CG, int ATM, int PT = 0>
int launch_fused_bn(int BN, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    switch (BN) {
        case 32: return launch_fused_t<32, IN, EPI, CG, ATM, PT>(tm, g, s);
        case 64: return launch_fused_t<64, IN, EPI, CG, ATM, PT>(tm, g, s);
        case 128: return launch_fused_t<128, IN, EPI, CG, ATM, PT>(tm, g, s);
        case 256: return launch_fused_t<256, IN, EPI, CG, ATM, PT>(tm, g, s);
        default: return fail(BNN_E_CONFIG, "fused layer: unsupported BN " + std::to_string(BN));
    }
}


// CTA-local tiles only. (An int8 CTA-pair variant and a shared-memory A operand for packed-bit
// inputs were measured no faster (profiles/r01_*) and were removed; the float-input first layer
// keeps A in shared memory: its producers run the im2col gather.)
template <int IN, int EPI>
int launch_fused_cg(int cg, int BN, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    if (cg != 1) return fail(BNN_E_CONFIG, "fused layer: cta_group " + std::to_string(cg) + " is not supported");
    if constexpr (IN == FIN_PIX)  // 3x3 first layer: the 9-tap pixel gather
        if (g.KH * g.KW == 9) return launch_fused_bn<IN, EPI, 1, 1, 9>(BN, tm, g, s);
    if constexpr (IN != FIN_F32) return launch_fused_bn<IN, EPI, 1, 1>(BN, tm, g, s);
    return launch_fused_bn<IN, EPI, 1, 0>(BN, tm, g, s);
}

}  // namespace

int make_tmap_2d_s8(CUtensorMap* map, const void* base, size_t rows, size_t K, size_t ld, uint32_t box_rows);

int fused_prep_weights(const uint32_t* packed, size_t ldw, int D, int K, int C, int T, int perm_bits, int Dpad,
                       int Kpad, int8_t* out, cudaStream_t s) {
    const size_t total = size_t(Dpad) * Kpad;
    const unsigned grid = unsigned(std::min<size_t>(ceil_div(total, 256), size_t(num_sms()) * 16));
    prep_weights_kernel<<<grid, 256, 0, s>>>(packed, ldw, D, K, C, T, perm_bits, Kpad, total, out);
    return launch_check("prep_weights_kernel");
}

int fused_prep_params(const int8_t* w8, int Kpad, int D, int Dp, int K, const float* bias, const float* scale,
                      const float* shift, int4* prm, int* bad_dev, cudaStream_t s) {
    prep_params_kernel<<<unsigned(ceil_div(size_t(Dp), 64)), 64, 0, s>>>(w8, Kpad, D, Dp, K, bias, scale, shift,
                                                                        prm, bad_dev);
    return launch_check("prep_params_kernel");
}

int fused_make_tmap(CUtensorMap* map, const int8_t* w, int Dpad, int Kpad, int BN) {
    return make_tmap_2d_s8(map, w, size_t(Dpad), size_t(Kpad), size_t(Kpad), uint32_t(BN));
}

// Four pixels per thread (HW % 4 == 0, 16-byte aligned input): one 16-byte load per channel
// and one 16-byte store; 32-bit index math. C is a template constant for the 3-channel input.
template <int CT>
__global__ void pack_pixels4_kernel(const float4* __restrict__ x, int C, unsigned HW4, unsigned total4,
                                    uint4* __restrict__ out) {
    // PDL: a dependent first conv (pix_popc_kernel) may become resident now; it waits for this
    // grid's completion before reading the words
    asm volatile("griddepcontrol.launch_dependents;");
    const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total4) return;
    const unsigned b = i / HW4, p = i - b * HW4;
    const int nc = CT ? CT : C;
    const float4* src = x + size_t(b) * nc * HW4 + p;
    uint4 w = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int c = 0; c < (CT ? CT : 32); ++c) {
        if (!CT && c >= nc) break;
        const float4 v = __ldg(src + size_t(c) * HW4);
        w.x |= uint32_t(v.x >= 0.0f) << c;
        w.y |= uint32_t(v.y >= 0.0f) << c;
        w.z |= uint32_t(v.z >= 0.0f) << c;
        w.w |= uint32_t(v.w >= 0.0f) << c;
    }
    out[i] = w;
}

int launch_pack_pixels(const float* x, size_t B, int C, size_t HW, uint32_t* out, cudaStream_t s) {
    const size_t total = B * HW;
    if (!total) return BNN_OK;
    if (HW % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
        total / 4 < (size_t(1) << 31)) {
        const unsigned t4 = unsigned(total / 4), hw4 = unsigned(HW / 4);
        const unsigned grid = unsigned(ceil_div(size_t(t4), size_t(256)));
        if (C == 3)
            pack_pixels4_kernel<3><<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(x), C, hw4, t4,
                                                        reinterpret_cast<uint4*>(out));
        else
            pack_pixels4_kernel<0><<<grid, 256, 0, s>>>(reinterpret_cast<const float4*>(x), C, hw4, t4,
                                                        reinterpret_cast<uint4*>(out));
        return launch_check("pack_pixels4_kernel");
    }
    const unsigned grid = unsigned(std::min<size_t>(ceil_div(total, 256), size_t(num_sms()) * 8));
    pack_pixels_kernel<<<grid, 256, 0, s>>>(x, C, HW, total, out);
    return launch_check("pack_pixels_kernel");
}


void fused_timeline_name(const char* name) { g_tl_names.push_back(name); }

unsigned long long* fused_timeline_slot(int slots) {
    if (g_tl_used < 0 || g_tl_used + slots > kTlSlots) return nullptr;
    unsigned long long* p = g_tl + size_t(g_tl_used) * kTlCtas * 4;
    g_tl_used += slots;
    return p;
}

int fused_timeline(int op) {
    if (op == 1) {
        if (!g_tl) BNN_CUDA(cudaMalloc(&g_tl, size_t(kTlSlots) * kTlCtas * 4 * sizeof(unsigned long long)));
        BNN_CUDA(cudaMemset(g_tl, 0, size_t(kTlSlots) * kTlCtas * 4 * sizeof(unsigned long long)));
        g_tl_used = 0;
        g_tl_names.clear();
        return BNN_OK;
    }
    if (g_tl_used < 0) return BNN_OK;
    BNN_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(size_t(kTlSlots) * kTlCtas * 4);
    BNN_CUDA(cudaMemcpy(h.data(), g_tl, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (auto v : h)
        if (v && v < t0) t0 = v;
    for (int sl = 0; sl < g_tl_used; ++sl) {
        double mn[4], md[4], mx[4];
        for (int k = 0; k < 4; ++k) {
            std::vector<double> v;
            for (int c = 0; c < kTlCtas; ++c) {
                const unsigned long long x = h[(size_t(sl) * kTlCtas + c) * 4 + k];
                if (x) v.push_back((x - t0) * 1e-3);
            }
            std::sort(v.begin(), v.end());
            mn[k] = v.empty() ? -1 : v.front();
            md[k] = v.empty() ? -1 : v[v.size() / 2];
            mx[k] = v.empty() ? -1 : v.back();
        }
        fprintf(stderr, "[timeline %2d %-28s] us: k0 %7.1f/%7.1f/%7.1f | k1 %7.1f/%7.1f/%7.1f | k2 %7.1f/%7.1f/%7.1f | k3 %7.1f/%7.1f/%7.1f\n",
                sl, sl < int(g_tl_names.size()) ? g_tl_names[sl].c_str() : "", mn[0], md[0], mx[0], mn[1], md[1], mx[1],
                mn[2], md[2], mx[2], mn[3], md[3], mx[3]);
    }
    g_tl_used = -1;
    return BNN_OK;
}

int prep_logit_bits(const int8_t* w8, int Kpad, int K, int D, int Kw, uint32_t* wbits, cudaStream_t s) {
    const int n = D * Kw;
    weights_to_bits_kernel<<<unsigned((n + 127) / 128), 128, 0, s>>>(w8, Kpad, K, D, Kw, wbits);
    return launch_check("weights_to_bits_kernel");
}

int launch_logits_popc(const FusedGeom& g, const uint32_t* wbits, cudaStream_t s) {
    const int n = g.D * g.rows;
    if (n == 0) return BNN_OK;
    set_last_gemm("logits_popc");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((n + 127) / 128));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, logits_popc_kernel, static_cast<const uint32_t*>(g.in), g.Cw, g.K, wbits, g.prm, g.D,
                       g.rows, g.out_f32, g.ldo);  // errors: launch_check
    return launch_check("logits_popc_kernel");
}

bool pix_popc_ok(const FusedGeom& g) { return g.K <= 32 && g.Dw >= 1 && g.Dw <= 8 && g.D == 32 * g.Dw; }

// Grid: the resident CTA count (occupancy x SMs), positions strided over it, so every SM gets
// the same share (262144 positions at B=256 are ~1.15 waves of 256-thread CTAs: a tail wave of
// whole CTAs would leave most SMs idle).
template <int DW, bool F32, bool POOL>
static void launch_pix_k(const FusedGeom& g, const PixParams& pp, size_t np, cudaStream_t s) {
    static int per_sm = 0;
    if (!per_sm) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pix_popc_kernel<DW, F32, POOL>, 256, 0) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(std::min<size_t>(ceil_div(np, size_t(256)), size_t(num_sms()) * per_sm)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol)
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, pix_popc_kernel<DW, F32, POOL>, g, pp);  // errors: launch_check
}

template <bool F32, bool POOL>
static void launch_pix_dw(const FusedGeom& g, const PixParams& pp, size_t np, cudaStream_t s) {
    switch (g.Dw) {
#define BNN_PIX_CASE(n) \
    case n: launch_pix_k<n, F32, POOL>(g, pp, np, s); break;
        BNN_PIX_CASE(1) BNN_PIX_CASE(2) BNN_PIX_CASE(3) BNN_PIX_CASE(4)
        BNN_PIX_CASE(5) BNN_PIX_CASE(6) BNN_PIX_CASE(7) BNN_PIX_CASE(8)
#undef BNN_PIX_CASE
    }
}

int make_pix_params(const uint32_t* wbits_host, const int4* prm_host, int D, int K, PixParams* pp) {
    if (D > 256 || D % 32) return fail(BNN_E_CONFIG, "pix_popc: needs 32..256 output channels, a multiple of 32");
    memset(pp, 0, sizeof *pp);
    for (int d = 0; d < D; ++d) {
        const int4 e = prm_host[d];  // (Tu, flip, S, bias bits)
        pp->w[d] = wbits_host[d];
        // K + S is even; popc is in [0, 32], so clamping to [-1, 33] keeps every decision and
        // keeps P - popc far from overflow (the kernels take its sign)
        pp->p[d] = int(std::max<long long>(-1, std::min<long long>(33, (long long)(K + e.z) / 2 - e.x)));
        if (e.y) pp->flip[d / 32] |= 1u << (d % 32);
    }
    return BNN_OK;
}

int launch_pix_popc(const FusedGeom& g, const PixParams& pp, bool f32_in, cudaStream_t s) {
    if (!pix_popc_ok(g)) return fail(BNN_E_CONFIG, "pix_popc: needs K <= 32 and 32..256 output channels");
    const size_t np = g.pool ? size_t(g.B) * (g.OH / 2) * (g.OW / 2) : size_t(g.B) * g.OH * g.OW;
    if (np == 0) return BNN_OK;
    set_last_gemm("pix_popc");
    if (f32_in && !g.pool && (g.OH * g.OW) % 256 == 0) {  // shared-memory tile of packed input rows
        const int rows_max = (256 + g.OW - 2) / g.OW + 1;  // output rows 256 positions can span
        const size_t smem = size_t((rows_max - 1) * g.SH + g.KH) * g.W * sizeof(uint32_t);
        if (smem <= 48 * 1024) {
            const int ntiles = int(np / 256);
            // resident CTAs per SM for this DW and tile size (cached per DW): the grid strides
            // the tiles over exactly the CTAs that fit, so no partial second wave
            static int occ[9] = {};
            auto kern_of = [](int dw) -> const void* {
                switch (dw) {
                    case 1: return (const void*)pix_tile_kernel<1>;
                    case 2: return (const void*)pix_tile_kernel<2>;
                    case 3: return (const void*)pix_tile_kernel<3>;
                    case 4: return (const void*)pix_tile_kernel<4>;
                    case 5: return (const void*)pix_tile_kernel<5>;
                    case 6: return (const void*)pix_tile_kernel<6>;
                    case 7: return (const void*)pix_tile_kernel<7>;
                    default: return (const void*)pix_tile_kernel<8>;
                }
            };
            const int dwi = std::min(std::max(g.Dw, 1), 8);
            if (!occ[dwi]) {
                int n = 0;
                BNN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern_of(dwi), 256, smem));
                occ[dwi] = std::max(1, n);
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(unsigned(std::min(ntiles, num_sms() * occ[dwi])));
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol)
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            switch (g.Dw) {
#define BNN_TILE_CASE(n) \
    case n: cudaLaunchKernelEx(&cfg, pix_tile_kernel<n>, g, pp); break;
                BNN_TILE_CASE(1) BNN_TILE_CASE(2) BNN_TILE_CASE(3) BNN_TILE_CASE(4)
                BNN_TILE_CASE(5) BNN_TILE_CASE(6) BNN_TILE_CASE(7) BNN_TILE_CASE(8)
#undef BNN_TILE_CASE
            }
            return launch_check("pix_tile_kernel");
        }
    }
    if (f32_in) {
        if (g.pool) launch_pix_dw<true, true>(g, pp, np, s);
        else launch_pix_dw<true, false>(g, pp, np, s);
    } else {
        if (g.pool) launch_pix_dw<false, true>(g, pp, np, s);
        else launch_pix_dw<false, false>(g, pp, np, s);
    }
    return launch_check("pix_popc_kernel");
}

int prep_weights4(const int8_t* w8, int Kpad, int K, int Dpad, int Kpad4, uint8_t* w4, cudaStream_t s) {
    const size_t total = size_t(Dpad) * (Kpad4 / 2);
    const unsigned grid = unsigned(std::min<size_t>(ceil_div(total, 256), size_t(num_sms()) * 16));
    prep_weights4_kernel<<<grid, 256, 0, s>>>(w8, Kpad, K, Dpad, Kpad4, w4);
    return launch_check("prep_weights4_kernel");
}

// CTA pairs for the FP4 swapped kernel on layers with >= 256 channels (bnn_set_fused_fp4_pair,
// BNN_FP4_PAIR): -1 env / default on
int g_fp4_pair = -1;

int fused_set_fp4_pair(int mode) {
    if (mode < 0 || mode > 3) return fail(BNN_E_CONFIG, "fp4 pair mode: 0 off, 1 auto, 2 192 positions, 3 224");
    g_fp4_pair = mode;
    return BNN_OK;
}

int launch_swap4(int in_mode, const CUtensorMap& tm4, const FusedGeom& g, cudaStream_t s) {
    if (g.rows <= 0) return BNN_OK;
    set_last_gemm("fused_swap_mxf4");
    // tile positions (BNN_FP4_NP, 192 or 224): 192 measured fastest (conv 128->128 at B=4096,
    // cycles per CTA: 192 -> 0.94 M, 224 -> 1.14 M; a 240-position variant measured 1.18 M and was
    // removed)
    static const int np = getenv("BNN_FP4_NP") ? atoi(getenv("BNN_FP4_NP")) : 192;
    if (in_mode == FIN_PIX) {
        if (g.KH * g.KW == 9) return launch_swap4_t<FIN_PIX, 9, 224>(tm4, g, s);
        return launch_swap4_t<FIN_PIX, 0, 224>(tm4, g, s);
    }
    if (in_mode == FIN_BITS) {
        if (g_fp4_pair < 0) g_fp4_pair = getenv("BNN_FP4_PAIR") ? atoi(getenv("BNN_FP4_PAIR")) : 1;
        if (g_fp4_pair && g.D >= 2 * kRows && np == 192) {
            // 192 or 224 positions per pair tile: whichever needs fewer rounds of the pairs
            // (e.g. 16 x 16 x 256 rows: 4.6 -> 5 rounds at 192, 3.95 -> 4 at 224)
            const size_t pairs = size_t(num_sms() / 2), mp = ceil_div(size_t(g.D), size_t(2 * kRows));
            const size_t r192 = ceil_div(mp * ceil_div(size_t(g.rows), size_t(192)), pairs);
            const size_t r224 = ceil_div(mp * ceil_div(size_t(g.rows), size_t(224)), pairs);
            if (g_fp4_pair == 3 || (g_fp4_pair == 1 && r224 < r192)) return launch_swap4_t<FIN_BITS, 0, 224, 2>(tm4, g, s);
            return launch_swap4_t<FIN_BITS, 0, 192, 2>(tm4, g, s);
        }
        if (np == 224) return launch_swap4_t<FIN_BITS, 0, 224>(tm4, g, s);
        static const int sp = getenv("BNN_FP4_SPLIT") ? atoi(getenv("BNN_FP4_SPLIT")) : 1;
        if (np == 192 && sp) {
            // 192 or 224 positions per tile (14 producer warps at 224): fewer rounds wins
            const size_t sms = size_t(num_sms()), mt = ceil_div(size_t(g.D), size_t(kRows));
            const size_t r192 = ceil_div(mt * ceil_div(size_t(g.rows), size_t(192)), sms);
            const size_t r224 = ceil_div(mt * ceil_div(size_t(g.rows), size_t(224)), sms);
            if (g_fp4_pair == 3 || (g_fp4_pair == 1 && r224 < r192))
                return launch_swap4_t<FIN_BITS, 0, 224, 1, 1>(tm4, g, s);
            return launch_swap4_t<FIN_BITS, 0, 192, 1, 1>(tm4, g, s);
        }
        return launch_swap4_t<FIN_BITS, 0, 192>(tm4, g, s);
    }
    return fail(BNN_E_CONFIG, "FP4 swapped fused layer: packed-bit or pixel input only");
}

int launch_swap(int in_mode, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    if (g.rows <= 0) return BNN_OK;
    set_last_gemm("fused_swap_umma_i8");
    if (in_mode == FIN_PIX) {
        if (g.KH * g.KW == 9) return launch_swap_t<FIN_PIX, 9>(tm, g, s);
        return launch_swap_t<FIN_PIX, 0>(tm, g, s);
    }
    if (in_mode == FIN_BITS) return launch_swap_t<FIN_BITS, 0>(tm, g, s);
    return fail(BNN_E_CONFIG, "swapped fused layer: packed-bit or pixel input only");
}

int launch_fused(int cg, int BN, int in_mode, int epi, const CUtensorMap& tm, const FusedGeom& g, cudaStream_t s) {
    if (g.rows <= 0) return BNN_OK;
    set_last_gemm(in_mode != FIN_F32 ? "fused_umma_i8_tmem_a" : "fused_umma_i8");
    if (in_mode == FIN_PIX) {
        if (epi == FEPI_BITS) return launch_fused_cg<FIN_PIX, FEPI_BITS>(cg, BN, tm, g, s);
        return launch_fused_cg<FIN_PIX, FEPI_NCHW>(cg, BN, tm, g, s);
    }
    if (in_mode == FIN_BITS) {
        if (epi == FEPI_BITS) return launch_fused_cg<FIN_BITS, FEPI_BITS>(cg, BN, tm, g, s);
        if (epi == FEPI_LOGITS) return launch_fused_cg<FIN_BITS, FEPI_LOGITS>(cg, BN, tm, g, s);
        return launch_fused_cg<FIN_BITS, FEPI_NCHW>(cg, BN, tm, g, s);
    }
    if (epi == FEPI_BITS) return launch_fused_cg<FIN_F32, FEPI_BITS>(cg, BN, tm, g, s);
    if (epi == FEPI_NCHW) return launch_fused_cg<FIN_F32, FEPI_NCHW>(cg, BN, tm, g, s);
    return fail(BNN_E_CONFIG, "fused layer: float input needs a bits or NCHW epilogue");
}

}  // namespace bnnk
