// K3 on the FP4 tensor cores for the standalone operator API: xnor_gemm (kernels.cpp:53-88),
// its float epilogue (to_float + bias_add, kernels.cpp:90-107) and the conv_forward_binary
// scatter (reshape_output, lowering.cpp:87-95), in ONE launch straight from the packed bits
// (xnor4_kernel); for large products (>= 2^32 bit-MACs, M, N >= 512) the operands are expanded
// once into HBM and streamed by TMA into CTA pairs (expand4_kernel + xnor4t_kernel, below).
//
// Both operands are the reference's packed lines (W row-packed [M x ldw], X col-packed
// [N x ldx], bit j of word q = element 32q + j, 1 = +1) expanded in shared memory to e2m1
// {+1.0, -1.0} (codes 0x2 / 0xA) and 0.0 (0x0) for the pad bits past L. The f32 accumulator of
// kind::mxf4 (block scales 2^0) then holds sum_k w_k x_k = L - 2 popc(w ^ x) exactly (|sum| <= L
// < 2^24): the reference's xnor_gemm value, with no correction term. (The previous tensor-core
// path unpacked both operands to int8 in HBM first: two extra launches and 8x the bytes.)
//
// CTA anatomy (448 threads): warp 1 TMEM allocator + MMA issuer (converged warp, elected
// lane), warps 2-5 epilogue (lane = output row m), warps 6-13 producers (thread t expands W line
// t and X line t of the tile for each 256-element K block). One 128 x NB tile per CTA (NB <= 256
// columns chosen so the tiles fill the SMs), persistent over tiles when there are more.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "bnn_common.cuh"
#include "umma.cuh"

#include <cuda.h>

namespace bnnk {

using namespace umma;

int make_tmap_2d_s8(CUtensorMap* map, const void* base, size_t rows, size_t K, size_t ld, uint32_t box_rows);

namespace {

constexpr int kGThreads = 448;
constexpr int kGMaxStages = 8;
constexpr int kGSfCol = 496;
constexpr size_t kGSmemMax = 232448;

struct G4 {
    const uint32_t* w;
    size_t ldw;
    const uint32_t* x;
    size_t ldx;
    int M, N, L, Lw;     // Lw = ceil(L / 32) words per line
    int KB;              // 256-element K blocks
    int NB, m_tiles, n_tiles, nst;
    int32_t* out_s32;    // [M, ldo] (s32 epilogue) or null
    size_t ldo;
    float* out_f32;      // [N / P][M][P] (f32 epilogue: float(acc) + bias[m])
    const float* bias;
    int P;
};

__host__ __device__ constexpr uint32_t idesc_mxf4_m128(int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_mxf4_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t sf,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sf)
        : "memory");
}

// 32 elements (bits b, valid mask m) -> 16 bytes of e2m1 at 16-byte chunk `chunk` of SW128 row r:
// element 8s + n holds element 4n + s of the word (the same permutation for both operands), code
// 0x2 (+1) for a set bit, 0xA (-1) for a clear one, 0x0 past L.
__device__ __forceinline__ void put_pm1(uint32_t tile, int r, int chunk, uint32_t b, uint32_t m) {
    uint32_t o[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const uint32_t xs = (b >> s) & 0x11111111u, ms = (m >> s) & 0x11111111u;
        o[s] = (ms << 1) | ((ms & ~xs) << 3);
    }
    st_shared_v4(tile + uint32_t(r) * 128u + (uint32_t(chunk ^ (r & 7)) << 4), o[0], o[1], o[2], o[3]);
}

// Words [8kb, 8kb + 8) of line `line` (8 words, zero past the line) and their valid-bit masks.
__device__ __forceinline__ void load_block(const uint32_t* base, size_t ld, int line, bool live, int kb, int Lw, int L,
                                           uint32_t (&w)[8], uint32_t (&m)[8]) {
    const uint32_t* src = base + size_t(live ? line : 0) * ld;
    // the block's 8 words are one 32-byte sector: two 16-byte loads when the line is 16-byte
    // aligned (a warp's scalar loads touch 32 lines each: L1 wavefronts bounded the kernel)
    const bool vec = live && ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && 8 * kb + 8 <= Lw;
    if (vec) {
        const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + 8 * kb));
        const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + 8 * kb + 4));
        w[0] = lo.x, w[1] = lo.y, w[2] = lo.z, w[3] = lo.w, w[4] = hi.x, w[5] = hi.y, w[6] = hi.z, w[7] = hi.w;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int q = 8 * kb + k;
        if (!vec) w[k] = (live && q < Lw) ? __ldg(src + q) : 0u;
        const int nv = L - 32 * q;  // valid elements in word q
        m[k] = !live || nv <= 0 ? 0u : nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u);
    }
}

// Epilogue of one 128 x NB tile: lane = output row m, TMEM columns from tb = output columns
// n0 + c. s32 output [M, ldo], or to_float + bias_add scattered to [N / P][M][P].
__device__ __forceinline__ void store_tile(const G4& g, uint32_t tb, int m, int n0) {
    const float bv = (g.out_f32 && g.bias && m < g.M) ? __ldg(g.bias + m) : 0.0f;
    for (int c = 0; c < (g.NB + 31) / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tb + uint32_t(32 * c), v);
        tmem_ld_wait();
        if (m >= g.M) continue;
        const int nb = n0 + 32 * c;
        if (g.out_s32) {
            int32_t* orow = g.out_s32 + size_t(m) * g.ldo + nb;
            const bool vec = nb + 32 <= g.N && 32 * c + 32 <= g.NB && (g.ldo & 3) == 0 &&
                             ((reinterpret_cast<uintptr_t>(g.out_s32) & 15) == 0);
            if (vec) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<int4*>(orow + j) =
                        make_int4(int(__uint_as_float(v[j])), int(__uint_as_float(v[j + 1])),
                                  int(__uint_as_float(v[j + 2])), int(__uint_as_float(v[j + 3])));
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (nb + j < g.N && 32 * c + j < g.NB) orow[j] = int(__uint_as_float(v[j]));
            }
        } else {
            // to_float (exact: |acc| < 2^24) + bias_add, scattered to [img][m][p]
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
                const int n = nb + j;
                if (n >= g.N || 32 * c + j >= g.NB) break;
                const int img = n / g.P, p = n - img * g.P;
                g.out_f32[(size_t(img) * g.M + m) * g.P + p] = __fadd_rn(__uint_as_float(v[j]), bv);
            }
        }
    }
}

__global__ void __launch_bounds__(kGThreads, 1) xnor4_kernel(const __grid_constant__ G4 g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const int nst = g.nst;
    uint8_t* sA = smem_raw + (base - raw);            // [nst][128 x 128 B]
    uint8_t* sB = sA + size_t(nst) * 16384;           // [nst][NB x 128 B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(nst) * g.NB * 128);
    uint64_t* full = bars;
    uint64_t* empty = bars + kGMaxStages;
    uint64_t* tfull = bars + 2 * kGMaxStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int units = g.m_tiles * g.n_tiles;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 8);  // the 8 producer warps
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 4);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    if (warp >= 2 && warp < 6) {  // block scales: every byte of columns [496, 512) = 2^0
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        const uint32_t lb = tmem_base + (uint32_t(32 * (warp & 3)) << 16);
        tmem_st8(lb + kGSfCol, v);
        tmem_st8(lb + kGSfCol + 8, v);
        tmem_st_wait();
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    if (warp == 1) {
        const uint32_t idesc = idesc_mxf4_m128(g.NB);
        int stage = 0, i = 0;
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            mbar_wait(tempty, (i & 1) ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < g.KB; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + size_t(stage) * 16384);
                const uint32_t b0 = smem_u32(sB + size_t(stage) * g.NB * 128);
                const int nk = min(4, (g.L - 256 * kb + 63) / 64);  // 64-element steps with data
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k >= nk) break;
                    mma_mxf4_w(tmem_base, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                               tmem_base + kGSfCol, (kb != 0 || k != 0));
                }
                mma_commit_w(&empty[stage]);
                if (kb == g.KB - 1) mma_commit_w(tfull);
                __syncwarp();
                if (++stage == nst) stage = 0, phase ^= 1;
            }
        }
        mbar_wait(tempty, (i & 1) ^ 1);
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    } else if (warp >= 2 && warp < 6) {
        // epilogue: lane = output row m, TMEM columns = output columns n
        const int q = warp & 3;
        int i = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            const int mt = u % g.m_tiles, nt = u / g.m_tiles;
            const int m = mt * 128 + q * 32 + lane, n0 = nt * g.NB;
            mbar_wait(tfull, i & 1);
            tc_fence_after();
            store_tile(g, tmem_base + (uint32_t(q * 32) << 16), m, n0);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
        }
    } else if (warp >= 6) {
        // producers: thread t expands W line mt*128 + t (t < 128) and X line nt*NB + t (t < NB)
        const int t = int(threadIdx.x) - 6 * 32;
        int stage = 0, pending = -1;  // pending: a filled stage whose fence + release waits for the next
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int mt = u % g.m_tiles, nt = u / g.m_tiles;
            const int am = mt * 128 + t, bn = nt * g.NB + t;
            const bool has_a = t < 128, has_b = t < g.NB;
            uint32_t naw[8], nam[8], nbw[8], nbm[8];  // the next block's words, loaded ahead
            load_block(g.w, g.ldw, am, has_a && am < g.M, 0, g.Lw, g.L, naw, nam);
            load_block(g.x, g.ldx, bn, has_b && bn < g.N, 0, g.Lw, g.L, nbw, nbm);
            for (int kb = 0; kb < g.KB; ++kb) {
                uint32_t aw[8], am8[8], bw[8], bm8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) aw[k] = naw[k], am8[k] = nam[k], bw[k] = nbw[k], bm8[k] = nbm[k];
                if (kb + 1 < g.KB) {
                    load_block(g.w, g.ldw, am, has_a && am < g.M, kb + 1, g.Lw, g.L, naw, nam);
                    load_block(g.x, g.ldx, bn, has_b && bn < g.N, kb + 1, g.Lw, g.L, nbw, nbm);
                }
                mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t ta = smem_u32(sA + size_t(stage) * 16384);
                const uint32_t tbb = smem_u32(sB + size_t(stage) * g.NB * 128);
                if (has_a) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) put_pm1(ta, t, k, aw[k], am8[k]);
                }
                if (has_b) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) put_pm1(tbb, t, k, bw[k], bm8[k]);
                }
                // one proxy fence per two filled stages (released together)
                if (pending >= 0) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(&full[pending]);
                        mbar_arrive(&full[stage]);
                    }
                    pending = -1;
                } else {
                    pending = stage;
                }
                if (++stage == nst) stage = 0, phase ^= 1;
            }
        }
        if (pending >= 0) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[pending]);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
}

// ---------------------------------------------------------------- large GEMMs: TMA-fed operands
//
// Above ~2^32 bit-MACs the in-CTA expansion above is the bound: every CTA re-expands its A and B
// lines for every tile, and the producers' shared-memory stores compete with the MMA's operand
// reads. For those products both operands are expanded ONCE into HBM scratch (expand4_kernel:
// 4 B of packed bits -> 16 B of e2m1, the same element order and codes as put_pm1, 0x0 past L),
// and xnor4t_kernel streams them with TMA (SWIZZLE_128B, the layout put_pm1 writes by hand; rows
// past M / N and bytes past the line are zero-filled by TMA, i.e. e2m1 0.0, the pad value).
//
// CTA anatomy (192 threads): warp 0 TMA producer (one lane), warp 1 TMEM allocator + MMA issuer,
// warps 2-5 epilogue. Two accumulators in TMEM (columns 0 and 256, NB <= 240; the block scales
// at 496) so the epilogue of tile i overlaps the MMAs of tile i + 1.

constexpr int kTThreads = 192;

// Packed lines [rows, ld words] (L valid bits each) -> e2m1 lines [rows, Lw * 16 bytes], both
// operands in one launch (blockIdx.y). Dense lines with no partial last word (ld = Lw, L = 32 Lw,
// the usual large-GEMM case) stream 4 words per thread (16-byte load, 4 x 16-byte stores).
struct Expand4Op {
    const uint32_t* src;
    size_t ld, rows;
    uint4* dst;
};

__device__ __forceinline__ uint4 pm1_word(uint32_t b, uint32_t m) {
    uint32_t o[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const uint32_t xs = (b >> s) & 0x11111111u, ms = (m >> s) & 0x11111111u;
        o[s] = (ms << 1) | ((ms & ~xs) << 3);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

__global__ void __launch_bounds__(256) expand4_kernel(const Expand4Op a, const Expand4Op b, int Lw, int L) {
    const Expand4Op& op = blockIdx.y ? b : a;
    const size_t total = op.rows * size_t(Lw);
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    const size_t t0 = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (op.ld == size_t(Lw) && L == 32 * Lw && (total & 3) == 0 && (reinterpret_cast<uintptr_t>(op.src) & 15) == 0) {
        const uint4* src4 = reinterpret_cast<const uint4*>(op.src);
        for (size_t i = t0; i < total / 4; i += stride) {
            const uint4 w = __ldg(src4 + i);
            op.dst[4 * i + 0] = pm1_word(w.x, 0xffffffffu);
            op.dst[4 * i + 1] = pm1_word(w.y, 0xffffffffu);
            op.dst[4 * i + 2] = pm1_word(w.z, 0xffffffffu);
            op.dst[4 * i + 3] = pm1_word(w.w, 0xffffffffu);
        }
        return;
    }
    for (size_t i = t0; i < total; i += stride) {
        const size_t r = i / size_t(Lw);
        const int q = int(i - r * size_t(Lw));
        const int nv = L - 32 * q;
        op.dst[i] = pm1_word(__ldg(op.src + r * op.ld + q), nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u));
    }
}

// CL = 2: a CTA pair (cluster of two) computes a 256-row x NB tile with cta_group::2 M = 256
// instructions issued by the even CTA: each CTA TMA-loads its own 128 A rows and half of the
// B tile (NB / 2 rows), completing bytes on the leader's full barrier; D rows 0-127 land in the
// leader's TMEM, 128-255 in the peer's; each CTA's epilogue reads its own TMEM and releases the
// accumulator on the leader's barrier. Per CTA and K block the shared memory then takes 16 KB +
// NB x 64 B of TMA writes and the same again of MMA reads: the single-CTA kernel moved 16 KB +
// NB x 128 B each way per 4 MMAs, more than the ~128 B/cycle an SM's shared memory sustains at
// the FP4 MMA rate (measured: 0.61 of the FP4 peak single-CTA).
__device__ __forceinline__ void mma_mxf4_cg2_w(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t sf, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sf)
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_mxf4_mn(int M, int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);
}

template <int CL>
__global__ void __launch_bounds__(kTThreads, 1)
    xnor4t_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                  const __grid_constant__ G4 g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const int nst = g.nst;
    const int BH = g.NB / CL;                // B rows per CTA
    uint8_t* sA = smem_raw + (base - raw);   // [nst][128 x 128 B]
    uint8_t* sB = sA + size_t(nst) * 16384;  // [nst][BH x 128 B]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(nst) * BH * 128);
    uint64_t* full = bars;
    uint64_t* empty = bars + kGMaxStages;
    uint64_t* tfull = bars + 2 * kGMaxStages;  // [2]
    uint64_t* tempty = tfull + 2;              // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    const int rank = CL == 2 ? int(cluster_ctarank()) : 0;
    const int mp_tiles = (g.m_tiles + CL - 1) / CL;  // row-tile groups (one per cluster)
    const int units = mp_tiles * g.n_tiles;
    const int u0 = int(blockIdx.x) / CL, ustep = int(gridDim.x) / CL;
    const uint32_t stage_tx = 16384u + uint32_t(BH) * 128u;  // this CTA's bytes per stage
    auto leader = [&](uint64_t* bar) { return CL == 2 ? mapa(smem_u32(bar), 0) : smem_u32(bar); };
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], CL);  // (the leader's) one expect_tx arrive per CTA
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * CL);  // (the leader's) four epilogue warps per CTA
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tA);
        tma_prefetch(&tB);
    }
    if (warp == 1) {
        if (CL == 2)
            tmem_alloc_cg2<512>(tmem_slot);
        else
            tmem_alloc<512>(tmem_slot);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    if (warp >= 2) {  // block scales: every byte of columns [496, 512) = 2^0
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        const uint32_t lb = tmem_base + (uint32_t(32 * (warp & 3)) << 16);
        tmem_st8(lb + kGSfCol, v);
        tmem_st8(lb + kGSfCol + 8, v);
        tmem_st_wait();
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (CL == 2) cluster_sync();  // the peer's barriers and scale factors are ready
    tc_fence_after();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = u0; u < units; u += ustep) {
                const int mt = (u % mp_tiles) * CL + rank, nt = u / mp_tiles;
                for (int kb = 0; kb < g.KB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* da = sA + size_t(stage) * 16384;
                    uint8_t* db = sB + size_t(stage) * BH * 128;
                    if (CL == 2) {
                        const uint32_t fb = leader(&full[stage]);
                        mbar_arrive_expect_tx_cluster(fb, stage_tx);
                        tma_load_2d_cg2(&tA, fb, da, kb * 128, mt * 128);
                        tma_load_2d_cg2(&tB, fb, db, kb * 128, nt * g.NB + rank * BH);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], stage_tx);
                        tma_load_2d(&tA, &full[stage], da, kb * 128, mt * 128);
                        tma_load_2d(&tB, &full[stage], db, kb * 128, nt * g.NB);
                    }
                    if (++stage == nst) stage = 0, phase ^= 1;
                }
            }
            if (CL == 2) {  // every stage's last release (the pair MMA's multicast commit) has landed
                for (int k = 0; k < nst; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (++stage == nst) stage = 0, phase ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (CL == 1 || rank == 0) {
            const uint32_t idesc = idesc_mxf4_mn(128 * CL, g.NB);
            int stage = 0, i = 0;
            uint32_t phase = 0;
            for (int u = u0; u < units; u += ustep, ++i) {
                const int acc = i & 1, use = i >> 1;
                const uint32_t d = tmem_base + uint32_t(acc * 256);
                mbar_wait(&tempty[acc], (use & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < g.KB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + size_t(stage) * 16384);
                    const uint32_t b0 = smem_u32(sB + size_t(stage) * BH * 128);
                    const int nk = min(4, (g.L - 256 * kb + 63) / 64);  // 64-element steps with data
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (k >= nk) break;
                        if (CL == 2)
                            mma_mxf4_cg2_w(d, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                           tmem_base + kGSfCol, (kb != 0 || k != 0));
                        else
                            mma_mxf4_w(d, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                                       tmem_base + kGSfCol, (kb != 0 || k != 0));
                    }
                    if (CL == 2) {
                        mma_commit_cg2_mc_w(&empty[stage], uint16_t(3));  // both CTAs' slots free
                        if (kb == g.KB - 1) mma_commit_cg2_mc_w(&tfull[acc], uint16_t(3));
                    } else {
                        mma_commit_w(&empty[stage]);
                        if (kb == g.KB - 1) mma_commit_w(&tfull[acc]);
                    }
                    __syncwarp();
                    if (++stage == nst) stage = 0, phase ^= 1;
                }
            }
            // the epilogues have released the last accumulators (CL = 2: the peer's remote
            // arrives have then all landed here)
            for (int k = 0; k < 2; ++k, ++i) mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);
        }
    } else {
        const int q = warp & 3;
        int i = 0;
        for (int u = u0; u < units; u += ustep, ++i) {
            const int acc = i & 1, use = i >> 1;
            const int mt = (u % mp_tiles) * CL + rank, nt = u / mp_tiles;
            mbar_wait(&tfull[acc], use & 1);
            tc_fence_after();
            store_tile(g, tmem_base + uint32_t(acc * 256) + (uint32_t(q * 32) << 16), mt * 128 + q * 32 + lane,
                       nt * g.NB);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (CL == 2)
                    mbar_arrive_cluster(leader(&tempty[acc]));
                else
                    mbar_arrive(&tempty[acc]);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (CL == 2) cluster_sync_relaxed();  // every cross-CTA operation has landed (drains above)
    if (warp == 1) {
        tc_fence_after();
        if (CL == 2)
            tmem_dealloc_cg2<512>(tmem_base);
        else
            tmem_dealloc<512>(tmem_base);
    }
}

// Tile width for the TMA kernel: NB in [16, 240] (multiple of 16, two accumulators) minimising
// waves x (NB + per-tile overhead) over the SMs; never wider than N needs.
int pick_nb_t(int m_tiles, int N, int sms) {
    const int n16 = (N + 15) / 16 * 16;
    int best = std::min(240, n16);
    double best_cost = 1e300;
    for (int nb = std::min(240, n16); nb >= 16; nb -= 16) {
        const long units = long(m_tiles) * ((N + nb - 1) / nb);
        const long waves = (units + sms - 1) / sms;
        const double cost = double(waves) * (nb + 40);
        if (cost < best_cost * 0.999) best_cost = cost, best = nb;
    }
    return best;
}

int launch_xnor4t(G4 g, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(xnor4t_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGSmemMax)));
        BNN_CUDA(cudaFuncSetAttribute(xnor4t_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGSmemMax)));
        attr_set = true;
    }
    g.Lw = (g.L + 31) / 32;
    g.KB = (g.L + 255) / 256;
    g.m_tiles = (g.M + 127) / 128;
    const int sms = num_sms();
    g.NB = pick_nb_t(g.m_tiles, g.N, sms);
    g.n_tiles = (g.N + g.NB - 1) / g.NB;
    // operands expanded once to e2m1 in stream-ordered scratch, 16 B per packed word
    const size_t lb = size_t(g.Lw) * 16;
    Scratch ea, eb;
    BNN_TRY(ea.alloc(size_t(g.M) * lb, s));
    BNN_TRY(eb.alloc(size_t(g.N) * lb, s));
    expand4_kernel<<<dim3(unsigned(sms * 4), 2), 256, 0, s>>>(Expand4Op{g.w, g.ldw, size_t(g.M), ea.as<uint4>()},
                                                              Expand4Op{g.x, g.ldx, size_t(g.N), eb.as<uint4>()}, g.Lw, g.L);
    BNN_TRY(launch_check("expand4_kernel"));
    CUtensorMap ta, tb;
    BNN_TRY(make_tmap_2d_s8(&ta, ea.p, size_t(g.M), lb, lb, 128));
    // CTA pairs (cta_group::2, 256 rows per pair) when there are at least two row tiles
    static const int cl_env = getenv("BNN_XNOR4T_CLUSTER") ? atoi(getenv("BNN_XNOR4T_CLUSTER")) : 2;
    const int CL = (cl_env == 2 && g.m_tiles >= 2) ? 2 : 1;
    const size_t stage_bytes = 16384 + size_t(g.NB / CL) * 128;
    g.nst = int(std::min<size_t>(kGMaxStages, (kGSmemMax - 1024 - 256) / stage_bytes));
    BNN_TRY(make_tmap_2d_s8(&tb, eb.p, size_t(g.N), lb, lb, uint32_t(g.NB / CL)));
    const int units = (g.m_tiles + CL - 1) / CL * g.n_tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(CL * std::min(units, sms / CL)));
    cfg.blockDim = dim3(unsigned(kTThreads));
    cfg.dynamicSmemBytes = 1024 + size_t(g.nst) * stage_bytes + 256;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(CL);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (CL == 2) {  // persistent: no more clusters than can be co-resident
        static int max_clusters = -1;
        if (max_clusters < 0) {
            int n = 0;
            max_clusters = cudaOccupancyMaxActiveClusters(&n, xnor4t_kernel<2>, &cfg) == cudaSuccess && n > 0 ? n : sms / 2;
        }
        cfg.gridDim = dim3(unsigned(2 * std::min(units, max_clusters)));
    }
    if (CL == 2)
        BNN_CUDA(cudaLaunchKernelEx(&cfg, xnor4t_kernel<2>, ta, tb, g));
    else
        BNN_CUDA(cudaLaunchKernelEx(&cfg, xnor4t_kernel<1>, ta, tb, g));
    set_last_gemm("xnor4t_kernel");
    return launch_check("xnor4t_kernel");
}

int launch_xnor4(G4 g, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(xnor4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGSmemMax)));
        attr_set = true;
    }
    g.Lw = (g.L + 31) / 32;
    g.KB = (g.L + 255) / 256;
    g.m_tiles = (g.M + 127) / 128;
    // image columns per tile: the widest NB (<= 256, multiple of 16) that still gives every SM a
    // tile, and never wider than N needs
    const int sms = num_sms();
    // the widest NB whose tiles still fit one wave, unless even NB = 16 needs more (then the
    // widest NB: fewest rounds)
    const int n16 = (g.N + 15) / 16 * 16;
    int nb = 256;
    while (nb > 16 && nb / 2 >= n16) nb /= 2;  // never wider than the batch needs
    auto tiles_of = [&](int b) { return long(g.m_tiles) * ((g.N + b - 1) / b); };
    while (nb > 16 && tiles_of(nb) * 2 <= sms) nb /= 2;  // narrower while it still fits one wave
    g.NB = std::min(nb, n16);
    g.n_tiles = (g.N + g.NB - 1) / g.NB;
    g.nst = int(std::min<size_t>(kGMaxStages, (kGSmemMax - 1024 - 256) / (16384 + size_t(g.NB) * 128)));
    const int units = g.m_tiles * g.n_tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(std::min(units, sms)));
    cfg.blockDim = dim3(unsigned(kGThreads));
    cfg.dynamicSmemBytes = 1024 + size_t(g.nst) * (16384 + size_t(g.NB) * 128) + 256;
    cfg.stream = s;
    BNN_CUDA(cudaLaunchKernelEx(&cfg, xnor4_kernel, g));
    set_last_gemm("xnor4_kernel");
    return launch_check("xnor4_kernel");
}

}  // namespace

// xnor_gemm on the FP4 tensor cores, s32 output [M, ldo] (kernels.cpp:53-88).
int xnor4_gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N, size_t L,
                   int32_t* out, size_t ldo, cudaStream_t s) {
    if (M == 0 || N == 0) return BNN_OK;
    G4 g{};
    g.w = w, g.ldw = ldw, g.x = x, g.ldx = ldx, g.M = int(M), g.N = int(N), g.L = int(L);
    g.out_s32 = out, g.ldo = ldo, g.P = 1;
    return launch_xnor4(g, s);
}

// xnor_gemm -> to_float -> bias_add, written as [N / P][M][P] (P = N for a linear layer,
// oh*ow for a conv: reshape_output, lowering.cpp:87-95).
int xnor4_gemm_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N, size_t L,
                   const float* bias, size_t P, float* out, cudaStream_t s) {
    if (M == 0 || N == 0) return BNN_OK;
    G4 g{};
    g.w = w, g.ldw = ldw, g.x = x, g.ldx = ldx, g.M = int(M), g.N = int(N), g.L = int(L);
    g.out_f32 = out, g.bias = bias, g.P = int(P ? P : N);
    return launch_xnor4(g, s);
}

// The same two products on the TMA-fed kernel (operands expanded once to e2m1 in HBM scratch).
int xnor4t_gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N, size_t L,
                    int32_t* out, size_t ldo, cudaStream_t s) {
    if (M == 0 || N == 0) return BNN_OK;
    G4 g{};
    g.w = w, g.ldw = ldw, g.x = x, g.ldx = ldx, g.M = int(M), g.N = int(N), g.L = int(L);
    g.out_s32 = out, g.ldo = ldo, g.P = 1;
    return launch_xnor4t(g, s);
}

int xnor4t_gemm_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N, size_t L,
                    const float* bias, size_t P, float* out, cudaStream_t s) {
    if (M == 0 || N == 0) return BNN_OK;
    G4 g{};
    g.w = w, g.ldw = ldw, g.x = x, g.ldx = ldx, g.M = int(M), g.N = int(N), g.L = int(L);
    g.out_f32 = out, g.bias = bias, g.P = int(P ? P : N);
    return launch_xnor4t(g, s);
}

}  // namespace bnnk
