// Halo-tile FP4 conv (kind::mxf4): the "same" binary convolutions with a packed-bit input
// (3x3 / pad 1, and 1x1, 1x3, 3x1), i.e. every VGG-small conv after the first, as
//
//   conv_forward_binary -> bias -> [maxpool2] -> affine_norm -> htanh -> sign
//   (network.cpp:65-79, 133-175; binarize.cpp:24-37)
//
// fused into one persistent launch that writes the next layer's packed NHWC bits (the same
// contract and the same exactness argument as fused_swap4_kernel in fused.cu).
//
// What is different: the activations are expanded to e2m1 once per input pixel, not once per
// (pixel, tap). The output positions live on a padded "canvas": G images side by side and the
// batch stacked vertically, each image with a 1-pixel frame of padding (sign(0.0) = +1, an
// all-ones word), pitch P pixels per canvas row. On the canvas, output position q reads input
// pixel q + (ky*P + kx) for tap (ky, kx): every tap is the SAME pixel sequence shifted by a
// constant. A tile is TR whole canvas rows (N = TR*P output columns, a few of them frame
// columns whose results are discarded); its halo (N + 2P + 2 pixels) is expanded once into
// shared memory in the no-swizzle K-major layout [channel chunk][pixel][16 B] (8-row core
// matrices 128 B apart, K chunks NH*16 B apart), and the UMMA B descriptor of tap t simply
// starts (ky*P + kx) rows further in. tools/halo_probe.cu checks this layout (any start row)
// and measures N/2 cycles per M128 x N x K64 instruction for N = 128..256, with or without
// concurrent shared-memory stores.
//
// Weights: the whole [128 channels x K] e2m1 slice of the CTA's channel tile stays resident in
// shared memory (TMA once per CTA, SW128, before the grid-dependency wait), so nothing but the
// 1-bit activations streams per tile. Layers whose slice does not fit fall back to
// fused_swap4_kernel.
//
// Pooled layers give each image its own 2-row / 2-column frame (S = H + 2 rows per image, even),
// so a tile of an even number of canvas rows never splits a 2x2 window; unpooled layers share
// the frame rows and columns between neighbours (S = H + 1, Q = W + 1).
//
// CTA anatomy (512 threads, one CTA per SM): warp 0 weight TMA, warp 1 TMEM allocator + MMA
// issuer (the converged warp, one elected lane issues), warps 4-11 epilogue (lane = channel, 2
// warps per TMEM lane quarter), warps 2, 3, 12, 14, 15 halo producers (none on sub-partition 1,
// the MMA warp's: its issue slots decide the MMA rate). Accumulators: 2 x N <= 2 x 240 TMEM
// columns, block scales (all 2^0) in columns [496, 512).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "bnn_common.cuh"
#include "fused.cuh"
#include "umma.cuh"

namespace bnnk {

using namespace umma;

namespace {

constexpr int kHThreads = 512;
constexpr int kHEpiWarps = 8;
constexpr int kHProdWarps = 6;
constexpr int kHProdThreads = kHProdWarps * 32;
constexpr int kHSfCol = 496;
constexpr int kHMaxN = 240;
constexpr int kHMaxStages = 4;
constexpr int kHMaxWst = 8;  // streamed-weight ring slots
constexpr size_t kHSmemMax = 232448;  // 227 KB opt-in per CTA
constexpr size_t kHBarBytes = 256;     // mbarriers + the TMEM slot
constexpr int kHTabs = kHMaxStages + 2;  // column-table ring: producers run <= nst + 2 tiles ahead of the epilogue
constexpr size_t kHTail = kHBarBytes + size_t(kHTabs) * kHMaxN * 4;  // + the epilogue's column tables

// K-major, no swizzle: core matrix = 8 rows x 16 bytes, 8-row groups 128 B apart (SBO), the two
// K core matrices of one K=64 e2m1 step LBO apart.
__device__ __forceinline__ uint64_t sdesc_k_none(uint32_t addr, uint32_t lbo) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t(128 >> 4) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

// kind::mxf4 block-scaled instruction descriptor: E2M1 A and B, K-major, UE8M0 scales, M = 128.
__host__ __device__ constexpr uint32_t idesc_mxf4_m128(int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
}

// Issued by the whole (converged) MMA warp with warp-uniform operands, so the descriptors stay in
// uniform registers; one elected lane issues. (Issuing from inside `if (lane == 0)` made every
// instruction go through R2UR and an ELECT loop: ~150-200 cycles per MMA, slower than the tensor
// core.) Each descriptor is passed as (lo, hi) halves: the per-step offsets only touch the low
// word (start address), so a step costs two 32-bit uniform adds.
__device__ __forceinline__ void mma_mxf4_lohi(uint32_t d_tmem, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                              uint32_t idesc, uint32_t sf, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 ad, bd;\n\t"
        "mov.b64 ad, {%1, %2};\n\t"
        "mov.b64 bd, {%3, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], ad, bd, %5, [%7], [%7], p;\n\t}" ::"r"(d_tmem),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(accumulate), "r"(sf)
        : "memory");
}

// One tile: taps x CPT K64 steps, fully unrolled (the per-tap loop overhead made the issue the
// bound at CPT = 2). Step s reads weight bytes [(s / 4) * 16 KB + (s % 4) * 32) of the resident
// SW128 blocks and halo rows from toff[t] (+ 2 K chunks per step).
template <int CPT>
__device__ __forceinline__ void issue_tile(uint32_t d, uint32_t alo0, uint32_t ahi, uint32_t blo0, uint32_t bhi,
                                           uint32_t idesc, uint32_t sf, const uint32_t (&toff)[9], int taps,
                                           uint32_t step16) {
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        if (t >= taps) break;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int s = t * CPT + c;
            mma_mxf4_lohi(d, alo0 + uint32_t((s >> 2) * 1024 + (s & 3) * 2), ahi, blo0 + toff[t] + uint32_t(c) * step16,
                          bhi, idesc, sf, s != 0);
        }
    }
}

// Streamed weights: the same steps, each block of 4 steps from ring slot ws (waited on wfull,
// released by a commit to wempty).
template <int CPT>
__device__ __forceinline__ void issue_tile_stream(uint32_t d, uint32_t alo0, uint32_t ahi, uint32_t blo0, uint32_t bhi,
                                                  uint32_t idesc, uint32_t sf, const uint32_t (&toff)[9], int taps,
                                                  uint32_t step16, uint64_t* wfull, uint64_t* wempty, int wst, int& ws,
                                                  uint32_t& wph) {
    const int steps = taps * CPT;
#pragma unroll
    for (int t = 0; t < 9; ++t) {
        if (t >= taps) break;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int st = t * CPT + c;
            if ((st & 3) == 0) {
                mbar_wait(&wfull[ws], wph);
                tc_fence_after();
            }
            mma_mxf4_lohi(d, alo0 + uint32_t(ws) * 1024u + uint32_t(st & 3) * 2u, ahi,
                          blo0 + toff[t] + uint32_t(c) * step16, bhi, idesc, sf, st != 0);
            if ((st & 3) == 3 || st == steps - 1) {
                mma_commit_w(&wempty[ws]);
                if (++ws == wst) ws = 0, wph ^= 1;
            }
        }
    }
}

__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// 32 activation bits -> 16 bytes of e2m1 nibbles (1.0 = 0x2, 0.0 = 0x0): element 8s + n holds
// bit 4n + s (the order of put_word4 in fused.cu; the FP4 weights from prep_weights4 match).
__device__ __forceinline__ void st_expand4(uint32_t addr, uint32_t w) {
    st_shared_v4(addr, (w << 1) & 0x22222222u, w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
}

__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x4(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x2(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(v[0]), "=r"(v[1]) : "r"(taddr));
}

// WN (2..32, a power of two) consecutive accumulator columns of this warp's 32 lanes (no wait).
template <int WN>
__device__ __forceinline__ void load_cols(uint32_t taddr, uint32_t (&v)[32]) {
    if constexpr (WN == 32) {
        tmem_ld32(taddr, v);
    } else if constexpr (WN == 16) {
        uint32_t t[16];
        tmem_ld16(taddr, t);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = t[j];
    } else if constexpr (WN == 8) {
        tmem_ld_x8(taddr, v);
    } else if constexpr (WN == 4) {
        tmem_ld_x4(taddr, v);
    } else {
        static_assert(WN == 2, "column count");
        tmem_ld_x2(taddr, v);
    }
}

// Pooled epilogue unit: WN columns of a canvas row pair (rows P columns apart in TMEM) ->
// WN / 2 pooled positions. The OR of the four (u >= T) ^ flip of a 2x2 window is
// (max u >= T) without flip and (min u < T) with it: 3 min/max, one compare, one ballot.
template <int WN>
__device__ __forceinline__ void pool_unit(uint32_t taddr, uint32_t pitch, float Tf, bool flip, int lane,
                                          uint32_t* dst, size_t dst_stride, bool wvalid) {
    uint32_t v0[32], v1[32];
    load_cols<WN>(taddr, v0);
    load_cols<WN>(taddr + pitch, v1);
    tmem_ld_wait();
    uint32_t mine = 0;
#pragma unroll
    for (int k = 0; k < WN / 2; ++k) {
        const float a = __uint_as_float(v0[2 * k]), b = __uint_as_float(v0[2 * k + 1]);
        const float c = __uint_as_float(v1[2 * k]), d = __uint_as_float(v1[2 * k + 1]);
        const float m = flip ? fminf(fminf(a, b), fminf(c, d)) : fmaxf(fmaxf(a, b), fmaxf(c, d));
        const uint32_t w = __ballot_sync(0xffffffffu, (m >= Tf) != flip);
        if (lane == k) mine = w;
    }
    if (wvalid && lane < WN / 2) dst[size_t(lane) * dst_stride] = mine;
}

// Canvas pixel idx -> NHWC pixel index of its source, or -1 for the frame / images past the batch.
__device__ __forceinline__ long long halo_src(const HaloGeom& g, int idx) {
    const int r = g.dP.div(idx), x = idx - r * g.P;
    const int grp = g.dS.div(r), rr = r - grp * g.S;
    const int slot = g.dQ.div(x), xx = x - slot * g.Q;
    const int b = grp * g.G + slot;
    if (rr == 0 || rr > g.H || xx == 0 || xx > g.W || slot >= g.G || b >= g.B) return -1;
    return (long long)(b * g.H + (rr - 1)) * g.W + (xx - 1);
}

// Halo rows j0 and j0 + kHProdThreads of a tile: every vector load of both rows is issued before
// the first store (one L2 round trip per pair of rows). V words per load (Cw <= 16).
// Halo row j is the input pixel of tap (1, 1) of tile column j - (P + 1), whose output pixel (a
// "same" conv on the same canvas) it therefore also is: unpooled layers record it in the tile's
// column table for the epilogue (tab, else null).
__device__ __forceinline__ void put_col(const HaloGeom& g, int* tab, int j, long long pix) {
    const int c = j - g.P - 1;  // columns past the tile's TR canvas rows (N is a multiple of 16): -1
    if (tab && c >= 0 && c < g.N) tab[c] = c < g.TR * g.P ? int(pix) : -1;
}

template <int V>
__device__ __forceinline__ void fill_rows(const HaloGeom& g, uint32_t hb, uint32_t lbo, int q0, int j0, int nh, int* tab) {
    using Vec = typename std::conditional<V == 4, uint4, uint2>::type;
    constexpr int kMaxV = 16 / V;
    const int nv = g.Cw / V;
    Vec a[2][kMaxV];
    bool has[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int j = j0 + h * kHProdThreads;
        has[h] = j < nh;
        const long long pix = has[h] ? halo_src(g, q0 + j) : -1;
        if (has[h]) put_col(g, tab, j, pix);
        const Vec* src = reinterpret_cast<const Vec*>(g.in + (pix < 0 ? 0 : pix) * g.Cw);
#pragma unroll
        for (int v = 0; v < kMaxV; ++v) {
            if (v >= nv) break;
            if constexpr (V == 4)
                a[h][v] = pix < 0 ? make_uint4(~0u, ~0u, ~0u, ~0u) : __ldg(src + v);
            else
                a[h][v] = pix < 0 ? make_uint2(~0u, ~0u) : __ldg(src + v);
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (!has[h]) break;
        const uint32_t dst = hb + uint32_t(j0 + h * kHProdThreads) * 16u;
#pragma unroll
        for (int v = 0; v < kMaxV; ++v) {
            if (v >= nv) break;
            const uint32_t d0 = dst + uint32_t(V * v) * lbo;
            st_expand4(d0, a[h][v].x);
            st_expand4(d0 + lbo, a[h][v].y);
            if constexpr (V == 4) {
                st_expand4(d0 + 2 * lbo, a[h][v].z);
                st_expand4(d0 + 3 * lbo, a[h][v].w);
            }
        }
    }
}

__device__ __forceinline__ long long hclock() { return clock64(); }
__device__ __forceinline__ unsigned long long hgtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// BNN_HALO_PROFILE: per-role cycle counters (g.dbg, summed over CTAs): mbarrier waits and role
// totals, plus the launch span in globaltimer ns.
struct HClock {
    long long t0 = 0, acc = 0;
    __device__ __forceinline__ void wait(bool on, uint64_t* bar, uint32_t parity) {
        if (!on) return mbar_wait(bar, parity);
        const long long a = hclock();
        mbar_wait(bar, parity);
        acc += hclock() - a;
    }
};

}  // namespace

template <bool STREAM>
__global__ void __launch_bounds__(kHThreads, 1)
    halo4_kernel(const __grid_constant__ CUtensorMap tmW4, const __grid_constant__ HaloGeom g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    // weights: KB4 resident blocks of 128 rows x 128 B (SW128), or a ring of wst blocks (streamed)
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* sW = smem_raw + (base - raw);
    const uint32_t wbytes = uint32_t(STREAM ? g.wst : g.KB4) * 16384u;
    const uint32_t lbo = uint32_t(g.NH) * 16u;         // K-chunk stride of a halo stage
    const uint32_t hbytes = uint32_t(g.Cw) * lbo;      // one halo stage
    const uint32_t sH = base + wbytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sW + wbytes + size_t(g.nst) * hbytes);
    uint64_t* full = bars;                  // [kHMaxStages] halo stage written (producer warps)
    uint64_t* empty = bars + kHMaxStages;   // [kHMaxStages] halo stage consumed (MMA commit)
    uint64_t* tfull = bars + 2 * kHMaxStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* wbar = tempty + 2;
    uint64_t* wfull = wbar + 1;                 // streamed weights: [kHMaxWst] ring slots
    uint64_t* wempty = wfull + kHMaxWst;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wempty + kHMaxWst);
    int* coltab = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(bars) + kHBarBytes);  // [nst + 2][kHMaxN]

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.launch_dependents;");
    const bool prof = g.dbg != nullptr;
    const long long k_start = prof ? hclock() : 0;
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 0] = hgtimer();
    if (prof && threadIdx.x == 0) atomicMin(g.dbg + 14, hgtimer());
    const int mt = int(blockIdx.x) % g.m_tiles;
    const int nstride = int(gridDim.x) / g.m_tiles;
    const int n0 = int(blockIdx.x) / g.m_tiles;

    if (threadIdx.x == 0) {
        tma_prefetch(&tmW4);
        for (int s = 0; s < g.nst; ++s) {
            mbar_init(&full[s], kHProdWarps);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kHEpiWarps);
        }
        mbar_init(wbar, 1);
        for (int w = 0; w < (STREAM ? g.wst : 0); ++w) {
            mbar_init(&wfull[w], 1);
            mbar_init(&wempty[w], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = warp_uniform(*tmem_slot);
    if (warp == 0 && lane == 0 && !STREAM) {
        // the resident weights are build-time constants: load them before the grid dependency
        mbar_arrive_expect_tx(wbar, wbytes);
        for (int kb = 0; kb < g.KB4; ++kb) tma_load_2d(&tmW4, wbar, sW + size_t(kb) * 16384, kb * 128, mt * 128);
    }
    if (warp >= 4 && warp < 8) {  // block scales: every byte of columns [496, 512) = 2^0
        uint32_t v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        const uint32_t lane_base = tmem_base + (uint32_t(32 * (warp & 3)) << 16);
        tmem_st8(lane_base + kHSfCol, v);
        tmem_st8(lane_base + kHSfCol + 8, v);
        tmem_st_wait();
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 2] = hgtimer();
    const long long k_main = prof ? hclock() : 0;
    if (prof && threadIdx.x == 0) atomicAdd(g.dbg + 12, (unsigned long long)(k_main - k_start));

    if (warp == 0 && STREAM) {
        // streamed weights: every tile walks the layer's KB4 blocks through the ring
        if (lane == 0) {
            int ws = 0;
            uint32_t wph = 0;
            for (int nt = n0; nt < g.n_tiles; nt += nstride)
                for (int kb = 0; kb < g.KB4; ++kb) {
                    mbar_wait(&wempty[ws], wph ^ 1);
                    mbar_arrive_expect_tx(&wfull[ws], 16384);
                    tma_load_2d(&tmW4, &wfull[ws], sW + size_t(ws) * 16384, kb * 128, mt * 128);
                    if (++ws == g.wst) ws = 0, wph ^= 1;
                }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_mxf4_m128(g.N);
        const uint32_t lbo16 = lbo >> 4;
        uint32_t toff[9];  // tap shifts on the canvas, in 16-byte units
#pragma unroll
        for (int t = 0; t < 9; ++t) toff[t] = uint32_t(g.toff[t]);
        HClock cw, ct, cf;
        if (!STREAM) cw.wait(prof, wbar, 0);
        tc_fence_after();
        long long t_first = 0;
        int hs = 0, i = 0, ws = 0;
        uint32_t hph = 0, wph = 0;
        for (int nt = n0; nt < g.n_tiles; nt += nstride, ++i) {
            const int acc = i & 1;
            ct.wait(prof, &tempty[acc], ((i >> 1) & 1) ^ 1);
            cf.wait(prof, &full[hs], hph);
            tc_fence_after();
            if (prof && i == 0) t_first = hclock() - k_main;
            {
                const uint32_t d = tmem_base + uint32_t(acc * g.N);
                // descriptors by 32-bit adds on the start-address field (every address < 256 KB)
                const uint64_t ad0 = sdesc_k_sw128(base);
                const uint64_t bd0 = sdesc_k_none(sH + uint32_t(hs) * hbytes, lbo);
                const uint32_t alo = uint32_t(ad0), ahi = uint32_t(ad0 >> 32);
                const uint32_t blo = uint32_t(bd0), bhi = uint32_t(bd0 >> 32);
                const int taps = (g.dbg_mode & 4) ? 0 : g.taps;
                const uint32_t sf = tmem_base + kHSfCol, step16 = 2u * lbo16;
                if constexpr (STREAM) {
                    switch (g.cpt) {
                        case 1: issue_tile_stream<1>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16, wfull, wempty, g.wst, ws, wph); break;
                        case 2: issue_tile_stream<2>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16, wfull, wempty, g.wst, ws, wph); break;
                        case 4: issue_tile_stream<4>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16, wfull, wempty, g.wst, ws, wph); break;
                        default: issue_tile_stream<8>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16, wfull, wempty, g.wst, ws, wph); break;
                    }
                } else {
                    switch (g.cpt) {
                    case 1: issue_tile<1>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16); break;
                    case 2: issue_tile<2>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16); break;
                    case 4: issue_tile<4>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16); break;
                    default: issue_tile<8>(d, alo, ahi, blo, bhi, idesc, sf, toff, taps, step16); break;
                    }
                }
                mma_commit_warp(&empty[hs]);
                mma_commit_warp(&tfull[acc]);
            }
            __syncwarp();
            if (++hs == g.nst) hs = 0, hph ^= 1;
        }
        if (prof && lane == 0) {
            atomicAdd(g.dbg + 0, (unsigned long long)cw.acc);
            atomicAdd(g.dbg + 1, (unsigned long long)ct.acc);
            atomicAdd(g.dbg + 2, (unsigned long long)cf.acc);
            atomicAdd(g.dbg + 3, (unsigned long long)(hclock() - k_main));
            atomicAdd(g.dbg + 8, (unsigned long long)t_first);
        }
        // the epilogue has read the last accumulators
        for (int k = 0; k < 2; ++k, ++i) mbar_wait(&tempty[i & 1], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
        if (g.tl && lane == 0) g.tl[blockIdx.x * 4 + 1] = hgtimer();
    } else if (warp >= 4 && warp < 4 + kHEpiWarps) {
        // epilogue: lane = output channel. Pass 1: aligned 32-column chunks of the accumulator
        // (the two warps of a lane quarter alternate chunks) -> per column, the 32-channel word of
        // decisions (u >= T) ^ flip. Unpooled: each lane stores the word of its column if that
        // column is a real output position. Pooled: the words go to shared memory and pass 2
        // ORs the four words of every 2x2 window (the pooled bit is the OR of the four
        // decisions, see fused_swap4_kernel).
        const int q = warp & 3, half = (warp - 4) >> 2;
        const int m0 = mt * 128 + q * 32;
        const bool wvalid = m0 < g.D;
        const int4 pc = wvalid ? __ldg(g.prm + m0 + lane) : make_int4(0x7fffffff, 0, 0, 0);
        const float Tf = float(pc.x);  // exact: |Tu| <= K < 2^24
        const float Tm1 = Tf - 1.0f;    // ge_bits form of the same threshold
        const bool flip = pc.y != 0;
        const int oword = m0 >> 5;
        const int nch = (g.dbg_mode & 1) ? 0 : (g.N + 31) >> 5;
        const int Hh = g.H >> 1, Wh = g.W >> 1;
        const int nwch = (g.W + 31) >> 5;  // pooled units per row pair and slot
        const int npu = (g.dbg_mode & 1) ? 0 : (g.TR >> 1) * g.G * nwch;
        int i = 0, ts = 0;
        HClock ce;
        long long t_ld = 0, t_cmp = 0, t_tile = 0, t_tail = 0;  // profile: unpooled chunk time in TMEM loads / in total
        for (int nt = n0; nt < g.n_tiles; nt += nstride, ++i) {
            const int acc = i & 1;
            ce.wait(prof, &tfull[acc], (i >> 1) & 1);
            const long long th0 = prof ? hclock() : 0;
            tc_fence_after();
            if (prof && i == 0 && warp == 4 && lane == 0) atomicAdd(g.dbg + 9, (unsigned long long)(hclock() - k_main));
            const uint32_t tb = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * g.N);
            const int r0 = nt * g.TR;
            if (!g.pool) {
                // the tile's column table (tile column -> NHWC output pixel, or -1 for frame columns
                // and images past the batch), written by the producers with the halo: slot ts of
                // the ring, whose next writer (tile i + nst + 2) waits for this tile's accumulator
                // release (tempty) through the halo and MMA barriers
                const int* tab = (g.dbg_mode & 2) ? nullptr : coltab + ts * kHMaxN;  // profile: no halo, no table
                if (++ts == g.nst + 2) ts = 0;
                // this warp's chunks are cc0, cc0 + 2, ... (the pair's first chunk alternates per
                // tile so odd chunk counts balance); two chunks per pass, both loads in flight
                const int cc0 = half ^ (i & 1);
                for (int cc = cc0; cc < nch; cc += 4) {
                    const bool two = cc + 2 < nch;  // warp-uniform
                    uint32_t v0[32], v1[32];
                    const long long c0 = prof ? hclock() : 0;
                    tmem_ld32(tb + uint32_t(32 * cc), v0);
                    if (two) tmem_ld32(tb + uint32_t(32 * (cc + 2)), v1);
                    tmem_ld_wait();
                    if (prof) t_ld += hclock() - c0;
                    const uint32_t fm = flip ? 0xFFFFFFFFu : 0u;
                    uint32_t m0 = ge_bits(v0, Tm1) ^ fm, m1 = two ? ge_bits(v1, Tm1) ^ fm : 0u;
                    m0 = transpose32(m0, lane);
                    if (two) m1 = transpose32(m1, lane);
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        if (k == 1 && !two) break;
                        const int col = 32 * (cc + 2 * k) + lane;
                        const int pix = tab && col < g.N ? tab[col] : -1;
                        if (pix >= 0 && wvalid) g.out[size_t(pix) * g.Dw + oword] = k ? m1 : m0;
                    }
                    if (prof) t_cmp += hclock() - c0;
                }
            } else {
                // units: (row pair, image slot, <= 32 columns), alternating between the two warps
                for (int u = half ^ (i & 1); u < npu; u += 2) {  // first unit alternates per tile
                    // (no integer division by runtime values: ~30 instructions each)
                    const int t2 = g.dNw.div(u), ch = u - t2 * nwch;
                    const int ti = g.dG.div(t2), slot = t2 - ti * g.G, ir = 2 * ti;
                    const int r = r0 + ir, grp = g.dS.div(r), h = r - grp * g.S;
                    const int b = grp * g.G + slot;
                    if (h >= g.H || b >= g.B) continue;  // frame rows, images past the batch (warp-uniform)
                    const int w0 = 32 * ch, wn = min(32, g.W - w0);
                    const uint32_t taddr = tb + uint32_t(ir * g.P + slot * g.Q + w0);
                    uint32_t* dst = g.out + (size_t(b * Hh + (h >> 1)) * Wh + (w0 >> 1)) * g.Dw + oword;
                    const uint32_t pitch = uint32_t(g.P);
                    const long long c0 = prof ? hclock() : 0;
                    switch (wn) {
                        case 32: pool_unit<32>(taddr, pitch, Tf, flip, lane, dst, size_t(g.Dw), wvalid); break;
                        case 16: pool_unit<16>(taddr, pitch, Tf, flip, lane, dst, size_t(g.Dw), wvalid); break;
                        case 8: pool_unit<8>(taddr, pitch, Tf, flip, lane, dst, size_t(g.Dw), wvalid); break;
                        case 4: pool_unit<4>(taddr, pitch, Tf, flip, lane, dst, size_t(g.Dw), wvalid); break;
                        default: pool_unit<2>(taddr, pitch, Tf, flip, lane, dst, size_t(g.Dw), wvalid); break;
                    }
                    if (prof) t_cmp += hclock() - c0, ++t_ld;  // pooled: unit time, unit count
                }
            }
            const long long tt0 = prof ? hclock() : 0;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);  // TMEM reads of this tile done
            if (prof) t_tile += tt0 - th0, t_tail += hclock() - tt0;
        }
        if (prof && warp == 4 && lane == 0) {
            atomicAdd(g.dbg + 6, (unsigned long long)ce.acc);
            atomicAdd(g.dbg + 7, (unsigned long long)(hclock() - k_main));
            atomicAdd(g.dbg + 10, (unsigned long long)t_ld);
            atomicAdd(g.dbg + 11, (unsigned long long)t_cmp);
            atomicAdd(g.dbg + 16, (unsigned long long)t_tile);
            atomicAdd(g.dbg + 17, (unsigned long long)t_tail);
        }
    } else if (warp == 2 || warp == 3 || warp >= 12) {
        // halo producers: canvas pixel j of the tile -> its Cw words (or the all-ones frame word)
        // -> e2m1 nibbles at [chunk][j][16 B]
        // (warps 2, 3, 12, 14, 15 and 13: six warps, so a 352-row halo (128-channel input at 16 x 16)
        // fills in one pass of two rows per thread; warp 13 shares the MMA warp's sub-partition,
        // measured: 0.1155 vs 0.1177 ms per step at batch 256, 4.07 vs 3.91 M img/s at 65536)
        const int pw = warp < 4 ? warp - 2 : warp == 12 ? 2 : warp == 13 ? 5 : warp - 11;
        const int pt = pw * 32 + lane;
        int hs = 0, ts = 0;
        uint32_t hph = 0;
        HClock cp;
        for (int nt = n0; nt < g.n_tiles; nt += nstride) {
            cp.wait(prof, &empty[hs], hph ^ 1);
            const uint32_t hb = sH + uint32_t(hs) * hbytes;
            int* tab = g.pool ? nullptr : coltab + ts * kHMaxN;
            if (++ts == g.nst + 2) ts = 0;
            const int q0 = nt * g.TR * g.P;
            const int nh = (g.dbg_mode & 2) ? 0 : g.NH;
            if (g.in_f32) {
                // first layer: sign bits of the pixel's creal float channels -> word 0; channels
                // 32..63 (zero weights) word 1; frame pixels all ones (sign(0.0) = +1)
                // two pixels per thread per pass, all their channel loads issued before use
                // (consecutive threads read consecutive pixels of a row: coalesced per channel)
                for (int j0 = pt; j0 < nh; j0 += 2 * kHProdThreads) {
                    long long pix[2];
                    const float* src[2];
                    const long long hw = (long long)g.H * g.W;
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int j = j0 + u * kHProdThreads;
                        pix[u] = j < nh ? halo_src(g, q0 + j) : -1;
                        const long long pp = pix[u] < 0 ? 0 : pix[u];
                        const long long b = pp / hw;
                        src[u] = g.in_f32 + (b * g.creal) * hw + (pp - b * hw);
                    }
                    uint32_t w0[2] = {0u, 0u};
                    int c = 0;
                    for (; c + 4 <= g.creal; c += 4) {
                        float v[2][4];
#pragma unroll
                        for (int u = 0; u < 2; ++u)
#pragma unroll
                            for (int k = 0; k < 4; ++k) v[u][k] = pix[u] >= 0 ? __ldg(src[u] + (c + k) * hw) : 0.0f;
#pragma unroll
                        for (int u = 0; u < 2; ++u)
#pragma unroll
                            for (int k = 0; k < 4; ++k) w0[u] |= uint32_t(v[u][k] >= 0.0f) << (c + k);
                    }
                    for (; c < g.creal; ++c) {
                        float v[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) v[u] = pix[u] >= 0 ? __ldg(src[u] + c * hw) : 0.0f;
#pragma unroll
                        for (int u = 0; u < 2; ++u) w0[u] |= uint32_t(v[u] >= 0.0f) << c;
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int j = j0 + u * kHProdThreads;
                        if (j >= nh) break;
                        put_col(g, tab, j, pix[u]);
                        const uint32_t dst = hb + uint32_t(j) * 16u;
                        // frame pixels all ones (sign(0.0) = +1); channels 32..63 carry zero weights
                        st_expand4(dst, pix[u] < 0 ? ~0u : w0[u]);
                        st_expand4(dst + lbo, pix[u] < 0 ? ~0u : 0u);
                    }
                }
            } else
            for (int j = pt; j < nh; j += 2 * kHProdThreads) {
                if ((g.Cw & 3) == 0)
                    fill_rows<4>(g, hb, lbo, q0, j, nh, tab);
                else
                    fill_rows<2>(g, hb, lbo, q0, j, nh, tab);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[hs]);
            if (++hs == g.nst) hs = 0, hph ^= 1;
        }
        if (prof && pt == 0) {
            atomicAdd(g.dbg + 4, (unsigned long long)cp.acc);
            atomicAdd(g.dbg + 5, (unsigned long long)(hclock() - k_main));
        }
    }
    // warp 0 (TMA) has nothing more to do: its one transaction is waited by the MMA warp
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 3] = hgtimer();
    if (prof && threadIdx.x == 0) {
        atomicAdd(g.dbg + 13, (unsigned long long)(hclock() - k_start));
        atomicMax(g.dbg + 15, hgtimer());
    }
}

namespace {

int round_up_i(int a, int b) { return (a + b - 1) / b * b; }

}  // namespace

// Host-side plan: canvas (images per canvas row G, frame kind), tile rows TR and MMA N, halo
// rows NH and stage count. Returns false when the layer is not a "same" conv this kernel covers
// or its weight slice does not fit in shared memory next to two halo stages.
bool halo4_plan(const FusedGeom& fg, HaloGeom& h) {
    if (fg.SH != 1 || fg.SW != 1) return false;
    if (fg.KH != 2 * fg.PH + 1 || fg.KW != 2 * fg.PW + 1 || fg.PH > 1 || fg.PW > 1) return false;
    if (fg.OH != fg.H || fg.OW != fg.W) return false;
    if (fg.C % 64 || fg.Cw != fg.C / 32 || fg.Cw > 16 || fg.D % 32) return false;
    if (fg.pool && (fg.H % 2 || fg.W % 2)) return false;
    // pooled epilogue units take 2..32 columns, a power of two (or whole 32-column chunks)
    if (fg.pool && !(fg.W % 32 == 0 || fg.W == 16 || fg.W == 8 || fg.W == 4 || fg.W == 2)) return false;
    const int K = fg.KH * fg.KW * fg.C;
    if (K != fg.K || K / 64 > kHaloMaxSteps) return false;
    const int KB4 = (K + 255) / 256;
    const int m_tiles = (fg.D + 127) / 128;
    const int sms = num_sms();
    if (sms < m_tiles) return false;
    const int per_m = sms / m_tiles;
    const int cpt = fg.C / 64;
    long best = -1;
    // weights resident (wst = 0) when the CTA's slice fits next to two halo stages, else a ring of
    // kHMaxWst streamed blocks (K chunks per tap a power of two)
    if (cpt & (cpt - 1)) return false;  // the unrolled issue loops take 1, 2, 4 or 8 K steps per tap
    for (int wst : {0, kHMaxWst}) {
        if (best >= 0) break;  // a resident plan exists
        const size_t wbytes = size_t(wst ? wst : KB4) * 16384;
        for (int G = 1; G <= 16; G *= 2) {
            if (G > 1 && G > fg.B) break;
            const int S = fg.pool ? fg.H + 2 : fg.H + 1;
            const int Q = fg.pool ? fg.W + 2 : fg.W + 1;
            const int P = fg.pool ? G * Q : G * Q + 1;
            const int rstep = fg.pool ? 2 : 1;
            if (rstep * P > kHMaxN) break;
            const int n_groups = (fg.B + G - 1) / G;
            const int total_rows = n_groups * S;
            for (int TR = rstep; TR * P <= kHMaxN; TR += rstep) {
                const int N = round_up_i(TR * P, 16);
                const int NH = round_up_i(N + 2 * P + 2, 8);
                const size_t hbytes = size_t(fg.Cw) * NH * 16;
                const size_t avail = kHSmemMax - 1024 - kHTail;
                if (wbytes + 2 * hbytes > avail) continue;
                const int n_tiles = (total_rows + TR - 1) / TR;
                const int ctas = std::min(per_m, n_tiles);
                const long rounds = (n_tiles + ctas - 1) / ctas;
                // MMA cycles per CTA (N/2 per step, plus a fixed per-tile cost); streamed: the
                // tile's weight blocks at ~40 B/cycle
                const long steps = K / 64;
                const long mma = steps * (N + 16) / 2;
                const long cost = rounds * (wst ? std::max(mma, long(KB4) * 16384 / 40) : mma);
                if (best < 0 || cost < best) {
                    best = cost;
                    h.G = G, h.S = S, h.Q = Q, h.P = P, h.TR = TR, h.N = N, h.NH = NH;
                    h.n_tiles = n_tiles, h.total_rows = total_rows;
                    h.nst = int(std::min<size_t>(kHMaxStages, (avail - wbytes) / hbytes));
                    h.grid = ctas * m_tiles;
                    h.wst = wst;
                }
            }
        }
    }
    if (best < 0) return false;
    h.in = static_cast<const uint32_t*>(fg.in);
    h.out = fg.out_bits;
    h.prm = fg.prm;
    h.B = fg.B, h.H = fg.H, h.W = fg.W, h.Cw = fg.Cw, h.D = fg.D, h.Dw = fg.Dw, h.pool = fg.pool;
    h.m_tiles = m_tiles;
    h.KB4 = KB4;
    h.steps = K / 64;
    h.dP = FastDiv::make(uint32_t(h.P));
    h.dS = FastDiv::make(uint32_t(h.S));
    h.dQ = FastDiv::make(uint32_t(h.Q));
    h.taps = fg.KH * fg.KW;
    h.cpt = fg.C / 64;
    for (int t = 0; t < 9; ++t) {
        const int ky = t / fg.KW, kx = t % fg.KW;
        h.toff[t] = t < h.taps ? (ky - fg.PH + 1) * h.P + (kx - fg.PW + 1) : 0;
    }
    h.smem = 1024 + size_t(h.wst ? h.wst : KB4) * 16384 + size_t(h.nst) * fg.Cw * h.NH * 16 + kHTail;
    h.dNw = FastDiv::make(uint32_t((fg.W + 31) / 32));
    h.dG = FastDiv::make(uint32_t(h.G));
    h.dbg = nullptr;
    h.dbg_mode = 0;
    h.in_f32 = nullptr;
    h.creal = 0;
    h.tl = nullptr;
    return true;
}

namespace {

// First-layer e2m1 weights for halo0: K' = T*64 positions, tap-major / channel-minor with the
// channels padded to 64 (zero weights past C); element e of a 32-group holds position
// 4 (e % 8) + e / 8 (put_word4's order); reference row bit r = (c*KH + kh)*KW + kw.
__global__ void prep_w4_pix_kernel(const uint32_t* __restrict__ packed, size_t wpl, int D, int C, int KH, int KW,
                                   int Dpad, int Kpad4, uint8_t* __restrict__ w4) {
    const size_t total = size_t(Dpad) * (Kpad4 / 2);
    const int T = KH * KW;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int d = int(i / (Kpad4 / 2)), e0 = int(i % (Kpad4 / 2)) * 2;
        uint8_t v = 0;
        for (int hh = 0; hh < 2; ++hh) {
            const int e = e0 + hh, q = e >> 5, el = e & 31;
            const int k = 32 * q + 4 * (el % 8) + el / 8;
            const int tap = k >> 6, c = k & 63;
            if (d >= D || tap >= T || c >= C) continue;
            const int kh = tap / KW, kw = tap - kh * KW, r = (c * KH + kh) * KW + kw;
            const uint32_t bit = (packed[size_t(d) * wpl + (r >> 5)] >> (r & 31)) & 1u;
            v |= uint8_t((bit ? 0x2 : 0xA) << (4 * hh));
        }
        w4[i] = v;
    }
}

}  // namespace

int prep_w4_pix(const uint32_t* packed, size_t wpl, int D, int C, int KH, int KW, int Dpad, int Kpad4, uint8_t* w4,
                cudaStream_t s) {
    const size_t total = size_t(Dpad) * (Kpad4 / 2);
    prep_w4_pix_kernel<<<unsigned(std::min<size_t>(ceil_div(total, 256), size_t(num_sms()) * 8)), 256, 0, s>>>(
        packed, wpl, D, C, KH, KW, Dpad, Kpad4, w4);
    return launch_check("prep_w4_pix_kernel");
}

int launch_halo4(const CUtensorMap& tm4, const HaloGeom& h, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(halo4_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHSmemMax)));
        BNN_CUDA(cudaFuncSetAttribute(halo4_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kHSmemMax)));
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(h.grid));
    cfg.blockDim = dim3(unsigned(kHThreads));
    cfg.dynamicSmemBytes = h.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const bool prof = getenv("BNN_HALO_PROFILE") != nullptr;
    HaloGeom ht = h;
    ht.tl = fused_timeline_slot(1);
    if (ht.tl) fused_timeline_name((std::string("halo4 D=") + std::to_string(h.D) + " C=" + std::to_string(h.Cw * 32) +
                                    " W=" + std::to_string(h.W) + (h.pool ? " pool" : "")).c_str());
    if (!prof) {
        BNN_CUDA(cudaLaunchKernelEx(&cfg, h.wst ? halo4_kernel<true> : halo4_kernel<false>, tm4, ht));
        BNN_TRY(launch_check("halo4_kernel"));
    } else {  // synchronous, not capturable: tools only
        HaloGeom hp = h;
        hp.dbg_mode = atoi(getenv("BNN_HALO_PROFILE")) >> 1;
        BNN_CUDA(cudaMalloc(&hp.dbg, 24 * sizeof(unsigned long long)));
        unsigned long long init[24] = {};
        init[14] = ~0ull;
        BNN_CUDA(cudaMemcpy(hp.dbg, init, sizeof init, cudaMemcpyHostToDevice));
        BNN_CUDA(cudaLaunchKernelEx(&cfg, h.wst ? halo4_kernel<true> : halo4_kernel<false>, tm4, hp));
        BNN_TRY(launch_check("halo4_kernel"));
        unsigned long long d[24];
        BNN_CUDA(cudaMemcpy(d, hp.dbg, sizeof d, cudaMemcpyDeviceToHost));
        cudaFree(hp.dbg);
        const double n = h.grid, k = 1e3;
        fprintf(stderr,
                "[halo4 mode=%d B=%d H=%d W=%d C=%d D=%d pool=%d | G=%d P=%d TR=%d N=%d NH=%d nst=%d tiles=%d grid=%d] "
                "span %.1f us | per-CTA kcyc: setup %.1f, total %.1f | mma: wait-w %.1f wait-acc %.1f wait-halo %.1f "
                "busy-total %.1f | prod: wait %.1f total %.1f | epi: wait %.1f total %.1f (chunks: ld %.1f all %.1f; pooled: units, all; tile body %.1f tail %.1f) | first halo %.1f first acc %.1f\n",
                hp.dbg_mode, h.B, h.H, h.W, h.Cw * 32, h.D, h.pool, h.G, h.P, h.TR, h.N, h.NH, h.nst, h.n_tiles, h.grid,
                (d[15] - d[14]) / 1e3, d[12] / n / k, d[13] / n / k, d[0] / n / k, d[1] / n / k, d[2] / n / k,
                d[3] / n / k, d[4] / n / k, d[5] / n / k, d[6] / n / k, d[7] / n / k, d[10] / n / k, d[11] / n / k, d[16] / n / k, d[17] / n / k, d[8] / n / k, d[9] / n / k);
    }
    set_last_gemm("halo4_kernel");
    return BNN_OK;
}

}  // namespace bnnk
