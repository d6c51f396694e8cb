// FP4 (kind::mxf4) binary linear layer with split-K, for the fused engine's linear stages:
//
//   linear_forward_packed (network.cpp:113-126) = xnor_gemm(W, pack_cols(sign x)) -> to_float
//   -> bias_add, then (between layers) affine_norm -> htanh -> sign (network.cpp:151-175)
//
// The operands are the same exact e2m1 encodings as the FP4 conv kernels (fused.cu, halo.cu):
// weights {-1.0, +1.0} (prep_weights4, engine K order), activations {0.0, 1.0} (the packed bits
// of the previous layer, expanded in shared memory), block scales 2^0, so the f32 accumulator
// is the exact integer u = sum bit * w and the reference's xnor value is 2u - S_d.
//
// Tiles: 128 output features (UMMA M, the weight rows, TMA SW128) x NB images (UMMA N, the
// batch rows, expanded by the producer warps) x a K slice. The small-batch layers of the default
// network have few (feature, image) tiles and a deep K (fc 8192 -> 1024 at batch 256: 8 tiles),
// so K is split over CTAs: each slice writes its partial integer sums u (exact) to a workspace
// [split][B][Dpad] and lin_finish_kernel adds the slices and applies the epilogue: the next
// layer's packed bits (u >= Tu) ^ flip, or the logits float(2u - S_d) + bias in the reference's
// [features, batch] layout. Integer sums are order-independent, so the split is bit-exact.
// Without a split the tile's epilogue is final.
//
// CTA anatomy (448 threads): warp 0 weight TMA, warp 1 TMEM allocator + MMA issuer (the
// converged warp, one elected lane), warps 2-5 epilogue (lane = output feature), warps 6-13
// producers (thread = image row of the tile: its packed words -> e2m1 nibbles, SW128).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "bnn_common.cuh"
#include "fused.cuh"
#include "umma.cuh"

namespace bnnk {

using namespace umma;

namespace {

constexpr int kLThreads = 448;
constexpr int kLStages = 12;  // maximum ring depth (the weight stream is latency-bound at small NB)
constexpr int kLSfCol = 496;
constexpr int kLPre = 4;  // producer prefetch depth in K blocks
constexpr size_t kLSmem = 232448;  // 227 KB opt-in per CTA

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

// 32 activation bits -> 16 bytes of e2m1 nibbles at 16-byte chunk `chunk` of 128-byte row r of a
// SW128 tile (element 8s + n holds bit 4n + s: put_word4's order, matched by prep_weights4).
__device__ __forceinline__ void put_word4_sw(uint32_t tile, int r, int chunk, uint32_t w) {
    st_shared_v4(tile + uint32_t(r) * 128u + (uint32_t(chunk ^ (r & 7)) << 4), (w << 1) & 0x22222222u,
                 w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
}

// One 32-feature decision word of the next layer's input: packed bits, or (out4 set: the next
// layer TMA-loads its images) the 16 bytes of e2m1 {0, 1.0} codes expand_act4_kernel would make.
__device__ __forceinline__ void store_act(const LinGeom& g, size_t word, uint32_t w) {
    if (g.out4)
        reinterpret_cast<uint4*>(g.out4)[word] =
            make_uint4((w << 1) & 0x22222222u, w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
    else
        g.out_bits[word] = w;
}

__device__ __forceinline__ unsigned long long lgtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

}  // namespace

__global__ void __launch_bounds__(kLThreads, 1)
    lin4_kernel(const __grid_constant__ CUtensorMap tmW4, const __grid_constant__ CUtensorMap tmX4,
                const __grid_constant__ LinGeom g) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    const int nst = g.nst;
    uint8_t* sA = smem_raw + (base - raw);                  // [nst][128 rows x 128 B] weights
    uint8_t* sB = sA + size_t(nst) * 16384;                 // [nst][NB rows x 128 B] images
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(nst) * g.NB * 128);
    uint64_t* full = bars;
    uint64_t* empty = bars + kLStages;
    uint64_t* tfull = bars + 2 * kLStages;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const int warp = warp_uniform(int(threadIdx.x >> 5)), lane = threadIdx.x & 31;
    asm volatile("griddepcontrol.launch_dependents;");
    const int units = g.m_tiles * g.n_tiles * g.ksplit;
    const unsigned long long t_start = (g.dbg || g.tl) ? lgtimer() : 0;
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 0] = t_start;
    // BNN_LIN4_PROFILE: per-phase times (ns since the CTA started, summed over CTAs)
    auto stamp = [&](int k) {
        if (g.dbg) atomicAdd(g.dbg + k, lgtimer() - t_start);
    };
    if (threadIdx.x == 0) {
        tma_prefetch(&tmW4);
        if (g.tmab) tma_prefetch(&tmX4);
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], g.tmab ? 1 : 1 + 8);  // TMA arrive (expect_tx) [+ 8 producer warps]
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
        tmem_st8(lb + kLSfCol, v);
        tmem_st8(lb + kLSfCol + 8, v);
        tmem_st_wait();
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();

    // unit u -> (k slice, image tile, feature tile); slices of one tile are adjacent CTAs
    auto decode = [&](int u, int& mt, int& nt, int& ks) {
        ks = u % g.ksplit;
        const int t = u / g.ksplit;
        mt = t % g.m_tiles;
        nt = t / g.m_tiles;
    };
    auto kb_range = [&](int ks, int& kb0, int& kb1) {
        kb0 = ks * g.kbs;
        kb1 = min(g.KB4, kb0 + g.kbs);
    };

    if (warp == 0) {
        // weights: build-time constants, loaded ahead of the grid dependency (with TMA-loaded
        // images: the first ring's weights, then the wait, then both operands)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t btx = g.tmab ? uint32_t(g.NB) * 128u : 0u;
            int pre = 0;  // K blocks of the first unit whose weights went out before the wait
            if (g.tmab && int(blockIdx.x) < units) {
                // the whole first ring of weights ahead of the grid dependency, their images after
                int mt, nt, ks, kb0, kb1;
                decode(int(blockIdx.x), mt, nt, ks);
                kb_range(ks, kb0, kb1);
                pre = min(nst, kb1 - kb0);
                for (int j = 0; j < pre; ++j) {
                    mbar_arrive_expect_tx(&full[j], 16384 + btx);
                    tma_load_2d(&tmW4, &full[j], sA + size_t(j) * 16384, (kb0 + j) * 128, mt * 128);
                }
                asm volatile("griddepcontrol.wait;" ::: "memory");
                for (int j = 0; j < pre; ++j)
                    tma_load_2d(&tmX4, &full[j], sB + size_t(j) * g.NB * 128, (kb0 + j) * 128, nt * g.NB);
                stage = pre == nst ? 0 : pre;
                phase = pre == nst ? 1u : 0u;
            }
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int mt, nt, ks, kb0, kb1;
                decode(u, mt, nt, ks);
                kb_range(ks, kb0, kb1);
                for (int kb = kb0 + (u == int(blockIdx.x) ? pre : 0); kb < kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], 16384 + btx);
                    tma_load_2d(&tmW4, &full[stage], sA + size_t(stage) * 16384, kb * 128, mt * 128);
                    if (g.tmab) tma_load_2d(&tmX4, &full[stage], sB + size_t(stage) * g.NB * 128, kb * 128, nt * g.NB);
                    if (++stage == nst) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_mxf4_m128(g.NB);
        int stage = 0, i = 0;
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            int mt, nt, ks, kb0, kb1;
            decode(u, mt, nt, ks);
            kb_range(ks, kb0, kb1);
            mbar_wait(tempty, (i & 1) ^ 1);
            tc_fence_after();
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint32_t a0 = smem_u32(sA + size_t(stage) * 16384);
                const uint32_t b0 = smem_u32(sB + size_t(stage) * g.NB * 128);
                const int nk = kb == g.KB4 - 1 ? g.kq_last : 4;  // 64-element steps past K: zeros
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (k >= nk) break;
                    mma_mxf4_w(tmem_base, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                               tmem_base + kLSfCol, (kb != kb0 || k != 0));
                }
                mma_commit_w(&empty[stage]);
                if (kb == kb1 - 1) mma_commit_w(tfull);
                __syncwarp();
                if (++stage == nst) stage = 0, phase ^= 1;
            }
        }
        mbar_wait(tempty, (i & 1) ^ 1);  // the epilogue has read the last accumulator
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
        if (g.tl && lane == 0) g.tl[blockIdx.x * 4 + 1] = lgtimer();
    } else if (warp < 6) {
        // epilogue: lane = output feature d, TMEM columns = images
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (g.tl && warp == 2 && lane == 0) g.tl[blockIdx.x * 4 + 2] = lgtimer();
        const int q = warp & 3;
        int i = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
            int mt, nt, ks;
            decode(u, mt, nt, ks);
            const int d0 = mt * 128 + q * 32, d = d0 + lane, b0 = nt * g.NB;
            const bool dvalid = d < g.D;
            if (warp == 2 && lane == 0) stamp(0);
            mbar_wait(tfull, i & 1);
            if (warp == 2 && lane == 0) stamp(1);
            tc_fence_after();
            const uint32_t tb = tmem_base + (uint32_t(q * 32) << 16);
            int4 pd = make_int4(0x7fffffff, 0, 0, 0);
            if (g.ksplit == 1 && dvalid) pd = __ldg(g.prm + d);
            const float Tf = float(pd.x);
            const bool flip = pd.y != 0;
            for (int c = 0; c < g.NB / 32 + ((g.NB & 31) ? 1 : 0); ++c) {
                uint32_t v[32];
                tmem_ld32(tb + uint32_t(32 * c), v);
                tmem_ld_wait();
                const int bc = b0 + 32 * c;
                if (g.ksplit > 1) {
                    // partial sums: ws[ks][b][d], one coalesced 128-byte row per image
                    int* dst = g.ws + (size_t(ks) * g.B + bc) * g.Dpad + d;
                    if (d < g.Dpad) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (bc + j < g.B && bc + j < b0 + g.NB) dst[size_t(j) * g.Dpad] = int(__uint_as_float(v[j]));
                    }
                } else if (g.epi == FEPI_BITS) {
                    const uint32_t mine = decisions_transposed(v, Tf - 1.0f, flip, lane);
                    if (d0 < g.D && bc + lane < g.B && lane < g.NB - 32 * c)
                        store_act(g, size_t(bc + lane) * g.Dw + (d0 >> 5), mine);
                } else {
                    // to_float(a) + bias (kernels.cpp:90-107): one rounding of an exact integer
                    if (dvalid) {
                        const float bias = __int_as_float(pd.w);
                        float* orow = g.out_f32 + size_t(d) * g.ldo + bc;
                        auto val = [&](int j) { return __fadd_rn(__int2float_rn(2 * int(__uint_as_float(v[j])) - pd.z), bias); };
                        if (bc + 32 <= g.B && 32 * c + 32 <= g.NB && (g.ldo & 3) == 0 &&
                            (reinterpret_cast<uintptr_t>(g.out_f32) & 15) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)  // 16-byte stores: a quarter of the store instructions
                                *reinterpret_cast<float4*>(orow + j) = make_float4(val(j), val(j + 1), val(j + 2), val(j + 3));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (bc + j < g.B && 32 * c + j < g.NB) orow[j] = val(j);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty);
            if (warp == 2 && lane == 0) stamp(5);
        }
        if (g.ksplit > 1) __threadfence();  // partial sums visible GPU-wide before the arrival
    } else if (!g.tmab) {
        // producers: thread = image row r of the tile; per 256-element K block its 8 packed words
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const int r = int(threadIdx.x) - 6 * 32;  // 0..255
        int stage = 0;
        uint32_t phase = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int mt, nt, ks, kb0, kb1;
            decode(u, mt, nt, ks);
            kb_range(ks, kb0, kb1);
            const int b = nt * g.NB + r;
            const bool live = r < g.NB;
            const bool real = live && b < g.B;
            const uint32_t* src = g.in + size_t(real ? b : 0) * g.Kw;
            const bool vec = (g.Kw & 3) == 0;
            // the slice's words are loaded kLPre blocks ahead of their stage (one L2 round trip
            // per kLPre blocks instead of one per block)
            uint32_t pf[kLPre][8];
            auto load_block = [&](int kb, uint32_t (&w)[8]) {
                const int wq = 8 * kb;
                if (real && vec && wq + 8 <= g.Kw) {
                    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src + wq));
                    const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src + wq + 4));
                    w[0] = lo.x, w[1] = lo.y, w[2] = lo.z, w[3] = lo.w, w[4] = hi.x, w[5] = hi.y, w[6] = hi.z, w[7] = hi.w;
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) w[k] = (real && kb < kb1 && wq + k < g.Kw) ? __ldg(src + wq + k) : 0u;
                }
            };
#pragma unroll
            for (int p = 0; p < kLPre; ++p)
                if (kb0 + p < kb1) load_block(kb0 + p, pf[p]);
            for (int kb = kb0; kb < kb1; kb += kLPre) {
#pragma unroll
                for (int p = 0; p < kLPre; ++p) {
                    if (kb + p >= kb1) break;
                    uint32_t w[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) w[k] = pf[p][k];
                    if (kb + p + kLPre < kb1) load_block(kb + p + kLPre, pf[p]);
                    mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t tile = smem_u32(sB + size_t(stage) * g.NB * 128);
                    if (live) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) put_word4_sw(tile, r, k, w[k]);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[stage]);
                    if (++stage == nst) stage = 0, phase ^= 1;
                }
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (g.ksplit > 1) {
        // Split-K completion in the same launch (one unit per CTA when split: lin4_plan). Once
        // every slice of this (feature, image) tile has written its partial sums, slice ks
        // reduces images [ks*chunk, (ks+1)*chunk) of the tile with all 14 warps: a warp takes one
        // image, lane = 4 consecutive features (16-byte loads), 3 shuffles assemble each 32-feature
        // word. All slices are co-resident (grid <= SMs, one CTA per SM, and the dependent launch
        // waits until every CTA has started), so the spin cannot hang.
        int mt, nt, ks;
        decode(blockIdx.x, mt, nt, ks);
        unsigned* arrive = g.sem + 2 * (blockIdx.x / g.ksplit);
        if (threadIdx.x == 0) {
            stamp(2);
            __threadfence();  // this CTA's partial sums (the epilogue warps' stores, ordered by the barrier)
            atomicAdd(arrive, 1u);
            while (ld_acquire(arrive) < unsigned(g.ksplit)) __nanosleep(32);
            stamp(3);
        }
        __syncthreads();
        const int b0 = nt * g.NB, m0 = mt * 128;
        const int chunk = (g.NB + g.ksplit - 1) / g.ksplit;
        const int bb0 = b0 + ks * chunk, bb1 = min(min(b0 + g.NB, g.B), bb0 + chunk);
        const int d = m0 + 4 * lane;  // this lane's 4 features
        const bool dv = d < g.Dpad;
        int4 p4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) p4[k] = d + k < g.D ? __ldg(g.prm + d + k) : make_int4(0x7fffffff, 0, 0, 0);
        for (int b = bb0 + warp; b < bb1; b += kLThreads / 32) {
            int4 acc = make_int4(0, 0, 0, 0);
            if (dv) {
                for (int sl = 0; sl < g.ksplit; ++sl) {
                    const int4 v = __ldcg(reinterpret_cast<const int4*>(g.ws + (size_t(sl) * g.B + b) * g.Dpad + d));
                    acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
                }
            }
            const int uu[4] = {acc.x, acc.y, acc.z, acc.w};
            if (g.epi == FEPI_BITS) {
                uint32_t bits = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) bits |= uint32_t((uu[k] >= p4[k].x) != (p4[k].y != 0)) << k;
                uint32_t w = bits << (4 * (lane & 7));
                w |= __shfl_xor_sync(0xffffffffu, w, 1);
                w |= __shfl_xor_sync(0xffffffffu, w, 2);
                w |= __shfl_xor_sync(0xffffffffu, w, 4);
                if ((lane & 7) == 0 && d < g.D) store_act(g, size_t(b) * g.Dw + (d >> 5), w);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (d + k < g.D)
                        g.out_f32[size_t(d + k) * g.ldo + b] =
                            __fadd_rn(__int2float_rn(2 * uu[k] - p4[k].z), __int_as_float(p4[k].w));
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            stamp(4);
            if (atomicAdd(arrive + 1, 1u) == unsigned(g.ksplit - 1)) {
                arrive[0] = 0;  // every slice of the tile is past its wait and its reads
                arrive[1] = 0;
            }
        }
    }
    if (threadIdx.x == 0) stamp(6);
    if (g.tl && threadIdx.x == 0) g.tl[blockIdx.x * 4 + 3] = lgtimer();
}

// Images [B, Kw] packed bits -> e2m1 lines [B, Kw * 16 B]: word q of image b becomes the 16
// bytes put_word4_sw writes for it (codes 0x2 = 1.0 for a set bit, 0x0 for a clear one), so a
// TMA SW128 box of these lines is the producers' tile byte for byte. Pad bits are 0 -> 0.0.
__global__ void __launch_bounds__(256) expand_act4_kernel(const uint32_t* __restrict__ in, size_t n, uint4* __restrict__ out) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = __ldg(in + i);
        out[i] = make_uint4((w << 1) & 0x22222222u, w & 0x22222222u, (w >> 1) & 0x22222222u, (w >> 2) & 0x22222222u);
    }
}

int launch_expand_act4(const LinGeom& l, cudaStream_t s) {
    const size_t n = size_t(l.B) * l.Kw;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(std::min<size_t>((n + 255) / 256, size_t(num_sms()) * 8)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BNN_CUDA(cudaLaunchKernelEx(&cfg, expand_act4_kernel, l.in, n, reinterpret_cast<uint4*>(l.in4)));
    return launch_check("expand_act4_kernel");
}

int g_lin4_tma = -2;  // -2 unread, -1 auto, 0 / 1 forced (bnn_set_fused_lin4 2 / 3, BNN_LIN4_TMA)
void set_lin4_tma(int mode) { g_lin4_tma = mode; }

// Host plan: images per tile (NB, <= 256, a multiple of 16), feature tiles of 128 and the K
// split that gives ~one wave of CTAs (at least 2 K blocks per slice, at most 8 slices).
bool lin4_plan(const FusedGeom& fg, int epi, LinGeom& l) {
    if (fg.KH != 1 || fg.KW != 1 || fg.H != 1 || fg.W != 1) return false;
    if (epi != FEPI_BITS && epi != FEPI_LOGITS) return false;
    if (fg.Cw * 32 < fg.K || fg.kb4 <= 0) return false;
    const int sms = num_sms();
    l.in = static_cast<const uint32_t*>(fg.in);
    l.B = fg.B, l.K = fg.K, l.Kw = fg.Cw, l.D = fg.D, l.Dw = (fg.D + 31) / 32;
    l.KB4 = fg.kb4, l.kq_last = fg.kq4;
    l.m_tiles = (fg.D + 127) / 128;
    // (NB, split) by a cycle model per CTA: MMA steps x max(48, NB/2) cycles (the measured
    // dispatch cost, tools/halo_probe.cu), the CTA's weight slice streamed at ~24 B/cycle, and
    // the partial-sum round trip of the in-kernel split-K completion.
    long best = -1;
    for (int nb = 256; nb >= 16; nb /= 2) {
        if (nb > 16 && nb / 2 >= (fg.B + 15) / 16 * 16) continue;  // narrower than the batch already
        const int nbr = std::min(nb, (fg.B + 15) / 16 * 16);
        const int nt = (fg.B + nbr - 1) / nbr;
        const int tiles = l.m_tiles * nt;
        for (int ks = 1; ks <= 16; ks *= 2) {
            if (ks > 1 && (l.KB4 + ks - 1) / ks < 2) break;
            const int kbs = (l.KB4 + ks - 1) / ks;
            const long units = long(tiles) * ((l.KB4 + kbs - 1) / kbs);
            if (ks > 1 && units > sms) break;  // split slices must all be co-resident (one round)
            const long rounds = (units + sms - 1) / sms;
            const long mma = long(kbs) * 4 * std::max(48, nbr / 2);
            // per CTA: the mainloop (MMA dispatch, or the weight slice streamed at ~24 B/cycle, plus
            // ~3000 cycles of first-load latency), the epilogue (~500 cycles per 32 images), and
            // when split: partial sums out (~32 B/cycle), the spin, and the reduction (14 warps,
            // ~1000 cycles per image each)
            const long wts = long(kbs) * 16384 / 24;
            const long main = std::max(mma, wts) + 3000;
            const long epi = ks > 1 ? long(nbr) * 128 * 4 / 32 + 1500 + ((nbr + ks - 1) / ks + 13) / 14 * 1000
                                    : long((nbr + 31) / 32) * 500;
            const long cost = rounds * (main + epi);
            if (best < 0 || cost < best) {
                best = cost;
                l.NB = nbr, l.n_tiles = nt, l.kbs = kbs, l.ksplit = (l.KB4 + kbs - 1) / kbs;
            }
        }
    }
    if (const char* f = getenv("BNN_LIN4_FORCE")) {  // experiments: "NB,split" for every lin4 layer
        int nb = 0, ks = 0;
        if (sscanf(f, "%d,%d", &nb, &ks) == 2 && nb >= 16 && nb <= 256 && nb % 16 == 0 && ks >= 1) {
            l.NB = nb, l.n_tiles = (fg.B + nb - 1) / nb;
            l.kbs = (l.KB4 + ks - 1) / ks, l.ksplit = (l.KB4 + l.kbs - 1) / l.kbs;
            if (l.ksplit > 1 && l.m_tiles * l.n_tiles * l.ksplit > sms) return false;
        }
    }
    l.nst = int(std::min<size_t>(kLStages, (kLSmem - 1024 - 256) / (16384 + size_t(l.NB) * 128)));
    l.Dpad = (fg.D + 31) / 32 * 32;
    l.prm = fg.prm;
    l.epi = epi;
    l.out_bits = fg.out_bits;
    l.out_f32 = fg.out_f32;
    l.ldo = fg.ldo;
    l.ws = nullptr;
    l.sem = nullptr;
    l.dbg = nullptr;
    l.tl = nullptr;
    // Images TMA-loaded from a once-expanded e2m1 copy (expand_act4_kernel, one extra launch)
    // instead of expanded by the producers in every CTA: pays when each image row would be
    // expanded by many feature tiles (BNN_LIN4_TMA=0/1 forces it off/on).
    if (g_lin4_tma == -2) g_lin4_tma = getenv("BNN_LIN4_TMA") ? atoi(getenv("BNN_LIN4_TMA")) : -1;
    l.tmab = g_lin4_tma >= 0 ? (g_lin4_tma != 0) : (l.m_tiles >= 4 && fg.B >= 512);
    l.in4 = nullptr;
    l.out4 = nullptr;
    return true;
}

size_t lin4_sem_count(const LinGeom& l) { return l.ksplit > 1 ? size_t(2) * l.m_tiles * l.n_tiles : 0; }

size_t lin4_ws_bytes(const LinGeom& l) { return l.ksplit > 1 ? size_t(l.ksplit) * l.B * l.Dpad * sizeof(int) : 0; }

int launch_lin4(const CUtensorMap& tm4, const CUtensorMap& tmx, const LinGeom& l, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        BNN_CUDA(cudaFuncSetAttribute(lin4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kLSmem)));
        attr_set = true;
    }
    const int units = l.m_tiles * l.n_tiles * l.ksplit;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(std::min(units, num_sms())));
    cfg.blockDim = dim3(unsigned(kLThreads));
    cfg.dynamicSmemBytes = 1024 + size_t(l.nst) * (16384 + size_t(l.NB) * 128) + 256;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const bool prof = getenv("BNN_LIN4_PROFILE") != nullptr;
    LinGeom lt = l;
    lt.tl = fused_timeline_slot(1);
    if (lt.tl) fused_timeline_name(("lin4 D=" + std::to_string(l.D) + " K=" + std::to_string(l.K) + " split=" +
                                    std::to_string(l.ksplit)).c_str());
    if (!prof) {
        BNN_CUDA(cudaLaunchKernelEx(&cfg, lin4_kernel, tm4, tmx, lt));
        BNN_TRY(launch_check("lin4_kernel"));
    } else {  // synchronous, not capturable: tools only
        LinGeom lp = l;
        BNN_CUDA(cudaMalloc(&lp.dbg, 8 * sizeof(unsigned long long)));
        BNN_CUDA(cudaMemset(lp.dbg, 0, 8 * sizeof(unsigned long long)));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        BNN_CUDA(cudaLaunchKernelEx(&cfg, lin4_kernel, tm4, tmx, lp));
        cudaEventRecord(e1, s);
        BNN_TRY(launch_check("lin4_kernel"));
        BNN_CUDA(cudaStreamSynchronize(s));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long d[8];
        BNN_CUDA(cudaMemcpy(d, lp.dbg, sizeof d, cudaMemcpyDeviceToHost));
        cudaFree(lp.dbg);
        const double n = double(cfg.gridDim.x) * 1e3;
        fprintf(stderr,
                "[lin4 B=%d K=%d D=%d | NB=%d m=%d n=%d split=%d kbs=%d nst=%d grid=%u] %.1f us | per-CTA us since start: "
                "epi ready %.2f, acc full %.2f, epilogue done %.2f, partials out %.2f, slices in %.2f, reduced %.2f, "
                "CTA end %.2f\n",
                l.B, l.K, l.D, l.NB, l.m_tiles, l.n_tiles, l.ksplit, l.kbs, l.nst, cfg.gridDim.x, ms * 1e3, d[0] / n,
                d[1] / n, d[5] / n, d[2] / n, d[3] / n, d[4] / n, d[6] / n);
    }
    set_last_gemm("lin4_kernel");
    return BNN_OK;
}

}  // namespace bnnk
