// Dev microbenchmark + layout check (not part of the library) for the halo conv design:
//  1. correctness of kind::mxf4 with A in TMEM (TS form, lane = row, 8 e2m1 nibbles per 32-bit
//     column, low nibble first) and B in shared memory, K-major, no swizzle, rows 16 B apart
//     starting at an arbitrary row offset (the tap shift of the halo tile); also the SS form;
//  2. cycles per dispatch of the TS form for the tile widths the halo kernel uses;
//  3. the SS form while other warps store to shared memory (producer contention).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_04477_b200/csrc \
//        tools/halo_probe.cu -o build/halo_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "umma.cuh"

using namespace bnnk::umma;

__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ uint64_t sdesc_k_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

__device__ __forceinline__ uint64_t sdesc_k_none(uint32_t addr, uint32_t lbo, uint32_t sbo);
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t sf, int acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sf), "r"(sf)
        : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sf, int acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sf), "r"(sf)
        : "memory");
}

constexpr int kRowsB = 320;  // allocated B rows per K chunk
constexpr int kSfCol = 496;  // 16 columns of 0x7F scale factors

// ---------------------------------------------------------------------------- correctness
// A: [128][64 bytes] packed nibbles (K = 128), B: [N][64 bytes]; out: [128][N] f32.
__global__ void __launch_bounds__(128, 1) check(const uint8_t* A, const uint8_t* B, int N, int shift, int ts, float* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t* sp = smem_raw + (base - raw);
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // A smem [4 chunks][128 rows][16 B] at base; B smem [4 chunks][kRowsB rows][16 B] at base + 8192
    for (int i = threadIdx.x; i < 128 * 4; i += blockDim.x) {
        const int r = i / 4, c = i % 4;
        memcpy(sp + c * 2048 + r * 16, A + r * 64 + c * 16, 16);
    }
    for (int i = threadIdx.x; i < kRowsB * 4; i += blockDim.x) {
        const int r = i / 4, c = i % 4;
        uint8_t* dst = sp + 8192 + c * kRowsB * 16 + r * 16;
        if (r >= shift && r - shift < N)
            memcpy(dst, B + (r - shift) * 64 + c * 16, 16);
        else
            memset(dst, 0xEE, 16);  // garbage rows: must not be read
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    const uint32_t lb = tm + (uint32_t(32 * warp) << 16);
    {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        tmem_st8(lb + kSfCol, v);
        tmem_st8(lb + kSfCol + 8, v);
        // A rows in TMEM at column 256: row = lane, 16 words
        const int r = 32 * warp + lane;
        uint32_t a0[8], a1[8];
        memcpy(a0, A + r * 64, 32);
        memcpy(a1, A + r * 64 + 32, 32);
        tmem_st8(lb + 256, a0);
        tmem_st8(lb + 264, a1);
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_mxf4(128, N);
        for (int s = 0; s < 2; ++s) {
            const uint64_t bd = sdesc_k_none(base + 8192 + 2 * s * kRowsB * 16 + 16 * shift, kRowsB * 16, 128);
            if (ts)
                mma_ts(tm, tm + 256 + 8 * s, bd, idesc, tm + kSfCol, s);
            else
                mma_ss(tm, sdesc_k_none(base + 2 * s * 2048, 2048, 128), bd, idesc, tm + kSfCol, s);
        }
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(lb + c0, v);
        tmem_ld_wait();
        for (int j = 0; j < 16; ++j) out[(32 * warp + lane) * N + c0 + j] = __uint_as_float(v[j]);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

static uint32_t rng = 12345;
static uint32_t nextr() {
    rng ^= rng << 13;
    rng ^= rng >> 17;
    rng ^= rng << 5;
    return rng;
}

static int run_check(int N, int shift, int ts) {
    const int M = 128, K = 128;
    std::vector<int> a(M * K), b(N * K);
    std::vector<uint8_t> ap(M * 64, 0), bp(N * 64, 0);
    for (int i = 0; i < M * K; ++i) a[i] = (nextr() & 1) ? 1 : -1;
    for (int i = 0; i < N * K; ++i) b[i] = nextr() & 1;
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) ap[m * 64 + k / 2] |= uint8_t((a[m * K + k] > 0 ? 0x2 : 0xA) << (4 * (k & 1)));
    for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) bp[n * 64 + k / 2] |= uint8_t((b[n * K + k] ? 0x2 : 0x0) << (4 * (k & 1)));
    uint8_t *dA, *dB;
    float* dO;
    cudaMalloc(&dA, ap.size());
    cudaMalloc(&dB, bp.size());
    cudaMalloc(&dO, M * N * 4);
    cudaMemcpy(dA, ap.data(), ap.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bp.data(), bp.size(), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    check<<<1, 128, 64 * 1024>>>(dA, dB, N, shift, ts, dO);
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<float> o(M * N);
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int s = 0;
            for (int k = 0; k < K; ++k) s += a[m * K + k] * b[n * K + k];
            if (float(s) != o[m * N + n]) {
                if (bad < 4) printf("   mismatch m=%d n=%d got %f want %d\n", m, n, o[m * N + n], s);
                ++bad;
            }
        }
    printf("check %s N=%3d shift=%d: %s (%d bad) err=%s\n", ts ? "TS" : "SS", N, shift, bad ? "FAIL" : "ok", bad,
           cudaGetErrorString(err));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dO);
    return bad;
}

// ---------------------------------------------------------------------------------- timing
// mode 0: TS; mode 1: SS; mode 2: SS while warps 1-3 store 16 B per lane continuously;
// mode 3: TS with the same store traffic.
template <int MODE>
__global__ void __launch_bounds__(128, 1) rate(int N, int iters, int shift, unsigned long long* out, int M = 128) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 120 * 1024 / 16; i += blockDim.x)
        st_shared_v4(base + 16 * i, 0x22222222u * (i & 1), 0x02020202u, 0u, 0x20202020u);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        fence_mbar_init();
        stop = 0;
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    {
        uint32_t v[32];
        for (int j = 0; j < 32; ++j) v[j] = 0x7F7F7F7Fu;
        tmem_st32(tm + (uint32_t(32 * warp) << 16) + 256, v);  // A region (any values)
        tmem_st32(tm + (uint32_t(32 * warp) << 16) + 288, v);
        tmem_st32(tm + (uint32_t(32 * warp) << 16) + 480, v);
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t b0 = base + 32768 + 16 * shift;
        const uint32_t idesc = idesc_mxf4(M, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int k = it & 3;
            const uint64_t bd = sdesc_k_none(b0 + 16 * kRowsB * 2 * (k & 1) + 16 * (k >> 1), 16 * kRowsB, 128);
            if (MODE == 0 || MODE == 3)
                mma_ts(tm, tm + 256 + 8 * k, bd, idesc, tm + 480, it != 0);
            else
                mma_ss(tm, sdesc_k_none(base + 4096 * k, 2048, 128), bd, idesc, tm + 480, it != 0);
        }
        long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        stop = 1;
        if (blockIdx.x == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    } else if ((MODE == 2 || MODE == 3) && warp >= 1) {
        // producer-like traffic into a region the MMA does not read
        const uint32_t dst = base + 96 * 1024 + 16 * (32 * (warp - 1) + lane);
        uint32_t x = threadIdx.x;
        long long n = 0;
        while (!stop) {
#pragma unroll 8
            for (int j = 0; j < 8; ++j) st_shared_v4(dst + 1536 * (j & 3), x, x + 1, x + 2, x + 3);
            x += 7;
            n += 8;
        }
        if (blockIdx.x == 0 && lane == 0) out[2 + warp] = n;
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int MODE>
void run_rate(int N, int shift, int M = 128) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto k = rate<MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 130 * 1024);
    const int iters = 8192;
    k<<<sms, 128, 130 * 1024>>>(N, 64, shift, d, M);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, 130 * 1024>>>(N, iters, shift, d, M);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[8];
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    const double cyc = double(h[1]) / iters;
    const double st_bytes = double(h[3] + h[4] + h[5]) * 32 * 16;
    static const char* names[] = {"TS", "SS", "SS+stores", "TS+stores"};
    printf("rate %-9s M=%3d N=%3d shift=%d: %6.1f cyc/mma (ideal at M=128 %5.1f)  %.1f T MAC-ops/s  stores %.1f B/cyc  err=%s\n",
           names[MODE], M, N, shift, cyc, N / 2.0, 2.0 * sms * iters * double(M) * N * 64 / (ms * 1e-3) / 1e12,
           st_bytes / double(h[1]), cudaGetErrorString(err));
    cudaFree(d);
}

// ------------------------------------------------------------- the halo kernel's MMA sequence
// A: KB4 SW128 blocks of 16 KB (resident weights), B: halo [cpt*2 chunks][NH rows][16 B];
// per tile: 9 taps x cpt steps, tap shifts (ky*P + kx) rows. FLAGS: 1 tap shifts zero,
// 2 A offsets fixed (block 0), 4 issue from `if (lane == 0)` instead of the converged warp.
__device__ __forceinline__ void mma_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sf, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sf)
        : "memory");
}

template <int FLAGS>
__global__ void __launch_bounds__(128, 1) seq(int N, int P, int cpt, int NH, int tiles, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KB4 = (9 * cpt + 3) / 4;
    const uint32_t hb = base + KB4 * 16384;
    for (int i = threadIdx.x; i < (KB4 * 16384 + 2 * cpt * NH * 16) / 16; i += blockDim.x)
        st_shared_v4(base + 16 * i, 0x22222222u * (i & 1), 0x02020202u, 0u, 0x20202020u);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot;
    {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        tmem_st8(tm + (uint32_t(32 * warp) << 16) + kSfCol, v);
        tmem_st8(tm + (uint32_t(32 * warp) << 16) + kSfCol + 8, v);
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint32_t idesc = idesc_mxf4(128, N);
        const uint32_t lbo = NH * 16;
        long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            const uint32_t d = tm + (t & 1) * ((FLAGS & 8) ? 256 : N);
            const uint64_t ad0 = sdesc_k_sw128(base);
            const uint64_t bd0 = sdesc_k_none(hb, lbo, 128);
            uint32_t aoff = 0;
            int s = 0;
            for (int tap = 0; tap < 9; ++tap) {
                uint32_t boff = (FLAGS & 1) ? 0 : uint32_t((tap / 3) * P + tap % 3);
                for (int c = 0; c < cpt; ++c, ++s) {
                    if (FLAGS & 4) {
                        if (lane == 0)
                            asm volatile(
                                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
                                "l"(ad0 + aoff), "l"(bd0 + boff), "r"(idesc), "r"(s != 0 ? 1 : 0), "r"(tm + kSfCol)
                                : "memory");
                    } else {
                        mma_warp(d, ad0 + aoff, bd0 + boff, idesc, tm + kSfCol, s != 0);
                    }
                    if (!(FLAGS & 2)) aoff += (s & 3) == 3 ? (16384u - 96u) / 16u : 2u;
                    boff += 2u * (lbo >> 4);
                }
            }
            if (FLAGS & 16) {  // a commit per tile (the kernel commits the halo stage and the accumulator)
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar2))
                    : "memory");
            }
        }
        long long t1 = clock64();
        if (lane == 0) {
            mma_commit(&bar);
            mbar_wait(&bar, 0);
        }
        __syncwarp();
        long long t2 = clock64();
        if (blockIdx.x == 0 && lane == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int FLAGS>
void run_seq(const char* name, int N, int P, int cpt, int NH) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto k = seq<FLAGS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int tiles = 100;
    k<<<sms, 128, 200 * 1024>>>(N, P, cpt, NH, 2, d);
    k<<<sms, 128, 200 * 1024>>>(N, P, cpt, NH, tiles, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double n = double(tiles) * 9 * cpt;
    printf("seq %-28s N=%3d P=%2d cpt=%d NH=%3d: %6.1f cyc/mma (ideal %5.1f), issue %6.1f  err=%s\n", name, N, P, cpt, NH,
           double(h[1]) / n, N / 2.0, double(h[0]) / n, cudaGetErrorString(err));
    cudaFree(d);
}

// ---------------------------------------------------------------- the kernel's issue path
// halo4_kernel's MMA issue (warp-uniform role, descriptors as 32-bit lo/hi adds, taps x CPT
// unrolled) and alternatives: V 0 elect.sync inside every MMA asm (the kernel), 1 one asm block
// per tap (elect once, CPT MMAs), 2 an elected lane issues the whole tile (CUTLASS style).
__device__ __forceinline__ void mma_lohi(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                         uint32_t sf, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 ad, bd;\n\t"
        "mov.b64 ad, {%1, %2};\n\t"
        "mov.b64 bd, {%3, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], ad, bd, %5, [%7], [%7], p;\n\t}" ::"r"(d),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc), "r"(sf)
        : "memory");
}
__device__ __forceinline__ void mma_plain(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi, uint32_t idesc,
                                          uint32_t sf, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\t"
        "mov.b64 ad, {%1, %2};\n\t"
        "mov.b64 bd, {%3, %4};\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], ad, bd, %5, [%7], [%7], p;\n\t}" ::"r"(d),
        "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc), "r"(sf)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(pred));
    return pred != 0;
}
// one tap, 2 K steps, elect once
__device__ __forceinline__ void mma_tap2(uint32_t d, uint32_t alo0, uint32_t alo1, uint32_t ahi, uint32_t blo0, uint32_t blo1,
                                         uint32_t bhi, uint32_t idesc, uint32_t sf, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a0, a1, b0, b1;\n\t"
        "mov.b64 a0, {%1, %3};\n\tmov.b64 a1, {%2, %3};\n\t"
        "mov.b64 b0, {%4, %6};\n\tmov.b64 b1, {%5, %6};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %8, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a0, b0, %7, [%9], [%9], p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], a1, b1, %7, [%9], [%9], 1;\n\t}" ::"r"(d),
        "r"(alo0), "r"(alo1), "r"(ahi), "r"(blo0), "r"(blo1), "r"(bhi), "r"(idesc), "r"(acc0), "r"(sf)
        : "memory");
}

template <int V, int CPT>
__global__ void __launch_bounds__(128, 1) seq2(int N, int P, int NH, int tiles, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    __shared__ uint64_t bar, bar2, bar3, bar4;
    __shared__ uint32_t tslot;
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int KB4 = (9 * CPT + 3) / 4;
    const uint32_t hb = base + KB4 * 16384;
    for (int i = threadIdx.x; i < (KB4 * 16384 + 2 * CPT * NH * 16) / 16; i += blockDim.x)
        st_shared_v4(base + 16 * i, 0x22222222u * (i & 1), 0x02020202u, 0u, 0x20202020u);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar2, 1);
        mbar_init(&bar3, 1);
        mbar_init(&bar4, 1);
        fence_mbar_init();
        mbar_arrive(&bar3);  // phase 0 complete: waits on parity 0 return at once
    }
    if (warp == 0) tmem_alloc<512>(&tslot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = __shfl_sync(0xffffffffu, tslot, 0);
    {
        uint32_t v[8];
        for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
        tmem_st8(tm + (uint32_t(32 * warp) << 16) + kSfCol, v);
        tmem_st8(tm + (uint32_t(32 * warp) << 16) + kSfCol + 8, v);
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        const uint32_t idesc = idesc_mxf4(128, N);
        const uint32_t lbo = NH * 16;
        uint32_t toff[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) toff[t] = uint32_t((t / 3) * P + t % 3);
        const uint64_t ad0 = sdesc_k_sw128(base);
        const uint64_t bd0 = sdesc_k_none(hb, lbo, 128);
        const uint32_t alo = uint32_t(ad0), ahi = uint32_t(ad0 >> 32), blo = uint32_t(bd0), bhi = uint32_t(bd0 >> 32);
        const uint32_t sf = tm + kSfCol, step16 = 2u * (lbo >> 4);
        long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            const uint32_t d = tm + (t & 1) * N;
            if constexpr (V >= 3) {  // the kernel's per-tile waits (already-completed phases) and fence
                mbar_wait(&bar3, 0);
                mbar_wait(&bar3, 0);
                tc_fence_after();
            }
            if constexpr (V == 0 || V >= 3) {
#pragma unroll
                for (int tp = 0; tp < 9; ++tp)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) {
                        const int st = tp * CPT + c;
                        mma_lohi(d, alo + uint32_t((st >> 2) * 1024 + (st & 3) * 2), ahi, blo + toff[tp] + uint32_t(c) * step16, bhi,
                                 idesc, sf, st != 0);
                    }
            } else if constexpr (V == 1) {
                static_assert(CPT == 2, "tap2");
#pragma unroll
                for (int tp = 0; tp < 9; ++tp) {
                    const int st = tp * 2;
                    mma_tap2(d, alo + uint32_t((st >> 2) * 1024 + (st & 3) * 2), alo + uint32_t(((st + 1) >> 2) * 1024 + ((st + 1) & 3) * 2),
                             ahi, blo + toff[tp], blo + toff[tp] + step16, bhi, idesc, sf, st != 0);
                }
            } else {
                if (elect_one()) {
#pragma unroll
                    for (int tp = 0; tp < 9; ++tp)
#pragma unroll
                        for (int c = 0; c < CPT; ++c) {
                            const int st = tp * CPT + c;
                            mma_plain(d, alo + uint32_t((st >> 2) * 1024 + (st & 3) * 2), ahi, blo + toff[tp] + uint32_t(c) * step16,
                                      bhi, idesc, sf, st != 0);
                        }
                }
                __syncwarp();
            }
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar2))
                : "memory");
            if constexpr (V >= 4)
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar4))
                    : "memory");
            if constexpr (V >= 5) __syncwarp();
        }
        long long t1 = clock64();
        if (lane == 0) {
            mma_commit(&bar);
            mbar_wait(&bar, 0);
        }
        __syncwarp();
        long long t2 = clock64();
        if (blockIdx.x == 0 && lane == 0) {
            out[0] = t1 - t0;
            out[1] = t2 - t0;
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <int V, int CPT>
void run_seq2(const char* name, int N, int P, int NH) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto k = seq2<V, CPT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int tiles = 100;
    k<<<sms, 128, 200 * 1024>>>(N, P, NH, 2, d);
    k<<<sms, 128, 200 * 1024>>>(N, P, NH, tiles, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double n = double(tiles) * 9 * CPT;
    printf("seq2 V%d %-22s N=%3d P=%2d cpt=%d NH=%3d: %6.1f cyc/mma (ideal %5.1f), issue %6.1f  err=%s\n", V, name, N, P, CPT, NH,
           double(h[1]) / n, N / 2.0, double(h[0]) / n, cudaGetErrorString(err));
    cudaFree(d);
}

// ---------------------------------------------------------------- TMEM load rate (tcgen05.ld)
// WPQ warps per lane quarter each load 32x32b.x32 (4 KB) `iters` times at column stride CS
// (aligned 32 or not), with (WAIT=1) or without a wait per load (WAIT=0: 4 loads per wait).
template <int WPQ, int WAIT>
__global__ void tmem_rate(int iters, int cs, unsigned long long* out) {
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tmem_alloc<512>(&tslot);
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tslot + (uint32_t(32 * (warp & 3)) << 16);
    uint32_t acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t v[32];
        if (WAIT) {
            tmem_ld32(tm + uint32_t((it * cs) & 255), v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += v[j];
        } else {
            uint32_t w[32];
            tmem_ld32(tm + uint32_t((it * cs) & 255), v);
            tmem_ld32(tm + uint32_t((it * cs + 64) & 255), w);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += v[j] ^ w[j];
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345678u) out[1] = acc;
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tslot);
}

template <int WPQ, int WAIT>
void run_tmem(int cs) {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096;
    tmem_rate<WPQ, WAIT><<<sms, 128 * WPQ>>>(64, cs, d);
    tmem_rate<WPQ, WAIT><<<sms, 128 * WPQ>>>(iters, cs, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double loads = double(iters) * (WAIT ? 1 : 2);
    printf("tmem ld32 warps/quarter=%d %s col stride %2d: %6.1f cyc per load per warp, SM rate %.1f B/cyc  err=%s\n", WPQ,
           WAIT ? "wait each" : "2 then wait", cs, double(h[0]) / loads, 4096.0 * 4 * WPQ * loads / double(h[0]),
           cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    run_tmem<1, 1>(32);
    run_tmem<1, 1>(17);
    run_tmem<2, 1>(32);
    run_tmem<2, 1>(34);
    run_tmem<1, 0>(32);
    run_tmem<2, 0>(32);
    run_tmem<4, 1>(32);
    if (getenv("HALO_PROBE_SKIP_SEQ")) return 0;
    // conv1 / conv3 / conv4 geometries of the halo kernel
    // (kind::mxf4 with M = 64 is an illegal instruction on sm_100a: run_rate<1>(n, 0, 64) faults)
    if (getenv("HALO_PROBE_SEQ2")) {
        run_seq2<0, 2>("kernel form", 208, 34, 280);
        run_seq2<3, 2>("+ 2 waits per tile", 208, 34, 280);
        run_seq2<4, 2>("+ 2 commits", 208, 34, 280);
        run_seq2<5, 2>("+ syncwarp", 208, 34, 280);
        run_seq2<5, 4>("+ syncwarp", 144, 18, 184);
        run_seq2<1, 2>("asm per tap", 208, 34, 280);
        run_seq2<2, 2>("elected lane", 208, 34, 280);
        run_seq2<0, 4>("kernel form", 144, 18, 184);
        run_seq2<2, 4>("elected lane", 144, 18, 184);
        run_seq2<0, 4>("kernel form", 160, 10, 184);
        run_seq2<2, 4>("elected lane", 160, 10, 184);
        run_seq2<0, 2>("kernel form", 256, 34, 336);
        run_seq2<1, 2>("asm per tap", 256, 34, 336);
        run_seq2<2, 2>("elected lane", 256, 34, 336);
        return 0;
    }
    if (getenv("HALO_PROBE_SWEEP")) {
        // LBO (halo rows NH) and K steps per tap, N = 208 / 224 / 256
        for (int N : {208, 256})
            for (int nh = N + 72; nh <= N + 136; nh += 8) {
                run_seq<0>("sweep real", N, 34, 2, nh);
                run_seq<3>("sweep no shift, A fixed", N, 34, 2, nh);
            }
        run_seq<0>("cpt4 real", 208, 34, 4, 280);
        run_seq<3>("cpt4 no shift, A fixed", 208, 34, 4, 280);
        run_seq<0>("cpt2 real", 224, 37, 2, 304);
        run_seq<3>("cpt2 no shift, A fixed", 224, 37, 2, 304);
        run_seq<0>("cpt1 real", 208, 34, 1, 280);
        run_seq<0>("P mult 8 real", 208, 40, 2, 296);
        run_seq<0>("P mult 8 real", 208, 48, 2, 304);
        return 0;
    }
    run_seq<0>("warp, real", 208, 34, 2, 280);
    run_seq<1>("warp, no tap shift", 208, 34, 2, 280);
    run_seq<2>("warp, A fixed", 208, 34, 2, 280);
    run_seq<3>("warp, no shift, A fixed", 208, 34, 2, 280);
    run_seq<4>("lane0, real", 208, 34, 2, 280);
    run_seq<0>("warp, real", 144, 18, 4, 184);
    run_seq<1>("warp, no tap shift", 144, 18, 4, 184);
    run_seq<0>("warp, real", 224, 37, 4, 304);
    run_seq<1>("warp, no tap shift", 224, 37, 4, 304);
    run_seq<0>("warp, real", 256, 34, 2, 336);
    run_seq<0>("warp, real, NH mult 8 rows", 208, 40, 2, 296);
    run_seq<8>("warp, real, acc at 256", 208, 34, 2, 280);
    run_seq<16>("warp, real, commit per tile", 208, 34, 2, 280);
    run_seq<24>("warp, real, acc 256, commit", 208, 34, 2, 280);
    run_seq<8>("warp, real, acc at 256", 144, 18, 4, 184);
    run_seq<0>("warp, real", 160, 10, 4, 184);
    run_seq<8>("warp, real, acc at 256", 160, 10, 4, 184);

    int bad = 0;
    if (getenv("HALO_PROBE_ALL")) {
        for (int ts : {1, 0})
            for (int n : {144, 176, 256})
                for (int s : {0, 1, 3, 37}) bad += run_check(n, s, ts);
        for (int n : {128, 144, 160, 176, 208, 240, 256}) run_rate<0>(n, 3);
        for (int n : {144, 208, 256}) run_rate<1>(n, 3);
        for (int n : {144, 208, 256}) run_rate<2>(n, 3);
        for (int n : {144, 208, 256}) run_rate<3>(n, 3);
    }
    printf("checks: %s\n", bad ? "FAIL" : "all ok");
    return 0;
}
