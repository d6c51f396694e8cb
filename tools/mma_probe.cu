// Dev microbenchmark (not part of the library): cycles per tcgen05.mma dispatch on this chip,
// for the operand kinds and layouts the conv kernels can use. One CTA per SM, one thread issues
// `iters` MMAs back to back on fixed shared-memory operands, then commits and waits; the other
// warps only write the block scale factors. Prints one line per configuration.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1911_04477_b200/csrc \
//        tools/mma_probe.cu -o build/mma_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "umma.cuh"

using namespace bnnk::umma;

__host__ __device__ constexpr uint32_t idesc_mxf4(int M, int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);
}

// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 contiguous bytes); LBO = K-direction
// core-matrix stride, SBO = 8-row-group stride.
__device__ __forceinline__ uint64_t sdesc_k_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((addr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

template <int KIND, int LAYOUT>  // KIND 0 = i8, 1 = mxf4; LAYOUT 0 = SW128, 1 = none
__global__ void __launch_bounds__(128, 1) probe(int N, int iters, int shift, unsigned long long* out) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
        st_shared_v4(base + 16 * i, 0x22222222u * (i & 1), 0x02020202u, 0u, 0x20202020u);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
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
        tmem_st32(tm + (uint32_t(32 * warp) << 16) + 448, v);
        tmem_st32(tm + (uint32_t(32 * warp) << 16) + 480, v);
        tmem_st_wait();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a0 = base, b0 = base + 32768 + 16 * shift;
        uint32_t idesc = KIND == 1 ? idesc_mxf4(128, N) : idesc_i8(128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int k = it & 3;
            uint64_t ad, bd;
            if (LAYOUT == 0) {
                ad = sdesc_k_sw128(a0 + 32 * k);
                bd = sdesc_k_sw128(b0 + 32 * k);
            } else {
                // A: [2 K-chunks][128 rows][16 B] -> LBO 2048, SBO 128;
                // B: [2 K-chunks][N + shift rows][16 B] -> LBO = 16 * 320, SBO 128
                ad = sdesc_k_none(a0 + 4096 * k, 2048, 128);
                bd = sdesc_k_none(b0 + 16 * 320 * 2 * k, 16 * 320, 128);
            }
            if (KIND == 1) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(it != 0 ? 1 : 0), "r"(tm + 448), "r"(tm + 480)
                    : "memory");
            } else {
                mma_i8(tm, ad, bd, idesc, it != 0);
            }
        }
        long long t1 = clock64();
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0) {
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

template <int KIND, int LAYOUT>
void run(int N, int shift, int sms) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    auto k = probe<KIND, LAYOUT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 8192;
    k<<<sms, 128, 100 * 1024>>>(N, 64, shift, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, 100 * 1024>>>(N, iters, shift, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double kel = KIND == 1 ? 64 : 32;
    const double macs = double(sms) * iters * 128.0 * N * kel;
    printf("%-5s %-6s N=%3d shift=%d sms=%3d: %7.1f cyc/mma (issue %6.1f)  %.3f ms  %.1f T MAC-ops/s  err=%s\n",
           KIND ? "mxf4" : "i8", LAYOUT ? "none" : "sw128", N, shift, sms, double(h[1]) / iters, double(h[0]) / iters, ms,
           2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int n : {64, 128, 192, 224, 256}) run<1, 0>(n, 0, sms);
    for (int n : {64, 128, 192, 224, 256}) run<1, 1>(n, 0, sms);
    for (int s : {1, 2, 3}) run<1, 1>(256, s, sms);
    for (int n : {128, 256}) run<0, 0>(n, 0, sms);
    for (int n : {128, 256}) run<0, 1>(n, 0, sms);
    run<1, 0>(256, 0, 1);
    run<1, 1>(256, 0, 1);
    return 0;
}
