// Pipe-peak microbenchmarks behind the K3 choice: the binary-op rate
// each GEMM candidate's instruction mix can reach on THIS chip at THIS run's clocks.
//
//   popc : the inner loop of candidate A with the shared-memory traffic removed — an 8x8
//          register tile of LOP3 (xor) + POPC + IADD per 32 bit-MACs.
//   bmma : candidate B, `mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc`. On sm_100a
//          ptxas lowers it to a CALL into an emulation routine built on IMMA.16832.U8 plus
//          bit-plane ALU work (no BMMA instruction exists); this measures what that is worth.
//
// Both report bops/s with bops = 2 per bit-MAC (SURVEY §8 notation).
#include "bnn_common.cuh"
#include "umma.cuh"

namespace bnnk {
namespace {

using namespace umma;

constexpr int kProbeIters = 2048;

__global__ void __launch_bounds__(256) popc_probe_kernel(uint32_t seed, int iters, int* sink) {
    uint32_t a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = seed * (threadIdx.x + 1) * 2654435761u + i * 40503u;
        b[i] = seed ^ (blockIdx.x * 97u + i * 131u + threadIdx.x);
    }
    int acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] += __popc(a[i] ^ b[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] += 0x9E3779B9u;  // defeat loop-invariant hoisting
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j];
    if (s == 0x7fffffff) *sink = s;
}

__global__ void __launch_bounds__(256) bmma_probe_kernel(uint32_t seed, int iters, int* sink) {
    // 4 independent accumulator chains per warp; A (16x256 bits) = 4 regs, B (256x8) = 2 regs
    uint32_t a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + 7 * i + 1) * 2654435761u;
#pragma unroll
    for (int i = 0; i < 2; ++i) b[i] = seed ^ (threadIdx.x * 131u + i);
    int c[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) c[k][i] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            asm volatile(
                "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.xor.popc "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                : "+r"(c[k][0]), "+r"(c[k][1]), "+r"(c[k][2]), "+r"(c[k][3])
                : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
        b[0] += 0x9E3779B9u;
    }
    int s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < 4; ++i) s += c[k][i];
    if (s == 0x7fffffff) *sink = s;
}

// tcgen05 dispatch rate: one CTA per SM, one thread issues `iters` back-to-back M=128 x N x K
// MMAs (K = 32 bytes of operand per row: K=32 int8, K=64 FP4) on fixed shared-memory operands
// (SWIZZLE_128B K-major, the layout the engine uses), then commits and waits. The rate the
// fused conv kernels are measured against (their roofline.peak cross-check).
// kind 0: kind::i8; kind 1: kind::mxf4 block-scaled (scales 2^0 in TMEM columns 448-511).
__global__ void __launch_bounds__(128, 1) umma_probe_kernel(int kind, int N, int iters, unsigned long long* cycles) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
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
#pragma unroll
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
        const uint32_t a0 = base, b0 = base + 16384;
        const uint32_t idesc = kind ? ((1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (8u << 24))
                                    : idesc_i8(128, N);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const int k = it & 3;
            const uint64_t ad = sdesc_k_sw128(a0 + 32 * k), bd = sdesc_k_sw128(b0 + 32 * k);
            if (kind) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(it != 0 ? 1 : 0), "r"(tm + 448), "r"(tm + 480)
                    : "memory");
            } else {
                mma_i8(tm, ad, bd, idesc, it != 0);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        if (blockIdx.x == 0) *cycles = (unsigned long long)(clock64() - t0);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(tm);
}

template <class Launch>
int time_probe(Launch launch, double ops, double* bops_per_s, double* ms_out, cudaStream_t s) {
    cudaEvent_t e0, e1;
    BNN_CUDA(cudaEventCreate(&e0));
    BNN_CUDA(cudaEventCreate(&e1));
    launch();  // warm-up (clocks ramp)
    launch();
    BNN_CUDA(cudaEventRecord(e0, s));
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    BNN_CUDA(cudaEventRecord(e1, s));
    BNN_TRY(launch_check("probe"));
    BNN_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms /= reps;
    if (ms_out) *ms_out = ms;
    if (bops_per_s) *bops_per_s = ops / (ms * 1e-3);
    return BNN_OK;
}

}  // namespace
}  // namespace bnnk

using namespace bnnk;

extern "C" {

int bnn_probe_popc_peak(double* bops_per_s, double* ms, bnn_stream_t st) {
    BNN_TRY(require_sm100());
    cudaStream_t s = S(st);
    Scratch sink;
    BNN_TRY(sink.alloc(4, s));
    const int blocks = num_sms() * 4;  // 8 warps x 4 CTAs = 32 warps per SM
    const double ops = double(blocks) * 256 * kProbeIters * 64 * 32 * 2;
    return time_probe([&] { popc_probe_kernel<<<blocks, 256, 0, s>>>(1u, kProbeIters, sink.as<int>()); },
                      ops, bops_per_s, ms, s);
}

int bnn_probe_bmma_peak(double* bops_per_s, double* ms, bnn_stream_t st) {
    BNN_TRY(require_sm100());
    cudaStream_t s = S(st);
    Scratch sink;
    BNN_TRY(sink.alloc(4, s));
    const int blocks = num_sms() * 4;
    const int iters = kProbeIters / 8;
    // per warp per iteration: 4 mma x (16 x 8 x 256) bit-MACs x 2
    const double ops = double(blocks) * (256 / 32) * iters * 4 * 16.0 * 8 * 256 * 2;
    return time_probe([&] { bmma_probe_kernel<<<blocks, 256, 0, s>>>(1u, iters, sink.as<int>()); },
                      ops, bops_per_s, ms, s);
}

// tcgen05 dispatch-rate probe: kind 0 = kind::i8 (K=32), 1 = kind::mxf4 (K=64), M=128, N in
// {64..256}; ops = 2 per MAC over all SMs; *cycles_per_mma from SM 0's clock.
int bnn_probe_umma_peak(int kind, int N, double* ops_per_s, double* cycles_per_mma, bnn_stream_t st) {
    BNN_TRY(require_sm100());
    if ((kind != 0 && kind != 1) || N < 64 || N > 256 || N % 16)
        return fail(BNN_E_CONFIG, "umma probe: kind 0 (i8) or 1 (mxf4), 64 <= N <= 256, N % 16 == 0");
    cudaStream_t s = S(st);
    Scratch cyc;
    BNN_TRY(cyc.alloc(8, s));
    const int smem = 64 * 1024 + 1024;
    BNN_CUDA(cudaFuncSetAttribute(umma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int blocks = num_sms(), iters = 8192;
    const double ops = 2.0 * blocks * iters * 128.0 * N * (kind ? 64 : 32);
    BNN_TRY(time_probe([&] { umma_probe_kernel<<<blocks, 128, smem, s>>>(kind, N, iters, cyc.as<unsigned long long>()); },
                       ops, ops_per_s, nullptr, s));
    unsigned long long c = 0;
    BNN_CUDA(cudaMemcpyAsync(&c, cyc.p, 8, cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    if (cycles_per_mma) *cycles_per_mma = double(c) / iters;
    return BNN_OK;
}

}  // extern "C"
