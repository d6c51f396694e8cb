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

namespace bnnk {
namespace {

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

}  // extern "C"
