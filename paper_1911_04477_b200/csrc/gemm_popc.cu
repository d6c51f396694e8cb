// K3 candidate A — xnor-popcount GEMM on the integer pipes (LOP3 + POPC).
//
// Replaces xnor_gemm + to_float + bias_add + reshape_output (kernels.cpp:53-107,
// lowering.cpp:87-95). With both operands' pad bits zero, the reference's
//     2*sum_k popc(~(w_k ^ x_k)) - 32*wpl - pad          (kernels.hpp:46-54)
// equals L - 2*sum_k popc(w_k ^ x_k): pad positions xor to 0 and drop out. Integer
// results are exact, so the output is bit-identical to the reference.
//
// Shape: block tile BM x BN outputs, K staged BK words at a time through shared memory
// (double-buffered via register prefetch), each of the 256 threads accumulating a TM x TN
// register tile. The inner loop is one LOP3 (xor) + one POPC + one IADD per 32 bit-MACs;
// the POPC issue rate bounds it ("K3 candidates").
//
// This kernel serves every shape (any ld, any L, any M/N); the tcgen05 path (gemm_umma.cu)
// takes over for large GEMMs.
#include "bnn_common.cuh"

namespace bnnk {
namespace {

constexpr int kBK = 8;  // words (256 bits) of K per stage

enum EpiMode { EPI_S32 = 0, EPI_F32 = 1 };

struct EpiParams {
    int32_t* out_s32;
    size_t ldo;
    float* out_f32;
    const float* bias;
    size_t P;  // columns per image for the scattered f32 layout
};

template <int BM, int BN, int TM, int TN, int MODE>
__global__ void __launch_bounds__(256)
    xnor_gemm_popc_kernel(const uint32_t* __restrict__ w, size_t ldw, const uint32_t* __restrict__ x,
                          size_t ldx, int M, int N, int L, int wpl, EpiParams ep) {
    constexpr int NT = 256;
    static_assert((BM / TM) * (BN / TN) == NT, "tile/thread mismatch");
    constexpr int PAD = 4;
    __shared__ __align__(16) uint32_t As[2][kBK][BM + PAD];
    __shared__ __align__(16) uint32_t Bs[2][kBK][BN + PAD];
    constexpr int A_LOADS = BM * kBK / NT;
    constexpr int B_LOADS = BN * kBK / NT;

    const int t = threadIdx.x;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tx = t % (BN / TN), ty = t / (BN / TN);

    uint32_t ra[A_LOADS], rb[B_LOADS];
    auto gload = [&](int kt) {
        const int kb = kt * kBK;
#pragma unroll
        for (int q = 0; q < A_LOADS; ++q) {
            const int idx = t + q * NT, line = idx / kBK, kw = idx % kBK;
            const int gm = m0 + line, gk = kb + kw;
            ra[q] = (gm < M && gk < wpl) ? __ldg(w + size_t(gm) * ldw + gk) : 0u;
        }
#pragma unroll
        for (int q = 0; q < B_LOADS; ++q) {
            const int idx = t + q * NT, line = idx / kBK, kw = idx % kBK;
            const int gn = n0 + line, gk = kb + kw;
            rb[q] = (gn < N && gk < wpl) ? __ldg(x + size_t(gn) * ldx + gk) : 0u;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < A_LOADS; ++q) {
            const int idx = t + q * NT;
            As[buf][idx % kBK][idx / kBK] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < B_LOADS; ++q) {
            const int idx = t + q * NT;
            Bs[buf][idx % kBK][idx / kBK] = rb[q];
        }
    };

    int acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0;

    const int ktiles = (wpl + kBK - 1) / kBK;
    gload(0);
    sstore(0);
    __syncthreads();
    for (int kt = 0; kt < ktiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) gload(kt + 1);
#pragma unroll
        for (int k = 0; k < kBK; ++k) {
            uint32_t a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; i += 4) {
                const uint4 v = *reinterpret_cast<const uint4*>(&As[buf][k][ty * TM + i]);
                a[i] = v.x, a[i + 1] = v.y, a[i + 2] = v.z, a[i + 3] = v.w;
            }
#pragma unroll
            for (int j = 0; j < TN; j += 4) {
                const uint4 v = *reinterpret_cast<const uint4*>(&Bs[buf][k][tx * TN + j]);
                b[j] = v.x, b[j + 1] = v.y, b[j + 2] = v.z, b[j + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] += __popc(a[i] ^ b[j]);
        }
        if (kt + 1 < ktiles) sstore(buf ^ 1);
        __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int gm = m0 + ty * TM + i;
        if (gm >= M) continue;
        if (MODE == EPI_S32) {
            int32_t* orow = ep.out_s32 + size_t(gm) * ep.ldo;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int gn = n0 + tx * TN + j;
                if (gn < N) orow[gn] = L - 2 * acc[i][j];
            }
        } else {
            const float bv = ep.bias ? ep.bias[gm] : 0.0f;
#pragma unroll
            for (int j = 0; j < TN; ++j) {
                const int gn = n0 + tx * TN + j;
                if (gn >= N) continue;
                const size_t img = size_t(gn) / ep.P, p = size_t(gn) % ep.P;
                // to_float then bias_add: one rounding of (exact integer) + bias
                ep.out_f32[(img * M + gm) * ep.P + p] = float(L - 2 * acc[i][j]) + bv;
            }
        }
    }
}

template <int MODE>
int launch_popc(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N,
                size_t L, const EpiParams& ep, cudaStream_t s) {
    const int wpl = int(wpl_of(L));
    const size_t big_tiles = ceil_div(M, 128) * ceil_div(N, 128);
    if (big_tiles >= size_t(num_sms())) {
        dim3 grid(unsigned(ceil_div(N, 128)), unsigned(ceil_div(M, 128)));
        xnor_gemm_popc_kernel<128, 128, 8, 8, MODE>
            <<<grid, 256, 0, s>>>(w, ldw, x, ldx, int(M), int(N), int(L), wpl, ep);
    } else {
        dim3 grid(unsigned(ceil_div(N, 64)), unsigned(ceil_div(M, 64)));
        xnor_gemm_popc_kernel<64, 64, 4, 4, MODE>
            <<<grid, 256, 0, s>>>(w, ldw, x, ldx, int(M), int(N), int(L), wpl, ep);
    }
    set_last_gemm("popc");
    return launch_check("xnor_gemm_popc_kernel");
}

}  // namespace

// Shared argument validation (kernels.cpp:55-68 semantics).
int check_gemm_args(size_t ldw, size_t ldx, size_t M, size_t N, size_t L) {
    if (M == 0 || N == 0 || L == 0) return fail(BNN_E_SHAPE, "xnor_gemm: extents must be >= 1");
    const size_t wpl = wpl_of(L);
    if (ldw < wpl || ldx < wpl) return fail(BNN_E_SHAPE, "xnor_gemm: words-per-line mismatch");
    if (wpl * 32 > (size_t(1) << 26))
        return fail(BNN_E_SHAPE, "xnor_gemm: reduction length exceeds the accumulator guard");
    if (M > 0x7fffffff || N > 0x7fffffff)
        return fail(BNN_E_SHAPE, "xnor_gemm: extent exceeds 2^31-1");
    return BNN_OK;
}

int popc_gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N,
                  size_t L, int32_t* out, size_t ldo, cudaStream_t s) {
    EpiParams ep{out, ldo, nullptr, nullptr, 1};
    return launch_popc<EPI_S32>(w, ldw, x, ldx, M, N, L, ep, s);
}

int popc_gemm_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N,
                  size_t L, const float* bias, size_t P, float* out, cudaStream_t s) {
    EpiParams ep{nullptr, 0, out, bias, P ? P : N};
    return launch_popc<EPI_F32>(w, ldw, x, ldx, M, N, L, ep, s);
}

}  // namespace bnnk
