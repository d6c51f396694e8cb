// K3 candidate C — the xnor-popcount GEMM on the 5th-generation tensor cores.
//
// tcgen05 has no 1-bit kind, and the legacy b1 mma.sync is software-emulated on sm_100a
// (probes.cu). But for v, w in {-1,+1}^L the xnor-popcount result IS the integer dot
// product:   L - 2*popc(a ^ w) = sum_k v_k * w_k   (kernels.hpp:46-54).
// So the packed lines are expanded to signed int8 {-1,+1} (pad positions 0, which add
// nothing) and multiplied with tcgen05.mma kind::i8 into exact int32 accumulators in TMEM.
// Every output is the same integer the reference computes.
//
// Kernel anatomy (persistent, one CTA per SM, 192 threads):
//   warp 0      TMA producer: A (weights, M x K int8) and B (lines, N x K int8) tiles,
//               K-major 128-byte rows, SWIZZLE_128B, into a kStages-deep smem ring
//   warp 1      TMEM allocator + single-thread UMMA issuer: M=128 x N=BN x K=32 per
//               instruction, 4 per 128-byte K block, commit -> smem slot release
//   warps 2-5   epilogue: TMEM -> registers (tcgen05.ld 32x32b.x32), int32 / float+bias
//               stores; two TMEM accumulator buffers so tile i's epilogue overlaps tile i+1's
//               MMAs.
#include <cuda.h>

#include <mutex>

#include "bnn_common.cuh"
#include "umma.cuh"

namespace bnnk {

using namespace umma;

namespace {

constexpr int kBM = 128;
constexpr int kBK = 128;  // bytes (= int8 elements) of K per stage: one swizzle atom row
constexpr int kStages = 4;
constexpr int kThreads = 192;

enum { UEPI_S32 = 0, UEPI_F32 = 1 };

struct UEpi {
    int32_t* out_s32;
    size_t ldo;
    float* out_f32;
    const float* bias;
    size_t P;
};

template <int BN>
constexpr size_t smem_bytes() {
    return 1024 /*align slack*/ + size_t(kStages) * (kBM + BN) * kBK + 256 /*barriers*/;
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    xnor_gemm_umma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          int M, int N, int K, UEpi ep) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base - smem_u32(smem_raw));
    uint8_t* sA = smem;                                  // [kStages][kBM * kBK]
    uint8_t* sB = smem + size_t(kStages) * kBM * kBK;    // [kStages][BN * kBK]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(kStages) * BN * kBK);
    uint64_t* full = bars;                 // [kStages]
    uint64_t* empty = bars + kStages;      // [kStages]
    uint64_t* tfull = bars + 2 * kStages;  // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tiles = (M + kBM - 1) / kBM, n_tiles = (N + BN - 1) / BN;
    const int tiles = m_tiles * n_tiles;
    const int kblocks = (K + kBK - 1) / kBK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<2 * BN>(tmem_slot);
    __syncwarp();  // reconverge role-divergent lanes: bar.sync counts a partial warp as whole
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int mt = t % m_tiles, nt = t / m_tiles;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], (kBM + BN) * kBK);
                    tma_load_2d(&tmA, &full[stage], sA + size_t(stage) * kBM * kBK, kb * kBK, mt * kBM);
                    tma_load_2d(&tmB, &full[stage], sB + size_t(stage) * BN * kBK, kb * kBK, nt * BN);
                    if (++stage == kStages) stage = 0, phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ UMMA issuer
        constexpr uint32_t idesc = idesc_i8(kBM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);  // epilogue drained this accumulator
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(sA + size_t(stage) * kBM * kBK);
                    const uint32_t b0 = smem_u32(sB + size_t(stage) * BN * kBK);
#pragma unroll
                    for (int k = 0; k < kBK / 32; ++k)
                        mma_i8(d_tmem, sdesc_k_sw128(a0 + 32 * k), sdesc_k_sw128(b0 + 32 * k), idesc,
                               (kb | k) != 0);
                    mma_commit(&empty[stage]);  // slot free once these MMAs have read it
                    if (kb == kblocks - 1) mma_commit(&tfull[acc]);
                }
                __syncwarp();
                if (++stage == kStages) stage = 0, phase ^= 1;
            }
            if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int mt = t % m_tiles, nt = t / m_tiles;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int m = mt * kBM + q * 32 + lane;
            const int n0 = nt * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c * 32), v);
                tmem_ld_wait();
                const int nb = n0 + c * 32;
                if (m < M && nb < N) {
                    if (EPI == UEPI_S32) {
                        int32_t* orow = ep.out_s32 + size_t(m) * ep.ldo + nb;
                        if (nb + 32 <= N && (ep.ldo & 3) == 0 && ((uintptr_t)ep.out_s32 & 15) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<int4*>(orow + j) =
                                    make_int4(int(v[j]), int(v[j + 1]), int(v[j + 2]), int(v[j + 3]));
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (nb + j < N) orow[j] = int(v[j]);
                        }
                    } else {
                        const float bv = ep.bias ? ep.bias[m] : 0.0f;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int n = nb + j;
                            if (n >= N) break;
                            const size_t img = size_t(n) / ep.P, p = size_t(n) % ep.P;
                            ep.out_f32[(img * M + m) * ep.P + p] = float(int(v[j])) + bv;
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) acc = 0, acc_phase ^= 1;
        }
    }

    __syncwarp();  // reconverge role-divergent lanes: bar.sync counts a partial warp as whole
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<2 * BN>(tmem_base);
}

// ------------------------------------------------------------------ tensor maps

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_fn() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(p);
    });
    return fn;
}

}  // namespace

// int8 matrix [rows, K] with row stride ld bytes (multiple of 16), box kBK x box_rows.
int make_tmap_2d_s8(CUtensorMap* map, const void* base, size_t rows, size_t K, size_t ld,
                    uint32_t box_rows) {
    PFN_encodeTiled enc = encode_fn();
    if (!enc) return fail(BNN_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (ld % 16 != 0 || (uintptr_t(base) & 15) != 0)
        return fail(BNN_E_CUDA, "TMA operand must be 16-byte aligned with a 16-byte row stride");
    cuuint64_t dims[2] = {K, rows};
    cuuint64_t strides[1] = {ld};
    cuuint32_t box[2] = {uint32_t(kBK), box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(BNN_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return BNN_OK;
}

namespace {

template <int BN, int EPI>
int launch_umma(const int8_t* a, size_t lda, const int8_t* b, size_t ldb, size_t M, size_t N, size_t K,
                const UEpi& ep, cudaStream_t s) {
    CUtensorMap ta, tb;
    BNN_TRY(make_tmap_2d_s8(&ta, a, M, K, lda, kBM));
    BNN_TRY(make_tmap_2d_s8(&tb, b, N, K, ldb, BN));
    auto kern = xnor_gemm_umma_kernel<BN, EPI>;
    BNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes<BN>())));
    const size_t tiles = ceil_div(M, kBM) * ceil_div(N, BN);
    const unsigned grid = unsigned(std::min<size_t>(tiles, size_t(num_sms())));
    kern<<<grid, kThreads, smem_bytes<BN>(), s>>>(ta, tb, int(M), int(N), int(K), ep);
    set_last_gemm("umma_i8");
    return launch_check("xnor_gemm_umma_kernel");
}

}  // namespace

// A: M x K int8 (+-1, 0 past L), row stride lda bytes; B: N x K int8, stride ldb.
int umma_gemm_s32(const int8_t* a, size_t lda, const int8_t* b, size_t ldb, size_t M, size_t N, size_t K,
                  int32_t* out, size_t ldo, cudaStream_t s) {
    UEpi ep{out, ldo, nullptr, nullptr, 1};
    if (N >= 256 * 8 || N % 256 == 0) return launch_umma<256, UEPI_S32>(a, lda, b, ldb, M, N, K, ep, s);
    return launch_umma<128, UEPI_S32>(a, lda, b, ldb, M, N, K, ep, s);
}

int umma_gemm_f32(const int8_t* a, size_t lda, const int8_t* b, size_t ldb, size_t M, size_t N, size_t K,
                  const float* bias, size_t P, float* out, cudaStream_t s) {
    UEpi ep{nullptr, 0, out, bias, P ? P : N};
    if (N >= 256 * 8 || N % 256 == 0) return launch_umma<256, UEPI_F32>(a, lda, b, ldb, M, N, K, ep, s);
    return launch_umma<128, UEPI_F32>(a, lda, b, ldb, M, N, K, ep, s);
}

}  // namespace bnnk
