// K1 — the sign-binarize + bit-pack encoder (and its strict / inverse twins).
//
// Replaces pack_rows / pack_cols / sign / htanh / unpack of the reference
// (binarize.cpp:19-90). Bit convention (tensor.hpp:63-70): bit 1 = +1, logical
// index 32k+b of a line is bit b of word k, pad bits 0. sign is `v >= 0`
// (binarize.cpp:9), so -0.0 -> +1 and NaN -> -1; the kernels use the same float
// comparison (FSETP.GE), never the IEEE sign bit.
//
// Both orientations are HBM-bound streams (4 bytes read per bit written):
//   rows: bits run along the contiguous dimension -> one coalesced 128-byte warp load
//         per word and __ballot_sync builds the word (VOTE.ANY); 32 words per warp are
//         kept one per lane so the word stores are coalesced too.
//   cols: bits run across rows -> each lane owns one column and accumulates 32 rows
//         (every row load is a coalesced 128-byte warp load); the [32 col x 8 word]
//         block tile is transposed through shared memory so the stores are line-contiguous.
#include "bnn_common.cuh"

namespace bnnk {
namespace {

constexpr int kColsWordsPerBlock = 8;

// STRICT = false: bit = (v >= 0)        -> pack_rows(sign(x))
// STRICT = true : bit = (v == +1), any v not in {+1,-1} records its row-major index
// E2M1 = true: each word is written as the 16 bytes of e2m1 {0, 1.0} codes the fused engine's
// TMA-fed linear kernel reads (expand_act4_kernel's format) to `words` viewed as uint4 [D, wpl].
template <bool STRICT, bool E2M1 = false>
__global__ void __launch_bounds__(256) pack_rows_kernel(const float* __restrict__ x, size_t D,
                                                        size_t L, uint32_t* __restrict__ words,
                                                        size_t ld, size_t wpl,
                                                        unsigned long long* first_bad) {
    // E2M1 (the fused engine's first layer): the dependent TMA-fed linear launch may start its
    // prologue and weight loads now; it waits for this grid before reading the images
    if (E2M1) asm volatile("griddepcontrol.launch_dependents;");
    const size_t warp = (size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t chunks = (wpl + 31) / 32;
    const size_t row = warp / chunks;
    if (row >= D) return;
    const size_t k0 = (warp % chunks) * 32;
    const float* src = x + row * L;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const size_t col = (k0 + j) * 32 + lane;
        v[j] = col < L ? __ldg(src + col) : -1.0f;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const size_t col = (k0 + j) * 32 + lane;
        bool bit;
        if (STRICT) {
            bit = v[j] == 1.0f && col < L;
            if (col < L && !(v[j] == 1.0f || v[j] == -1.0f))
                atomicMin(first_bad, (unsigned long long)(row * L + col));
        } else {
            bit = v[j] >= 0.0f && col < L;
        }
        const uint32_t wbits = __ballot_sync(0xffffffffu, bit);
        if (lane == j) mine = wbits;
    }
    if (k0 + lane < wpl) {
        if (E2M1)
            reinterpret_cast<uint4*>(words)[row * wpl + k0 + lane] =
                make_uint4((mine << 1) & 0x22222222u, mine & 0x22222222u, (mine >> 1) & 0x22222222u, (mine >> 2) & 0x22222222u);
        else
            words[row * ld + k0 + lane] = mine;
    }
}

template <bool STRICT>
__global__ void __launch_bounds__(256) pack_cols_kernel(const float* __restrict__ x, size_t L,
                                                        size_t N, uint32_t* __restrict__ words,
                                                        size_t ld, size_t wpl,
                                                        unsigned long long* first_bad) {
    __shared__ uint32_t tile[32][kColsWordsPerBlock + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const size_t j0 = size_t(blockIdx.x) * 32;
    const size_t k0 = size_t(blockIdx.y) * kColsWordsPerBlock;
    const size_t col = j0 + tx;
    const size_t word = k0 + ty;
    uint32_t w = 0;
    if (col < N && word < wpl) {
        const size_t r0 = word * 32;
        float v[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) v[b] = (r0 + b < L) ? __ldg(x + (r0 + b) * N + col) : -1.0f;
#pragma unroll
        for (int b = 0; b < 32; ++b) {
            if (STRICT) {
                if (r0 + b < L && !(v[b] == 1.0f || v[b] == -1.0f))
                    atomicMin(first_bad, (unsigned long long)((r0 + b) * N + col));
                w |= uint32_t(v[b] == 1.0f) << b;
            } else {
                w |= uint32_t(v[b] >= 0.0f && r0 + b < L) << b;
            }
        }
    }
    tile[tx][ty] = w;
    __syncthreads();
    const int t = ty * 32 + tx;
    const int line = t / kColsWordsPerBlock, kk = t % kColsWordsPerBlock;
    if (j0 + line < N && k0 + kk < wpl) words[(j0 + line) * ld + k0 + kk] = tile[line][kk];
}

// pack_cols with 16-byte loads: lane owns 4 adjacent columns, so one warp load covers 512
// contiguous bytes of a row (4x the bytes per request of the scalar kernel, which is what
// keeps this access pattern — 32 rows per word, each row a different DRAM page — near the
// HBM roofline). Needs N % 4 == 0 and a 16-byte aligned x. Block: 128 columns x 8 words.
template <bool STRICT>
__global__ void __launch_bounds__(256) pack_cols4_kernel(const float* __restrict__ x, size_t L,
                                                         size_t N, uint32_t* __restrict__ words,
                                                         size_t ld, size_t wpl,
                                                         unsigned long long* first_bad) {
    __shared__ uint32_t tile[128][kColsWordsPerBlock + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const size_t j0 = size_t(blockIdx.x) * 128;
    const size_t k0 = size_t(blockIdx.y) * kColsWordsPerBlock;
    const size_t col = j0 + 4 * tx;
    const size_t word = k0 + ty;
    uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
    if (col < N && word < wpl) {
        const size_t r0 = word * 32;
        const float4* src = reinterpret_cast<const float4*>(x + r0 * N + col);
        const size_t stride = N / 4;
#pragma unroll 8
        for (int b = 0; b < 32; ++b) {
            if (r0 + b < L) {
                const float4 v = __ldg(src + b * stride);
                if (STRICT) {
                    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (!(e[i] == 1.0f || e[i] == -1.0f))
                            atomicMin(first_bad, (unsigned long long)((r0 + b) * N + col + i));
                    w0 |= uint32_t(v.x == 1.0f) << b, w1 |= uint32_t(v.y == 1.0f) << b;
                    w2 |= uint32_t(v.z == 1.0f) << b, w3 |= uint32_t(v.w == 1.0f) << b;
                } else {
                    w0 |= uint32_t(v.x >= 0.0f) << b, w1 |= uint32_t(v.y >= 0.0f) << b;
                    w2 |= uint32_t(v.z >= 0.0f) << b, w3 |= uint32_t(v.w >= 0.0f) << b;
                }
            }
        }
    }
    tile[4 * tx + 0][ty] = w0;
    tile[4 * tx + 1][ty] = w1;
    tile[4 * tx + 2][ty] = w2;
    tile[4 * tx + 3][ty] = w3;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int t = i * 256 + ty * 32 + tx;
        const int line = t / kColsWordsPerBlock, kk = t % kColsWordsPerBlock;
        if (j0 + line < N && k0 + kk < wpl) words[(j0 + line) * ld + k0 + kk] = tile[line][kk];
    }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ words, size_t ld, size_t rows,
                              size_t cols, int col_packed, float* __restrict__ out) {
    const size_t n = rows * cols;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / cols, c = i % cols;
        const size_t line = col_packed ? c : r, bit = col_packed ? r : c;
        out[i] = ((words[line * ld + (bit >> 5)] >> (bit & 31)) & 1u) ? 1.0f : -1.0f;
    }
}

template <int OP>
__global__ void unary_kernel(const float* __restrict__ x, size_t n, float* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const float v = x[i];
        if (OP == 0)
            out[i] = v >= 0.0f ? 1.0f : -1.0f;  // binarize.cpp:9
        else
            out[i] = v > 1.0f ? 1.0f : (v < -1.0f ? -1.0f : v);  // binarize.cpp:10
    }
}

unsigned grid_for(size_t n, unsigned block) {
    size_t g = ceil_div(n, block);
    const size_t cap = size_t(num_sms()) * 16;
    return unsigned(g < cap ? (g ? g : 1) : cap);
}

int check_ld(size_t ld, size_t extent) {
    if (ld < wpl_of(extent))
        return fail(BNN_E_SHAPE, "leading dimension " + std::to_string(ld) +
                                     " words is smaller than ceil(extent/32) = " +
                                     std::to_string(wpl_of(extent)));
    return BNN_OK;
}

}  // namespace

int launch_pack_rows(const float* x, size_t D, size_t L, uint32_t* words, size_t ld,
                     unsigned long long* first_bad, cudaStream_t s) {
    if (D == 0 || L == 0) return fail(BNN_E_SHAPE, "pack_rows: extents must be >= 1");
    BNN_TRY(check_ld(ld, L));
    const size_t wpl = wpl_of(L);
    const size_t warps = D * ceil_div(wpl, 32);
    const unsigned blocks = unsigned(ceil_div(warps * 32, 256));
    if (first_bad)
        pack_rows_kernel<true><<<blocks, 256, 0, s>>>(x, D, L, words, ld, wpl, first_bad);
    else
        pack_rows_kernel<false><<<blocks, 256, 0, s>>>(x, D, L, words, ld, wpl, nullptr);
    return launch_check("pack_rows_kernel");
}

// pack_rows(sign(x)) written as e2m1 lines [D, wpl * 16 bytes] (the fused engine's first linear
// layer when its images are TMA-loaded: one pass instead of pack_rows + expand_act4).
int launch_pack_rows_e2m1(const float* x, size_t D, size_t L, void* out4, cudaStream_t s) {
    if (D == 0 || L == 0) return fail(BNN_E_SHAPE, "pack_rows: extents must be >= 1");
    const size_t wpl = wpl_of(L);
    const size_t warps = D * ceil_div(wpl, 32);
    const unsigned blocks = unsigned(ceil_div(warps * 32, 256));
    pack_rows_kernel<false, true><<<blocks, 256, 0, s>>>(x, D, L, static_cast<uint32_t*>(out4), wpl, wpl, nullptr);
    return launch_check("pack_rows_kernel");
}

int launch_pack_cols(const float* x, size_t L, size_t N, uint32_t* words, size_t ld,
                     unsigned long long* first_bad, cudaStream_t s) {
    if (L == 0 || N == 0) return fail(BNN_E_SHAPE, "pack_cols: extents must be >= 1");
    BNN_TRY(check_ld(ld, L));
    const size_t wpl = wpl_of(L);
    dim3 block(32, kColsWordsPerBlock);
    // 16-byte kernel when it still fills the GPU (>= 2 blocks per SM); small matrices take the
    // scalar kernel's 4x more blocks
    const bool wide_grid = ceil_div(N, 128) * ceil_div(wpl, kColsWordsPerBlock) >= size_t(2 * num_sms());
    if (N % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && wide_grid) {
        dim3 grid4(unsigned(ceil_div(N, 128)), unsigned(ceil_div(wpl, kColsWordsPerBlock)));
        if (first_bad)
            pack_cols4_kernel<true><<<grid4, block, 0, s>>>(x, L, N, words, ld, wpl, first_bad);
        else
            pack_cols4_kernel<false><<<grid4, block, 0, s>>>(x, L, N, words, ld, wpl, nullptr);
        return launch_check("pack_cols4_kernel");
    }
    dim3 grid(unsigned(ceil_div(N, 32)), unsigned(ceil_div(wpl, kColsWordsPerBlock)));
    if (first_bad)
        pack_cols_kernel<true><<<grid, block, 0, s>>>(x, L, N, words, ld, wpl, first_bad);
    else
        pack_cols_kernel<false><<<grid, block, 0, s>>>(x, L, N, words, ld, wpl, nullptr);
    return launch_check("pack_cols_kernel");
}

int launch_unary(int op, const float* x, size_t n, float* out, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    const unsigned g = grid_for(n, 256);
    if (op == 0)
        unary_kernel<0><<<g, 256, 0, s>>>(x, n, out);
    else
        unary_kernel<1><<<g, 256, 0, s>>>(x, n, out);
    return launch_check("unary_kernel");
}

}  // namespace bnnk

using namespace bnnk;

extern "C" {

int bnn_sign_pack_cols_f32(const float* x, size_t L, size_t N, uint32_t* words, size_t ld,
                           bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_pack_cols(x, L, N, words, ld, nullptr, S(s));
}

int bnn_sign_pack_rows_f32(const float* x, size_t D, size_t L, uint32_t* words, size_t ld,
                           bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_pack_rows(x, D, L, words, ld, nullptr, S(s));
}

int bnn_pack_cols_f32(const float* x, size_t L, size_t N, uint32_t* words, size_t ld,
                      int64_t* first_bad, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_pack_cols(x, L, N, words, ld, reinterpret_cast<unsigned long long*>(first_bad),
                            S(s));
}

int bnn_pack_rows_f32(const float* x, size_t D, size_t L, uint32_t* words, size_t ld,
                      int64_t* first_bad, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_pack_rows(x, D, L, words, ld, reinterpret_cast<unsigned long long*>(first_bad),
                            S(s));
}

int bnn_unpack_f32(const uint32_t* words, size_t ld, size_t rows, size_t cols, int orientation,
                   float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    if (rows == 0 || cols == 0) return fail(BNN_E_SHAPE, "unpack: extents must be >= 1");
    unpack_kernel<<<grid_for(rows * cols, 256), 256, 0, S(s)>>>(words, ld, rows, cols,
                                                              orientation ? 1 : 0, out);
    return launch_check("unpack_kernel");
}

int bnn_sign_f32(const float* x, size_t n, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_unary(0, x, n, out, S(s));
}

int bnn_htanh_f32(const float* x, size_t n, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_unary(1, x, n, out, S(s));
}

}  // extern "C"
