// K2 — binary im2col: the lowered patch matrix is produced already sign-binarized and
// packed along K, for the whole batch in one launch.
//
// Replaces pack_cols(sign(im2col(x, b, g))) of conv_forward_binary (network.cpp:71-72,
// lowering.cpp:7-43, binarize.cpp:55-73). The float patch matrix of the reference
// ([K, oh*ow] per image, 4 bytes per bit) is never materialised.
//
// Line n = b*oh*ow + oy*ow + ox (one output position), bit r = (c*kH + kh)*kW + kw
// (the c-major patch order, lowering.hpp:8-10). Input outside the image reads as 0.0,
// and sign(0.0) = +1, so spatial padding is bit 1 (README.md:150-153). Bits past K are 0.
//
// Two kernels: im2col_rowbits_kernel (W <= 32) sign-packs each input row once and builds
// every output word from kW-bit fields of those row words; im2col_sign_pack_kernel is the
// general one (a load and compare per bit).
#include "bnn_common.cuh"

namespace bnnk {
namespace {

constexpr int kWordsPerBlock = 8;

// General fallback (any W): thread (tx, ty) owns output position j0+tx and word k0+ty; for a
// fixed patch row r the 32 lanes read 32 consecutive output positions -> consecutive input
// columns, a coalesced load. The [32 line x 8 word] tile goes through shared memory so the
// stores are line-contiguous.
__global__ void __launch_bounds__(256)
    im2col_sign_pack_kernel(const float* __restrict__ x, int C, int H, int W, int kH, int kW,
                            int sH, int sW, int pH, int pW, int oh, int ow, size_t lines,
                            int K, int wpl, uint32_t* __restrict__ words, size_t ld) {
    __shared__ uint32_t tile[32][kWordsPerBlock + 1];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const size_t j0 = size_t(blockIdx.x) * 32;
    const int k0 = blockIdx.y * kWordsPerBlock;
    const size_t n = j0 + tx;
    const int word = k0 + ty;
    uint32_t w = 0;
    if (n < lines && word < wpl) {
        const int P = oh * ow;
        const size_t img = n / P;
        const int p = int(n % P);
        const int oy = p / ow, ox = p % ow;
        const int iy0 = oy * sH - pH, ix0 = ox * sW - pW;
        const float* xb = x + img * size_t(C) * H * W;
        int r = word * 32;
        const int kk = kH * kW;
        int c = r / kk, rem = r % kk;
        int kh = rem / kW, kw = rem % kW;
#pragma unroll 4
        for (int b = 0; b < 32; ++b, ++r) {
            if (r >= K) break;
            const int iy = iy0 + kh, ix = ix0 + kw;
            float v = 0.0f;  // outside the input: im2col writes 0.0 (lowering.cpp:32-36)
            if (iy >= 0 && iy < H && ix >= 0 && ix < W) v = __ldg(xb + (size_t(c) * H + iy) * W + ix);
            w |= uint32_t(v >= 0.0f) << b;
            if (++kw == kW) {
                kw = 0;
                if (++kh == kH) {
                    kh = 0;
                    ++c;
                }
            }
        }
    }
    tile[tx][ty] = w;
    __syncthreads();
    const int t = ty * 32 + tx;
    const int line = t / kWordsPerBlock, kq = t % kWordsPerBlock;
    if (j0 + line < lines && k0 + kq < wpl) words[(j0 + line) * ld + k0 + kq] = tile[line][kq];
}

// Row-bits kernel (W <= 32, the CIFAR-class shapes): one block per (image, output row).
//  1. Sign-pack every input row the block needs — rows iy = oy*sH - pH + kh of all C
//     channels — into one word each (warp load of the row + __ballot_sync), in smem.
//  2. Warp w builds output word q (w, w+8, ...) for all ow positions of the row at once:
//     lane b owns patch row r = 32q + b = (c*kH + kh)*kW + kw, i.e. input row (c, kh) and
//     tap kw; for position ox its bit is bit ox*sW - pW + kw of that row word (padding
//     columns are 1 bits of a 64-bit window), and one __ballot_sync over the lanes yields
//     the whole word for that position (the lane = r bit order is the word's bit order).
//     With stride 1 the 32 ballots are one 32 x 32 bit transpose across the warp (five
//     shuffle-xor butterfly rounds), about one instruction per output word.
//  3. The block's [ow lines x wpl words] output is staged in smem and stored line-contiguous.
__global__ void __launch_bounds__(256)
    im2col_rowbits_kernel(const float* __restrict__ x, int C, int H, int W, int kH, int kW, int sH, int sW,
                          int pH, int pW, int oh, int ow, int K, int wpl, uint32_t* __restrict__ words,
                          size_t ld) {
    extern __shared__ uint32_t sm[];
    const int nrows = C * kH;
    uint32_t* rows = sm;                // [C * kH] row words
    uint32_t* tile = rows + nrows;      // [ow][wpl]
    const int oy = blockIdx.x, img = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    // 1. input rows -> sign words (bit ix = x[img, c, iy, ix] >= 0; columns >= W are 1 = padding).
    // Warp w takes channels [4w, 4w + 4), [4w + 32, ...): kH rows each.
    const float* xb = x + size_t(img) * C * H * W + (lane < W ? lane : 0);
    const int iy0 = oy * sH - pH;
    constexpr int kU = 4;  // measured: 4 beats 16 (0.164 vs 0.207 ms at [256,128,32,32])
    for (int c0 = warp * kU; c0 < C; c0 += nwarps * kU) {
        for (int kh = 0; kh < kH; ++kh) {
            const int iy = iy0 + kh;
            const bool rin = unsigned(iy) < unsigned(H);
            float v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u)
                v[u] = rin && c0 + u < C && lane < W ? __ldg(xb + (size_t(c0 + u) * H + iy) * W) : 0.0f;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                // a padding row (iy outside): every tap reads 0.0 -> +1
                const uint32_t bits = __ballot_sync(0xffffffffu, v[u] >= 0.0f);
                if (lane == 0 && c0 + u < C) rows[(c0 + u) * kH + kh] = bits;
            }
        }
    }
    __syncthreads();
    // 2. word q of every position: lane = patch row r
    const int kk = kH * kW;
    const uint64_t pad = ~(((1ull << W) - 1ull) << 16);  // row at bits [16, 16 + W), the rest 1
    for (int q = warp; q < wpl; q += nwarps) {
        const int r = q * 32 + lane;
        const bool rv = r < K;  // bits past K are 0
        const int c = r / kk, t = r - c * kk, kh = t / kW, kw = t - kh * kW;
        const uint64_t win = rv ? ((uint64_t(rows[c * kH + kh]) << 16) | pad) : 0ull;
        const int sh0 = 16 - pW + kw;  // window bit of position ox: sh0 + ox * sW
        for (int ox0 = 0; ox0 < ow; ox0 += 32) {
            uint32_t mine = 0;
            if (sW == 1) {
                // lane r holds its bits for 32 consecutive positions; a 32 x 32 bit transpose
                // across the warp (5 shuffle-xor butterfly rounds) gives lane ox its word
                uint32_t v = uint32_t(win >> (sh0 + ox0));
#pragma unroll
                for (int j = 16; j >= 1; j >>= 1) {
                    const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                                     : j == 2 ? 0x33333333u : 0x55555555u;
                    const uint32_t p = __shfl_xor_sync(0xffffffffu, v, j);
                    v = (lane & j) ? ((v & ~m) | ((p >> j) & m)) : ((v & m) | ((p & m) << j));
                }
                mine = v;
            } else {
#pragma unroll 8
                for (int j = 0; j < 32; ++j) {
                    const int ox = ox0 + j;
                    const uint32_t wbits = __ballot_sync(0xffffffffu, (win >> (sh0 + ox * sW)) & 1ull);
                    if (lane == j) mine = wbits;
                }
            }
            if (ox0 + lane < ow) tile[(ox0 + lane) * wpl + q] = mine;
        }
    }
    __syncthreads();
    // 3. store the [ow x wpl] tile: lines img*oh*ow + oy*ow + ox
    const int total = ow * wpl;
    uint32_t* dst = words + (size_t(img) * oh * ow + size_t(oy) * ow) * ld;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int ox = t / wpl, q = t - ox * wpl;
        dst[size_t(ox) * ld + q] = tile[t];
    }
}

}  // namespace

int launch_im2col_sign_pack(const float* x, size_t B, size_t C, size_t H, size_t W,
                            const bnn_conv_geom* g, uint32_t* words, size_t ld, cudaStream_t s) {
    if (g->in_channels != C)
        return fail(BNN_E_SHAPE, "im2col: input has " + std::to_string(C) +
                                     " channels, geometry expects " + std::to_string(g->in_channels));
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    const size_t K = g->kernel_h * g->kernel_w * C;
    const size_t wpl = wpl_of(K);
    if (ld < wpl) return fail(BNN_E_SHAPE, "im2col: leading dimension smaller than ceil(K/32)");
    const size_t lines = B * oh * ow;
    if (lines == 0) return BNN_OK;
    const size_t kW = g->kernel_w, pW = g->pad_w;
    const size_t smem = (C * g->kernel_h + ow * wpl) * sizeof(uint32_t);
    // row-bits kernel: rows fit one word, padding windows stay inside the 64-bit shift (input
    // column of a tap in [-16, 48)), and enough (image, row) blocks to fill the GPU (a batch-1
    // layer takes the general kernel)
    if (W <= 32 && pW <= 16 && smem <= 48 * 1024 && oh < 65536 && B < 65536 &&
        (ow - 1) * g->stride_w + kW <= 48 + pW && B * oh >= size_t(num_sms())) {
        im2col_rowbits_kernel<<<dim3(unsigned(oh), unsigned(B)), 256, smem, s>>>(
            x, int(C), int(H), int(W), int(g->kernel_h), int(kW), int(g->stride_h), int(g->stride_w),
            int(g->pad_h), int(pW), int(oh), int(ow), int(K), int(wpl), words, ld);
        return launch_check("im2col_rowbits_kernel");
    }
    dim3 grid(unsigned(ceil_div(lines, 32)), unsigned(ceil_div(wpl, kWordsPerBlock)));
    im2col_sign_pack_kernel<<<grid, dim3(32, kWordsPerBlock), 0, s>>>(
        x, int(C), int(H), int(W), int(g->kernel_h), int(g->kernel_w), int(g->stride_h),
        int(g->stride_w), int(g->pad_h), int(g->pad_w), int(oh), int(ow), lines, int(K), int(wpl),
        words, ld);
    return launch_check("im2col_sign_pack_kernel");
}

}  // namespace bnnk

extern "C" int bnn_im2col_sign_pack_f32(const float* x, size_t B, size_t C, size_t H, size_t W,
                                        const bnn_conv_geom* g, uint32_t* words, size_t ld,
                                        bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    return bnnk::launch_im2col_sign_pack(x, B, C, H, W, g, words, ld, bnnk::S(s));
}
