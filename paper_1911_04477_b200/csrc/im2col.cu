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
// Thread (tx, ty) of a block owns output position j0+tx and word k0+ty: for a fixed patch
// row r, the 32 lanes read 32 consecutive output positions -> consecutive input columns
// (stride 1), a coalesced load. The [32 line x 8 word] tile goes through shared memory so
// the stores are line-contiguous.
#include "bnn_common.cuh"

namespace bnnk {
namespace {

constexpr int kWordsPerBlock = 8;

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
