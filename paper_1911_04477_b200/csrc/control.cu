// The paper's control group on the GPU: the float path the binary
// kernel is compared against, with no vendor library.
//
//   float_gemm          kernels.cpp:33-51   out[i, j] = sum_k w[i, k] x[k, j], k ascending.
//                       The reference's inner statement orow[j] += a * xrow[j] is compiled
//                       with FMA contraction (-O3 -march=native, SURVEY.md §7 hard part 3), so
//                       every output is the chain acc = fma(w[i, k], x[k, j], acc) from 0.0:
//                       each thread keeps exactly that order (k tiles in ascending order),
//                       which makes the result bit-identical to the reference.
//   conv_forward_float  network.cpp:50-63   float im2col (lowering.cpp:7-43, zero padding),
//                       float_gemm, bias_add (one rounding), reshape_output.
//   linear (Float)      network.cpp:113-120 float_gemm + bias_add.
//
// Kernel: 64 x 64 output tile per 256-thread block, 4 x 4 outputs per thread, k staged
// through shared memory 16 at a time. CUDA-core FP32 (FFMA), as the paper's control group.
#include "bnn_common.cuh"

namespace bnnk {
namespace {

constexpr int kT = 64, kK = 16;

// out[img*M*P + i*P + p] = fma-chain(w[i, :], x[:, j]) + bias[i], j = img*P + p (P = N: [M, N])
__global__ void __launch_bounds__(256) float_gemm_kernel(const float* __restrict__ w, const float* __restrict__ x,
                                                         int M, int N, int K, const float* __restrict__ bias,
                                                         int P, float* __restrict__ out) {
    __shared__ float sw[kK][kT + 1];  // [k][i]
    __shared__ float sx[kK][kT];      // [k][j]
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int i0 = blockIdx.y * kT, j0 = blockIdx.x * kT;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += kK) {
        for (int e = threadIdx.x; e < kK * kT; e += 256) {
            {  // w rows: consecutive threads walk k (64-byte row segments)
                const int c = e / kK, kk = e % kK, i = i0 + c, k = k0 + kk;
                sw[kk][c] = (i < M && k < K) ? w[size_t(i) * K + k] : 0.0f;
            }
            {  // x rows: consecutive threads walk j
                const int kk = e / kT, c = e % kT, j = j0 + c, k = k0 + kk;
                sx[kk][c] = (j < N && k < K) ? x[size_t(k) * N + j] : 0.0f;
            }
        }
        __syncthreads();
        const int kn = min(kK, K - k0);
        for (int kk = 0; kk < kn; ++kk) {  // ascending k: the reference's accumulation order
            float a[4], b[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = sw[kk][ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; ++c) b[c] = sx[kk][tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] = __fmaf_rn(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = i0 + ty * 4 + r;
        if (i >= M) continue;
        const float bi = bias ? bias[i] : 0.0f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int j = j0 + tx * 4 + c;
            if (j >= N) continue;
            const int img = j / P, p = j - img * P;
            out[(size_t(img) * M + i) * P + p] = bias ? __fadd_rn(acc[r][c], bi) : acc[r][c];
        }
    }
}

// im2col for the whole batch (lowering.cpp:7-43): cols[r, n], r = (c*kH + kh)*kW + kw,
// n = b*oh*ow + oy*ow + ox, 0.0 outside the input.
__global__ void im2col_f32_kernel(const float* __restrict__ x, int C, int H, int W, int kH, int kW, int sH, int sW,
                                  int pH, int pW, int oh, int ow, size_t N, int K, float* __restrict__ cols) {
    const size_t total = size_t(K) * N;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
        const int r = int(e / N);
        const size_t n = e - size_t(r) * N;
        const int P = oh * ow;
        const size_t b = n / P;
        const int p = int(n - b * P), oy = p / ow, ox = p - oy * ow;
        const int kk = kH * kW, c = r / kk, t = r - c * kk, kh = t / kW, kw = t - kh * kW;
        const int iy = oy * sH - pH + kh, ix = ox * sW - pW + kw;
        cols[e] = (unsigned(iy) < unsigned(H) && unsigned(ix) < unsigned(W))
                      ? x[((b * C + c) * size_t(H) + iy) * W + ix]
                      : 0.0f;
    }
}

// conv_forward_naive (network.cpp:96-111) with naive_conv (kernels.cpp:109-147): one thread per
// output, acc = fma(w[d, c, kh, kw], x[b, c, ih, iw], acc) over kh, kw, c in the reference's loop
// order with out-of-image taps skipped (the reference's contracted acc += w * x), then + bias
// (the separate slice += bias[d] add).
__global__ void naive_conv_kernel(const float* __restrict__ x, int C, int H, int W, const float* __restrict__ w,
                                  const float* __restrict__ bias, int D, int kH, int kW, int sH, int sW, int pH,
                                  int pW, int oh, int ow, size_t total, float* __restrict__ out) {
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
        const int ox = int(e % ow);
        const size_t t = e / ow;
        const int oy = int(t % oh);
        const size_t t2 = t / oh;
        const int d = int(t2 % D);
        const size_t b = t2 / D;
        const float* xb = x + b * size_t(C) * H * W;
        const float* wd = w + size_t(d) * C * kH * kW;
        float acc = 0.0f;
        for (int kh = 0; kh < kH; ++kh) {
            const int ih = oy * sH + kh - pH;
            if (ih < 0 || ih >= H) continue;
            for (int kw = 0; kw < kW; ++kw) {
                const int iw = ox * sW + kw - pW;
                if (iw < 0 || iw >= W) continue;
                for (int c = 0; c < C; ++c)
                    acc = __fmaf_rn(wd[(size_t(c) * kH + kh) * kW + kw], xb[(size_t(c) * H + ih) * W + iw], acc);
            }
        }
        out[e] = bias ? __fadd_rn(acc, bias[d]) : acc;  // naive_conv alone: no bias
    }
}

// col2im (lowering.cpp:45-84) as a gather: input element (c, ih, iw) sums its contributions
// in the reference's scatter order, rows r = (c*kH + kh)*kW + kw ascending (each row adds at
// most one column to a given element), starting from 0.0 -- the same float additions in the
// same order, so bit-identical.
__global__ void col2im_kernel(const float* __restrict__ m, int C, int in_h, int in_w, int kH, int kW, int sH, int sW,
                              int pH, int pW, int oh, int ow, float* __restrict__ x) {
    const size_t total = size_t(C) * in_h * in_w;
    const size_t cols = size_t(oh) * ow;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
        const int iw = int(e % in_w), ih = int((e / in_w) % in_h), c = int(e / (size_t(in_w) * in_h));
        float acc = 0.0f;
        for (int kh = 0; kh < kH; ++kh) {
            const int th = ih + pH - kh;
            if (th < 0 || th % sH) continue;
            const int y = th / sH;
            if (y >= oh) continue;
            for (int kw = 0; kw < kW; ++kw) {
                const int tw = iw + pW - kw;
                if (tw < 0 || tw % sW) continue;
                const int xo = tw / sW;
                if (xo >= ow) continue;
                const size_t r = (size_t(c) * kH + kh) * kW + kw;
                acc = __fadd_rn(acc, m[r * cols + size_t(y) * ow + xo]);
            }
        }
        x[e] = acc;
    }
}

}  // namespace

int launch_naive_conv(const float* x, size_t B, size_t C, size_t H, size_t W, const float* w, const float* bias,
                      const bnn_conv_geom* g, float* out, cudaStream_t s) {
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    const size_t total = B * g->out_channels * oh * ow;
    if (total == 0) return BNN_OK;
    const unsigned grid = unsigned(std::min<size_t>(ceil_div(total, 256), size_t(num_sms()) * 32));
    naive_conv_kernel<<<grid, 256, 0, s>>>(x, int(C), int(H), int(W), w, bias, int(g->out_channels), int(g->kernel_h),
                                           int(g->kernel_w), int(g->stride_h), int(g->stride_w), int(g->pad_h),
                                           int(g->pad_w), int(oh), int(ow), total, out);
    return launch_check("naive_conv_kernel");
}

int launch_float_gemm(const float* w, const float* x, size_t M, size_t N, size_t K, const float* bias, size_t P,
                      float* out, cudaStream_t s) {
    if (M == 0 || N == 0) return BNN_OK;
    if (P == 0 || N % P) return fail(BNN_E_SHAPE, "float_gemm: N must be a multiple of P");
    if (M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return fail(BNN_E_SHAPE, "float_gemm: extents too large");
    dim3 grid(unsigned(ceil_div(N, kT)), unsigned(ceil_div(M, kT)));
    float_gemm_kernel<<<grid, 256, 0, s>>>(w, x, int(M), int(N), int(K), bias, int(P), out);
    return launch_check("float_gemm_kernel");
}

int launch_im2col_f32(const float* x, size_t B, size_t C, size_t H, size_t W, const bnn_conv_geom* g, float* cols,
                      cudaStream_t s) {
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    const size_t N = B * oh * ow, K = g->kernel_h * g->kernel_w * C;
    if (N * K == 0) return BNN_OK;
    const unsigned grid = unsigned(std::min<size_t>(ceil_div(N * K, 256), size_t(num_sms()) * 32));
    im2col_f32_kernel<<<grid, 256, 0, s>>>(x, int(C), int(H), int(W), int(g->kernel_h), int(g->kernel_w),
                                           int(g->stride_h), int(g->stride_w), int(g->pad_h), int(g->pad_w), int(oh),
                                           int(ow), N, int(K), cols);
    return launch_check("im2col_f32_kernel");
}

}  // namespace bnnk

extern "C" {

// float_gemm (kernels.cpp:33-51) + optional bias / reshape epilogue, device pointers.
int bnn_float_gemm_f32(const float* w, size_t M, size_t K, const float* x, size_t N, const float* bias, size_t P,
                       float* out, bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    return bnnk::launch_float_gemm(w, x, M, N, K, bias, P ? P : N, out, bnnk::S(s));
}

// im2col (lowering.cpp:7-43) of images [b0, b0 + nb) of x [B, C, H, W]: cols [K, nb*oh*ow]
// (nb = 1: the reference's [K, oh*ow] patch matrix of batch slice b0), 0.0 outside the input.
int bnn_im2col_f32(const float* x, size_t B, size_t C, size_t H, size_t W, size_t b0, size_t nb,
                   const bnn_conv_geom* g, float* cols, bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    if (g->in_channels != C)
        return bnnk::fail(BNN_E_SHAPE, "im2col: input has " + std::to_string(C) + " channels, geometry expects " +
                                           std::to_string(g->in_channels));
    if (b0 >= B || nb == 0 || b0 + nb > B)
        return bnnk::fail(BNN_E_SHAPE, "im2col: batch index " + std::to_string(b0) + " out of range " + std::to_string(B));
    return bnnk::launch_im2col_f32(x + b0 * C * H * W, nb, C, H, W, g, cols, bnnk::S(s));
}

// col2im (lowering.cpp:45-84): m [C*kH*kW, oh*ow] -> x [1, C, in_h, in_w].
int bnn_col2im_f32(const float* m, size_t rows, size_t cols, const bnn_conv_geom* g, size_t oh, size_t ow,
                   float* x, size_t* in_h_out, size_t* in_w_out, bnn_stream_t s) {
    const size_t patch = g->kernel_h * g->kernel_w * g->in_channels;
    if (rows != patch)
        return bnnk::fail(BNN_E_SHAPE, "col2im: matrix has " + std::to_string(rows) + " rows, geometry expects " +
                                           std::to_string(patch));
    if (cols != oh * ow)
        return bnnk::fail(BNN_E_SHAPE, "col2im: matrix has " + std::to_string(cols) + " columns, expected " +
                                           std::to_string(oh * ow));
    const size_t span_h = (oh - 1) * g->stride_h + g->kernel_h, span_w = (ow - 1) * g->stride_w + g->kernel_w;
    if (span_h <= 2 * g->pad_h || span_w <= 2 * g->pad_w)
        return bnnk::fail(BNN_E_SHAPE, "col2im: geometry implies an empty input");
    const size_t in_h = span_h - 2 * g->pad_h, in_w = span_w - 2 * g->pad_w;
    if (in_h_out) *in_h_out = in_h;
    if (in_w_out) *in_w_out = in_w;
    if (!x) return BNN_OK;  // extents query
    BNN_TRY(bnnk::require_sm100());
    const size_t total = g->in_channels * in_h * in_w;
    const unsigned grid = unsigned(std::min<size_t>(bnnk::ceil_div(total, 256), size_t(bnnk::num_sms()) * 32));
    bnnk::col2im_kernel<<<grid, 256, 0, bnnk::S(s)>>>(m, int(g->in_channels), int(in_h), int(in_w), int(g->kernel_h),
                                                      int(g->kernel_w), int(g->stride_h), int(g->stride_w),
                                                      int(g->pad_h), int(g->pad_w), int(oh), int(ow), x);
    return bnnk::launch_check("col2im_kernel");
}

// conv_forward_naive (network.cpp:96-111): w [D, C, kH, kW] -> [B, D, oh, ow].
int bnn_conv_forward_naive_f32(const float* x, size_t B, size_t C, size_t H, size_t W, const float* w,
                               const float* bias, const bnn_conv_geom* g, float* out, bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    if (g->in_channels != C) return bnnk::fail(BNN_E_SHAPE, "naive_conv: input channels do not match geometry");
    return bnnk::launch_naive_conv(x, B, C, H, W, w, bias, g, out, bnnk::S(s));
}

// conv_forward_float (network.cpp:50-63): x [B, C, H, W], w_flat [D, C*kH*kW] -> [B, D, oh, ow].
int bnn_conv_forward_float_f32(const float* x, size_t B, size_t C, size_t H, size_t W, const float* w_flat,
                               const float* bias, const bnn_conv_geom* g, float* out, bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    if (g->in_channels != C)
        return bnnk::fail(BNN_E_SHAPE, "im2col: input has " + std::to_string(C) + " channels, geometry expects " +
                                           std::to_string(g->in_channels));
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    const size_t K = g->kernel_h * g->kernel_w * C, N = B * oh * ow;
    bnnk::Scratch cols;
    BNN_TRY(cols.alloc(K * N * sizeof(float), bnnk::S(s)));
    BNN_TRY(bnnk::launch_im2col_f32(x, B, C, H, W, g, cols.as<float>(), bnnk::S(s)));
    return bnnk::launch_float_gemm(w_flat, cols.as<float>(), g->out_channels, N, K, bias, oh * ow, out, bnnk::S(s));
}

}  // extern "C"
