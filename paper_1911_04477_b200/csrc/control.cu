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

}  // namespace

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
