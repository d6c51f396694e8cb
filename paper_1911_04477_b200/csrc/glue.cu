// K4/K5 — glue operators between binary layers and the device RNG.
//
// maxpool2 (network.cpp:133-149), affine_norm (network.cpp:151-175), flatten_to_columns
// (network.cpp:177-184) and fill_random (tensor.cpp:65-96). These run only on the
// unfused (general-topology) path of the network engine and behind the C ABI; the fused
// VGG path folds them into the GEMM epilogue.
//
// affine_norm: the reference is compiled with -march=native, where GCC contracts
// `s * p[i] + t` into one FMA (survey probe: 10 vfmadd in bnn::affine_norm). The device
// uses __fmaf_rn(s, x, t) so every sign decision downstream matches bit for bit.
#include <vector>

#include "bnn_common.cuh"

namespace bnnk {
namespace {

unsigned grid_for(size_t n, unsigned block) {
    size_t g = ceil_div(n, block);
    const size_t cap = size_t(num_sms()) * 16;
    return unsigned(g < cap ? (g ? g : 1) : cap);
}

__device__ __forceinline__ float max_ref(float a, float b) { return a < b ? b : a; }  // std::max

__global__ void maxpool2_kernel(const float* __restrict__ x, size_t planes, int H, int W,
                                float* __restrict__ out) {
    const int oh = H / 2, ow = W / 2;
    const size_t n = planes * oh * ow;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t p = i / (size_t(oh) * ow);
        const int r = int(i % (size_t(oh) * ow));
        const int y = r / ow, xx = r % ow;
        const float* s = x + p * size_t(H) * W;
        const float a = s[(2 * y) * W + 2 * xx], b = s[(2 * y) * W + 2 * xx + 1];
        const float c = s[(2 * y + 1) * W + 2 * xx], d = s[(2 * y + 1) * W + 2 * xx + 1];
        out[i] = max_ref(max_ref(a, b), max_ref(c, d));
    }
}

__global__ void affine_kernel(const float* __restrict__ x, size_t n, size_t channels,
                              size_t plane, const float* __restrict__ scale,
                              const float* __restrict__ shift, float* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t c = (i / plane) % channels;
        out[i] = __fmaf_rn(scale[c], x[i], shift[c]);
    }
}

// to_float (kernels.cpp:90-95): exact int32 -> float conversion (round to nearest).
__global__ void to_float_kernel(const int32_t* __restrict__ a, size_t n, float* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = __int2float_rn(a[i]);
}

// bias_add (kernels.cpp:97-107): a[d, j] += bias[d], one rounding per element.
__global__ void bias_add_kernel(float* __restrict__ a, size_t rows, size_t cols, const float* __restrict__ bias) {
    const size_t n = rows * cols;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        a[i] = __fadd_rn(a[i], bias[i / cols]);
}

__global__ void transpose_kernel(const float* __restrict__ x, size_t rows, size_t cols,
                                 float* __restrict__ out) {
    __shared__ float tile[32][33];
    const size_t c0 = size_t(blockIdx.x) * 32, r0 = size_t(blockIdx.y) * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const size_t r = r0 + k, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[k][threadIdx.x] = x[r * cols + c];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const size_t c = c0 + k, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][k];
    }
}

__global__ void fill_random_kernel(uint64_t seed, uint64_t offset, size_t n, float* __restrict__ out) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = unit_random(seed, offset + i);
}

// scale = 1 + 0.5 * u (network.cpp:285); 0.5*u is exact, so contraction cannot differ
__global__ void affine_scale_kernel(float* __restrict__ v, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        v[i] = 1.0f + 0.5f * v[i];
}

}  // namespace

int launch_maxpool2(const float* x, size_t B, size_t C, size_t H, size_t W, float* out,
                    cudaStream_t s) {
    if (H % 2 || W % 2)
        return fail(BNN_E_SHAPE, "maxpool2: spatial extents must be even, got " + std::to_string(H) +
                                     "x" + std::to_string(W));
    const size_t n = B * C * (H / 2) * (W / 2);
    if (n == 0) return BNN_OK;
    maxpool2_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, B * C, int(H), int(W), out);
    return launch_check("maxpool2_kernel");
}

int launch_affine(const float* x, size_t n, size_t channels, size_t plane, const float* scale,
                  const float* shift, float* out, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    affine_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, n, channels, plane, scale, shift, out);
    return launch_check("affine_kernel");
}

int launch_transpose(const float* x, size_t rows, size_t cols, float* out, cudaStream_t s) {
    if (rows == 0 || cols == 0) return BNN_OK;
    dim3 grid(unsigned(ceil_div(cols, 32)), unsigned(ceil_div(rows, 32)));
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(x, rows, cols, out);
    return launch_check("transpose_kernel");
}

int launch_fill_random(uint64_t seed, uint64_t offset, size_t n, float* out, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    fill_random_kernel<<<grid_for(n, 256), 256, 0, s>>>(seed, offset, n, out);
    return launch_check("fill_random_kernel");
}

int launch_affine_scale(float* v, size_t n, cudaStream_t s) {
    if (n == 0) return BNN_OK;
    affine_scale_kernel<<<grid_for(n, 256), 256, 0, s>>>(v, n);
    return launch_check("affine_scale_kernel");
}

// max |a[i] - b[i]| (verify_network's deviation, bench.cpp:178-181): each thread folds its
// elements, the warp reduces, one atomicMax per warp on the float's bits (non-negative floats
// order like their unsigned bit patterns). NaN deviations map to +inf.
__global__ void max_abs_diff_kernel(const float* __restrict__ a, const float* __restrict__ b, size_t n,
                                    unsigned* __restrict__ out) {
    float m = 0.0f;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float d = fabsf(a[i] - b[i]);
        m = d != d ? __int_as_float(0x7f800000) : fmaxf(m, d);
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

}  // namespace bnnk

using namespace bnnk;

extern "C" {

int bnn_maxpool2_f32(const float* x, size_t B, size_t C, size_t H, size_t W, float* out,
                     bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_maxpool2(x, B, C, H, W, out, S(s));
}

int bnn_affine_f32(const float* x, size_t n, size_t channels, size_t plane, const float* scale,
                   const float* shift, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    if (channels == 0 || plane == 0) return fail(BNN_E_SHAPE, "affine_norm: empty parameters");
    return launch_affine(x, n, channels, plane, scale, shift, out, S(s));
}

int bnn_to_float_s32(const int32_t* a, size_t n, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    if (n == 0) return BNN_OK;
    to_float_kernel<<<grid_for(n, 256), 256, 0, S(s)>>>(a, n, out);
    return launch_check("to_float_kernel");
}

int bnn_bias_add_f32(float* a, size_t rows, size_t cols, const float* bias, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    if (rows * cols == 0) return BNN_OK;
    bias_add_kernel<<<grid_for(rows * cols, 256), 256, 0, S(s)>>>(a, rows, cols, bias);
    return launch_check("bias_add_kernel");
}

int bnn_flatten_to_columns_f32(const float* x, size_t B, size_t F, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_transpose(x, B, F, out, S(s));
}

int bnn_fill_random_f32(uint64_t seed, uint64_t offset, size_t n, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return launch_fill_random(seed, offset, n, out, S(s));
}

uint64_t bnn_mix64(uint64_t seed, uint64_t counter) { return mix64(seed, counter); }

int bnn_max_abs_diff_f32(const float* a, const float* b, size_t n, double* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    Scratch m;
    BNN_TRY(m.alloc(sizeof(unsigned), S(s)));
    BNN_CUDA(cudaMemsetAsync(m.p, 0, sizeof(unsigned), S(s)));
    if (n) {
        max_abs_diff_kernel<<<grid_for(n, 256), 256, 0, S(s)>>>(a, b, n, m.as<unsigned>());
        BNN_TRY(launch_check("max_abs_diff_kernel"));
    }
    unsigned h = 0;
    BNN_CUDA(cudaMemcpyAsync(&h, m.p, sizeof h, cudaMemcpyDeviceToHost, S(s)));
    BNN_CUDA(cudaStreamSynchronize(S(s)));
    float f;
    memcpy(&f, &h, 4);
    *out = double(f);
    return BNN_OK;
}

int bnn_fnv1a_f32(const float* x, size_t n, uint64_t* hash, bnn_stream_t s) {
    std::vector<float> h(n);
    BNN_CUDA(cudaMemcpyAsync(h.data(), x, n * sizeof(float), cudaMemcpyDeviceToHost, S(s)));
    BNN_CUDA(cudaStreamSynchronize(S(s)));
    uint64_t v = 1469598103934665603ull;  // bench.cpp:23-33
    for (float f : h) {
        uint32_t bits;
        memcpy(&bits, &f, 4);
        for (int i = 0; i < 4; ++i) {
            v ^= (bits >> (8 * i)) & 0xFF;
            v *= 1099511628211ull;
        }
    }
    *hash = v;
    return BNN_OK;
}

}  // extern "C"
