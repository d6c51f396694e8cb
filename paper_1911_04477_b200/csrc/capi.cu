// C-ABI plumbing: error state, device checks, shape helpers, GEMM dispatch, the two layer
// forwards, and the host-buffer (reference-exact) entry points.
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "bnn_common.cuh"

namespace bnnk {

namespace {
thread_local std::string g_err;
thread_local const char* g_last_gemm = "none";
}  // namespace

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

void set_last_gemm(const char* name) { g_last_gemm = name; }

int launch_check(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(BNN_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return BNN_OK;
}

namespace {
constexpr int kMaxDev = 64;
int g_sms[kMaxDev];
int g_arch_ok[kMaxDev];  // 0 unknown, 1 ok, -1 bad
std::mutex g_dev_mu;

int probe(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_arch_ok[dev] == 0) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
        g_sms[dev] = p.multiProcessorCount;
        g_arch_ok[dev] = (p.major == 10 && p.minor == 0) ? 1 : -1;
        if (g_arch_ok[dev] == 1) {
            // Stream-ordered scratch (Scratch: im2col lines, unpacked operands) comes from the
            // device's default memory pool. Its default release threshold (0) hands the memory
            // back at every synchronize, so the next cudaMallocAsync remaps it (~ms). Keep it.
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
    }
    return g_arch_ok[dev];
}
}  // namespace

int require_sm100() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return fail(BNN_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (dev < 0 || dev >= kMaxDev) return fail(BNN_E_CUDA, "device index out of range");
    const int ok = probe(dev);
    if (ok != 1)
        return fail(BNN_E_CUDA, "bnn_b200 kernels are built for sm_100a (B200); device " +
                                    std::to_string(dev) + " is not compute capability 10.0");
    return BNN_OK;
}

int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev || probe(dev) == -1) return 148;
    return g_sms[dev] ? g_sms[dev] : 148;
}

// defined in the kernel translation units
int check_gemm_args(size_t ldw, size_t ldx, size_t M, size_t N, size_t L);
int popc_gemm_s32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t,
                  int32_t*, size_t, cudaStream_t);
int popc_gemm_f32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t,
                  const float*, size_t, float*, cudaStream_t);
int launch_pack_cols(const float*, size_t, size_t, uint32_t*, size_t, unsigned long long*,
                     cudaStream_t);
int launch_pack_rows(const float*, size_t, size_t, uint32_t*, size_t, unsigned long long*,
                     cudaStream_t);
int launch_im2col_sign_pack(const float*, size_t, size_t, size_t, size_t, const bnn_conv_geom*,
                            uint32_t*, size_t, cudaStream_t);
int conv_rowbits_fused(const float*, size_t, size_t, size_t, size_t, const uint32_t*, size_t, const float*,
                       const bnn_conv_geom*, float*, cudaStream_t, int*);

int xnor4_gemm_s32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t, int32_t*, size_t,
                   cudaStream_t);
int xnor4_gemm_f32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t, const float*, size_t,
                   float*, cudaStream_t);
int xnor4t_gemm_s32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t, int32_t*, size_t,
                    cudaStream_t);
int xnor4t_gemm_f32(const uint32_t*, size_t, const uint32_t*, size_t, size_t, size_t, size_t, const float*, size_t,
                    float*, cudaStream_t);

namespace {
int g_policy = BNN_GEMM_AUTO;

// Size rule: both paths are one launch straight from the packed
// bits (gemm4.cu expands the operands to e2m1 in shared memory); the integer-pipe kernel is
// faster only for the smallest products (below ~2^26 bit-MACs, measured in
// profiles/r02_gemm_crossover.jsonl).
bool use_umma(size_t M, size_t N, size_t L) {
    if (g_policy == BNN_GEMM_POPC) return false;
    if (g_policy == BNN_GEMM_UMMA || g_policy == BNN_GEMM_UMMA_TMA) return true;
    return double(M) * double(N) * double(L) >= 67108864.0;
}
// Among the tensor-core kernels: the TMA-fed one (operands expanded once into HBM) for the
// large products, where the in-CTA expansion is the bound (measured crossover in
// profiles/r02_gemm_crossover_t.jsonl).
bool use_tma(size_t M, size_t N, size_t L) {
    if (g_policy == BNN_GEMM_UMMA_TMA) return true;
    if (g_policy != BNN_GEMM_AUTO) return false;
    // M = 128 x 262144 positions: one weight tile, every line expanded once anyway
    return double(M) * double(N) * double(L) >= 4294967296.0 && M >= 512 && N >= 512;
}
}  // namespace

// GEMM dispatch (device pointers). Kept in one place so every caller (C ABI, layer
// forwards, network engine) takes the same kernel for the same shape.
int gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N,
             size_t L, int32_t* out, size_t ldo, cudaStream_t s) {
    BNN_TRY(check_gemm_args(ldw, ldx, M, N, L));
    if (use_umma(M, N, L))
        return use_tma(M, N, L) ? xnor4t_gemm_s32(w, ldw, x, ldx, M, N, L, out, ldo, s)
                                : xnor4_gemm_s32(w, ldw, x, ldx, M, N, L, out, ldo, s);
    return popc_gemm_s32(w, ldw, x, ldx, M, N, L, out, ldo, s);
}

int gemm_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M, size_t N,
             size_t L, const float* bias, size_t P, float* out, cudaStream_t s) {
    BNN_TRY(check_gemm_args(ldw, ldx, M, N, L));
    if (P == 0 || N % P != 0) return fail(BNN_E_SHAPE, "xnor_gemm: N must be a multiple of P");
    if (use_umma(M, N, L))
        return use_tma(M, N, L) ? xnor4t_gemm_f32(w, ldw, x, ldx, M, N, L, bias, P, out, s)
                                : xnor4_gemm_f32(w, ldw, x, ldx, M, N, L, bias, P, out, s);
    return popc_gemm_f32(w, ldw, x, ldx, M, N, L, bias, P, out, s);
}

int gemm_policy() { return g_policy; }

int conv_forward(const float* x, size_t B, size_t C, size_t H, size_t W, const uint32_t* pw,
                 size_t ldw, const float* bias, const bnn_conv_geom* g, float* out, cudaStream_t s) {
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    if (g->in_channels != C)
        return fail(BNN_E_SHAPE, "im2col: input has " + std::to_string(C) +
                                     " channels, geometry expects " + std::to_string(g->in_channels));
    const size_t K = g->kernel_h * g->kernel_w * C, wpl = wpl_of(K);
    const size_t lines = B * oh * ow;
    if (!use_umma(g->out_channels, lines, K)) {
        // small layers: im2col and the xnor-popcount GEMM in one launch (no scratch)
        int handled = 0;
        BNN_TRY(conv_rowbits_fused(x, B, C, H, W, pw, ldw, bias, g, out, s, &handled));
        if (handled) return BNN_OK;
    }
    Scratch col;
    BNN_TRY(col.alloc(lines * wpl * sizeof(uint32_t), s));
    BNN_TRY(launch_im2col_sign_pack(x, B, C, H, W, g, col.as<uint32_t>(), wpl, s));
    return gemm_f32(pw, ldw, col.as<uint32_t>(), wpl, g->out_channels, lines, K, bias, oh * ow, out, s);
}

int linear_forward(const float* x, size_t K, size_t N, const uint32_t* pw, size_t ldw, size_t M,
                   const float* bias, float* out, cudaStream_t s) {
    const size_t wpl = wpl_of(K);
    Scratch px;
    BNN_TRY(px.alloc(N * wpl * sizeof(uint32_t), s));
    BNN_TRY(launch_pack_cols(x, K, N, px.as<uint32_t>(), wpl, nullptr, s));
    return gemm_f32(pw, ldw, px.as<uint32_t>(), wpl, M, N, K, bias, N, out, s);
}

// One non-blocking stream per host thread for the synchronous host-buffer API.
cudaStream_t host_stream() {
    thread_local cudaStream_t st = nullptr;
    if (!st) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    return st;
}

}  // namespace bnnk

using namespace bnnk;

extern "C" {

const char* bnn_last_error(void) { return g_err.c_str(); }
int bnn_version(void) { return 1; }
const char* bnn_last_gemm_kernel(void) { return g_last_gemm; }

int bnn_set_gemm_policy(int policy) {
    if (policy < BNN_GEMM_AUTO || policy > BNN_GEMM_UMMA_TMA) return fail(BNN_E_CONFIG, "bad GEMM policy");
    g_policy = policy;
    return BNN_OK;
}

size_t bnn_words_per_line(size_t extent) { return wpl_of(extent); }

int bnn_output_dims(const bnn_conv_geom* g, size_t in_h, size_t in_w, size_t* out_h, size_t* out_w) {
    const size_t in[2] = {in_h, in_w};
    const size_t k[2] = {g->kernel_h, g->kernel_w}, st[2] = {g->stride_h, g->stride_w},
                 pd[2] = {g->pad_h, g->pad_w};
    const char* axis[2] = {"height", "width"};
    size_t out[2];
    for (int a = 0; a < 2; ++a) {  // tensor.cpp:48-61
        if (st[a] == 0) return fail(BNN_E_SHAPE, std::string("stride along ") + axis[a] + " must be >= 1");
        const size_t padded = in[a] + 2 * pd[a];
        if (padded < k[a])
            return fail(BNN_E_SHAPE, std::string("kernel larger than padded input along ") + axis[a]);
        const size_t span = padded - k[a];
        if (span % st[a] != 0)
            return fail(BNN_E_SHAPE, std::string("output ") + axis[a] + " is not integral: (" +
                                         std::to_string(in[a]) + " + 2*" + std::to_string(pd[a]) +
                                         " - " + std::to_string(k[a]) +
                                         ") not divisible by stride " + std::to_string(st[a]));
        out[a] = span / st[a] + 1;
    }
    *out_h = out[0];
    *out_w = out[1];
    return BNN_OK;
}

int bnn_xnor_gemm_s32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M,
                      size_t N, size_t L, int32_t* out, size_t ldo, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    if (ldo < N) return fail(BNN_E_SHAPE, "xnor_gemm: output leading dimension < N");
    return gemm_s32(w, ldw, x, ldx, M, N, L, out, ldo, S(s));
}

int bnn_xnor_gemm_bias_f32(const uint32_t* w, size_t ldw, const uint32_t* x, size_t ldx, size_t M,
                           size_t N, size_t L, const float* bias, size_t P, float* out,
                           bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return gemm_f32(w, ldw, x, ldx, M, N, L, bias, P, out, S(s));
}

int bnn_conv_forward_binary_f32(const float* x, size_t B, size_t C, size_t H, size_t W,
                                const uint32_t* packed_w, size_t ldw, const float* bias,
                                const bnn_conv_geom* g, float* out, bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return conv_forward(x, B, C, H, W, packed_w, ldw, bias, g, out, S(s));
}

int bnn_linear_forward_packed_f32(const float* x, size_t K, size_t N, const uint32_t* packed_w,
                                  size_t ldw, size_t M, const float* bias, float* out,
                                  bnn_stream_t s) {
    BNN_TRY(require_sm100());
    return linear_forward(x, K, N, packed_w, ldw, M, bias, out, S(s));
}

// ----------------------------------------------------------- host-buffer entry points

int bnn_host_sign_pack(const float* x, size_t rows, size_t cols, int orientation, int apply_sign,
                       uint32_t* words) {
    BNN_TRY(require_sm100());
    if (rows == 0 || cols == 0) return fail(BNN_E_SHAPE, "pack: extents must be >= 1");
    cudaStream_t s = host_stream();
    const size_t extent = orientation == 0 ? cols : rows;
    const size_t lines = orientation == 0 ? rows : cols;
    const size_t wpl = wpl_of(extent);
    Scratch dx, dw, bad;
    BNN_TRY(dx.alloc(rows * cols * sizeof(float), s));
    BNN_TRY(dw.alloc(lines * wpl * sizeof(uint32_t), s));
    BNN_CUDA(cudaMemcpyAsync(dx.p, x, rows * cols * sizeof(float), cudaMemcpyHostToDevice, s));
    unsigned long long* badp = nullptr;
    if (!apply_sign) {
        BNN_TRY(bad.alloc(sizeof(unsigned long long), s));
        BNN_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
        badp = bad.as<unsigned long long>();
    }
    if (orientation == 0)
        BNN_TRY(launch_pack_rows(dx.as<float>(), rows, cols, dw.as<uint32_t>(), wpl, badp, s));
    else
        BNN_TRY(launch_pack_cols(dx.as<float>(), rows, cols, dw.as<uint32_t>(), wpl, badp, s));
    BNN_CUDA(cudaMemcpyAsync(words, dw.p, lines * wpl * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    unsigned long long first_bad = ~0ull;
    if (badp)
        BNN_CUDA(cudaMemcpyAsync(&first_bad, badp, sizeof first_bad, cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    if (first_bad != ~0ull) {  // binarize.cpp:12-15
        const size_t r = first_bad / cols, c = first_bad % cols;
        char buf[128];
        std::snprintf(buf, sizeof buf, "pack: entry at (%zu,%zu) is %f, expected -1 or +1", r, c,
                      double(x[first_bad]));
        return fail(BNN_E_ENCODING, buf);
    }
    return BNN_OK;
}

int bnn_host_xnor_gemm(const uint32_t* w, size_t M, const uint32_t* x, size_t N, size_t L,
                       int32_t* out) {
    BNN_TRY(require_sm100());
    BNN_TRY(check_gemm_args(wpl_of(L), wpl_of(L), M, N, L));
    cudaStream_t s = host_stream();
    const size_t wpl = wpl_of(L);
    Scratch dw, dx, dout;
    BNN_TRY(dw.alloc(M * wpl * 4, s));
    BNN_TRY(dx.alloc(N * wpl * 4, s));
    BNN_TRY(dout.alloc(M * N * 4, s));
    BNN_CUDA(cudaMemcpyAsync(dw.p, w, M * wpl * 4, cudaMemcpyHostToDevice, s));
    BNN_CUDA(cudaMemcpyAsync(dx.p, x, N * wpl * 4, cudaMemcpyHostToDevice, s));
    BNN_TRY(gemm_s32(dw.as<uint32_t>(), wpl, dx.as<uint32_t>(), wpl, M, N, L, dout.as<int32_t>(), N, s));
    BNN_CUDA(cudaMemcpyAsync(out, dout.p, M * N * 4, cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    return BNN_OK;
}

int bnn_host_conv_forward_binary(const float* x, size_t B, size_t C, size_t H, size_t W,
                                 const uint32_t* packed_w, const float* bias,
                                 const bnn_conv_geom* g, float* out) {
    BNN_TRY(require_sm100());
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    cudaStream_t s = host_stream();
    const size_t D = g->out_channels, K = g->kernel_h * g->kernel_w * g->in_channels;
    const size_t wpl = wpl_of(K);
    const size_t nx = B * C * H * W, ny = B * D * oh * ow;
    Scratch dx, dw, db, dy;
    BNN_TRY(dx.alloc(nx * 4, s));
    BNN_TRY(dw.alloc(D * wpl * 4, s));
    BNN_TRY(db.alloc(D * 4, s));
    BNN_TRY(dy.alloc(ny * 4, s));
    BNN_CUDA(cudaMemcpyAsync(dx.p, x, nx * 4, cudaMemcpyHostToDevice, s));
    BNN_CUDA(cudaMemcpyAsync(dw.p, packed_w, D * wpl * 4, cudaMemcpyHostToDevice, s));
    BNN_CUDA(cudaMemcpyAsync(db.p, bias, D * 4, cudaMemcpyHostToDevice, s));
    BNN_TRY(conv_forward(dx.as<float>(), B, C, H, W, dw.as<uint32_t>(), wpl, db.as<float>(), g,
                         dy.as<float>(), s));
    BNN_CUDA(cudaMemcpyAsync(out, dy.p, ny * 4, cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    return BNN_OK;
}

int bnn_host_linear_forward_packed(const float* x, size_t K, size_t N, const uint32_t* packed_w,
                                   size_t M, const float* bias, float* out) {
    BNN_TRY(require_sm100());
    if (K == 0 || N == 0 || M == 0) return fail(BNN_E_SHAPE, "linear: extents must be >= 1");
    cudaStream_t s = host_stream();
    const size_t wpl = wpl_of(K);
    Scratch dx, dw, db, dy;
    BNN_TRY(dx.alloc(K * N * 4, s));
    BNN_TRY(dw.alloc(M * wpl * 4, s));
    BNN_TRY(db.alloc(M * 4, s));
    BNN_TRY(dy.alloc(M * N * 4, s));
    BNN_CUDA(cudaMemcpyAsync(dx.p, x, K * N * 4, cudaMemcpyHostToDevice, s));
    BNN_CUDA(cudaMemcpyAsync(dw.p, packed_w, M * wpl * 4, cudaMemcpyHostToDevice, s));
    BNN_CUDA(cudaMemcpyAsync(db.p, bias, M * 4, cudaMemcpyHostToDevice, s));
    BNN_TRY(linear_forward(dx.as<float>(), K, N, dw.as<uint32_t>(), wpl, M, db.as<float>(),
                           dy.as<float>(), s));
    BNN_CUDA(cudaMemcpyAsync(out, dy.p, M * N * 4, cudaMemcpyDeviceToHost, s));
    BNN_CUDA(cudaStreamSynchronize(s));
    return BNN_OK;
}

}  // extern "C"
