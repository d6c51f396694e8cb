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
#include <algorithm>
#include <cstdlib>

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

// Phase 2 of the row-bits im2col (shared by the per-group and the pipelined kernels): from the
// group's sign-packed input rows `rows` [C][nrow], word q of every output position of its ry
// rows into `tile` [ry * ow][wpl]; lane = patch row r = 32 q + lane.
__device__ __forceinline__ void rowbits_words(const uint32_t* __restrict__ rows, uint32_t* __restrict__ tile, int W,
                                              int kH, int kW, int sH, int sW, int pW, int ow, int K, int wpl, int ry,
                                              int nrow, int warp, int nwarps, int lane) {
    // 2. word q of every position of every row of the group: lane = patch row r
    const int kk = kH * kW;
    const uint64_t pad = ~(((1ull << W) - 1ull) << 16);  // row at bits [16, 16 + W), the rest 1
    // per-lane transpose constants (see transpose32 in umma.cuh): round j keeps the half of the
    // word selected by k_j (~k_j in lanes with bit j set) and rotates the partner's word by j
    uint32_t keep[5];
    int rot[5];
#pragma unroll
    for (int jj = 0; jj < 5; ++jj) {
        const int j = 16 >> jj;
        const uint32_t k = jj == 0 ? 0x0000FFFFu : jj == 1 ? 0x00FF00FFu : jj == 2 ? 0x0F0F0F0Fu : jj == 3 ? 0x33333333u
                                                                                                     : 0x55555555u;
        const bool up = (lane & j) != 0;
        keep[jj] = up ? ~k : k;
        rot[jj] = up ? 32 - j : j;
    }
    // word q outer (the lane's patch row decode once), the group's rows inner
    for (int q = warp; q < wpl; q += nwarps) {
        const int r = q * 32 + lane;
        const bool rv = r < K;  // bits past K are 0
        const int c = r / kk, t = r - c * kk, kh = t / kW, kw = t - kh * kW;
        const int sh0 = 16 - pW + kw;  // window bit of position ox: sh0 + ox * sW
        const uint32_t* rowp = rows + c * nrow + kh;
        for (int yy = 0; yy < ry; ++yy) {
            const uint64_t win = rv ? ((uint64_t(rowp[yy * sH]) << 16) | pad) : 0ull;
            for (int ox0 = 0; ox0 < ow; ox0 += 32) {
                uint32_t mine = 0;
                if (sW == 1) {
                    // lane r holds its bits for 32 consecutive positions; a 32 x 32 bit transpose
                    // across the warp gives lane ox its word: per round a shuffle, a funnel-shift
                    // rotate and one LOP3 with the lane's loop-invariant keep mask and rotation
                    uint32_t v = uint32_t(win >> (sh0 + ox0));
#pragma unroll
                    for (int jj = 0; jj < 5; ++jj) {
                        const int j = 16 >> jj;
                        const uint32_t p = __shfl_xor_sync(0xffffffffu, v, j);
                        const uint32_t qv = __funnelshift_l(p, p, rot[jj]);
                        v = (v & keep[jj]) | (qv & ~keep[jj]);
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
                if (ox0 + lane < ow) tile[(yy * ow + ox0 + lane) * wpl + q] = mine;
            }
        }
    }
}

// Row-bits kernel (W <= 32, the CIFAR-class shapes): one block per (image, group of R output
// rows).
//  1. Sign-pack every input row the group needs — rows (oy0*sH - pH) .. of all C channels, each
//     read ONCE per group (R rows share their kH - sH halo rows) — into one word each, in smem.
//     W % 4 == 0: float4 loads, 8 lanes per input row (4 rows per warp instruction), the row
//     word assembled with 3 shuffle-xor ORs; otherwise a warp-wide load and a ballot per row.
//  2. Warp w builds output word q (w, w+8, ...) for all ow positions of each row of the group:
//     lane b owns patch row r = 32q + b = (c*kH + kh)*kW + kw, i.e. input row (c, kh) and tap
//     kw; for position ox its bit is bit ox*sW - pW + kw of that row word (padding columns are
//     1 bits of a 64-bit window). With stride 1 the 32 positions' words are one 32 x 32 bit
//     transpose across the warp (five shuffle-xor butterfly rounds), else one ballot each.
//  3. The group's [R*ow lines x wpl words] output is staged in smem and stored line-contiguous.
__global__ void __launch_bounds__(256, 5)
    im2col_rowbits_kernel(const float* __restrict__ x, int C, int H, int W, int kH, int kW, int sH, int sW,
                          int pH, int pW, int oh, int ow, int K, int wpl, int R, uint32_t* __restrict__ words,
                          size_t ld, const uint32_t* __restrict__ cw, size_t ldw, int D, const float* __restrict__ bias,
                          float* __restrict__ y) {
    extern __shared__ uint32_t sm[];
    const int oy0 = blockIdx.x * R, img = blockIdx.y;
    const int ry = min(R, oh - oy0);                  // output rows of this group
    const int nrow = (ry - 1) * sH + kH;              // input rows per channel
    uint32_t* rows = sm;                              // [C][nrow] row words
    uint32_t* tile = rows + C * nrow;                 // [ry * ow][wpl]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int iyb = oy0 * sH - pH;                    // input row of local row 0
    const float* xb = x + size_t(img) * C * H * W;
    // 1. input rows -> sign words (bit ix = x[img, c, iy, ix] >= 0; an out-of-image row reads
    // 0.0 everywhere -> all +1; bits >= W are don't-care: the window below masks them to 1)
    const int total = C * nrow;
    if ((W & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        // kU float4 loads in flight per lane (kU * 4 rows per warp per round): one memory round
        // trip per round instead of one per 4 rows
        constexpr int kU = 4;
        const int sub = lane >> 3, col = 4 * (lane & 7);
        for (int t0 = warp * 4 * kU; t0 < total; t0 += nwarps * 4 * kU) {
            float4 v[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int t = t0 + 4 * u + sub;
                const int c = t / nrow, lr = t - c * nrow, iy = iyb + lr;
                v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (t < total && unsigned(iy) < unsigned(H) && col < W)
                    v[u] = __ldg(reinterpret_cast<const float4*>(xb + (size_t(c) * H + iy) * W + col));
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int t = t0 + 4 * u + sub;
                uint32_t b = (uint32_t(v[u].x >= 0.0f) | (uint32_t(v[u].y >= 0.0f) << 1) |
                              (uint32_t(v[u].z >= 0.0f) << 2) | (uint32_t(v[u].w >= 0.0f) << 3))
                             << col;
                b |= __shfl_xor_sync(0xffffffffu, b, 1);
                b |= __shfl_xor_sync(0xffffffffu, b, 2);
                b |= __shfl_xor_sync(0xffffffffu, b, 4);
                if ((lane & 7) == 0 && t < total) rows[t] = b;
            }
        }
    } else {
        for (int t = warp; t < total; t += nwarps) {
            const int c = t / nrow, lr = t - c * nrow, iy = iyb + lr;
            const float v = unsigned(iy) < unsigned(H) && lane < W ? __ldg(xb + (size_t(c) * H + iy) * W + lane) : 0.0f;
            const uint32_t bits = __ballot_sync(0xffffffffu, v >= 0.0f);
            if (lane == 0) rows[t] = bits;
        }
    }
    __syncthreads();
    rowbits_words(rows, tile, W, kH, kW, sH, sW, pW, ow, K, wpl, ry, nrow, warp, nwarps, lane);
    __syncthreads();
    if (y) {
        // Fused conv_forward_binary (network.cpp:65-79) for small layers: the xnor-popcount GEMM
        // of the group's patch words against the D packed weight rows (CUDA cores), then
        // to_float + bias_add (kernels.cpp:90-107) into the NCHW output (reshape_output,
        // lowering.cpp:87-95). a = L - 2 * sum popc(w ^ x) (pad bits are 0 in both operands).
        // blockIdx.z: this block's slice of output channels [d0, d0 + nd) (more blocks in flight
        // for batch-1 layers; the patch words are rebuilt per slice, from L2)
        const int dch = (D + gridDim.z - 1) / gridDim.z;
        const int d0 = blockIdx.z * dch, nd = min(D, d0 + dch) - d0;
        uint32_t* wsm = tile + ry * ow * wpl;  // [nd][wpl]
        for (int t = threadIdx.x; t < nd * wpl; t += blockDim.x) {
            const int d = t / wpl, q = t - d * wpl;
            wsm[t] = __ldg(cw + size_t(d0 + d) * ldw + q);
        }
        __syncthreads();
        const int nl = ry * ow;
        for (int t = threadIdx.x; t < nd * nl; t += blockDim.x) {
            const int dl = t / nl, l = t - dl * nl, d = d0 + dl;
            const uint32_t* xr = tile + l * wpl;
            const uint32_t* wr = wsm + dl * wpl;
            int pc = 0;
            for (int q = 0; q < wpl; ++q) pc += __popc(xr[q] ^ wr[q]);
            y[(size_t(img) * D + d) * oh * ow + size_t(oy0) * ow + l] =
                __fadd_rn(__int2float_rn(K - 2 * pc), bias ? __ldg(bias + d) : 0.0f);
        }
        return;
    }
    // 3. store the [ry*ow x wpl] tile: lines img*oh*ow + oy0*ow + (yy*ow + ox)
    const int tot = ry * ow * wpl;
    uint32_t* dst = words + (size_t(img) * oh * ow + size_t(oy0) * ow) * ld;
    if (ld == size_t(wpl)) {
        for (int t = threadIdx.x; t < tot; t += blockDim.x) dst[t] = tile[t];
    } else {
        for (int t = threadIdx.x; t < tot; t += blockDim.x) {
            const int l = t / wpl, q = t - l * wpl;
            dst[size_t(l) * ld + q] = tile[t];
        }
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
    const size_t kW = g->kernel_w, pW = g->pad_w, kH = g->kernel_h, sH = g->stride_h;
    // row-bits kernel: rows fit one word, padding windows stay inside the 64-bit shift (input
    // column of a tap in [-16, 48)). Output rows per block R: the most that keep the block's
    // smem <= 48 KB and still give every SM two blocks (a batch-1 layer: R = 1, or the general
    // kernel when even that leaves SMs idle).
    if (W <= 32 && pW <= 16 && oh < 65536 && B < 65536 && (ow - 1) * g->stride_w + kW <= 48 + pW) {
        auto smem_of = [&](size_t R) { return (C * ((R - 1) * sH + kH) + R * ow * wpl) * sizeof(uint32_t); };
        size_t R = 1;
        while (R < 16 && R * 2 <= oh && smem_of(R * 2) <= 48 * 1024 &&
               B * ceil_div(oh, R * 2) >= 2 * size_t(num_sms()))
            R *= 2;
        if (const char* e = getenv("BNN_IM2COL_R")) R = std::max(1, atoi(e));  // experiments
        if (smem_of(R) <= 48 * 1024) {
            im2col_rowbits_kernel<<<dim3(unsigned(ceil_div(oh, R)), unsigned(B)), 256, smem_of(R), s>>>(
                x, int(C), int(H), int(W), int(kH), int(kW), int(sH), int(g->stride_w), int(g->pad_h), int(pW),
                int(oh), int(ow), int(K), int(wpl), int(R), words, ld, nullptr, 0, 0, nullptr, nullptr);
            return launch_check("im2col_rowbits_kernel");
        }
    }
    dim3 grid(unsigned(ceil_div(lines, 32)), unsigned(ceil_div(wpl, kWordsPerBlock)));
    im2col_sign_pack_kernel<<<grid, dim3(32, kWordsPerBlock), 0, s>>>(
        x, int(C), int(H), int(W), int(g->kernel_h), int(g->kernel_w), int(g->stride_h),
        int(g->stride_w), int(g->pad_h), int(g->pad_w), int(oh), int(ow), lines, int(K), int(wpl),
        words, ld);
    return launch_check("im2col_sign_pack_kernel");
}

// conv_forward_binary in ONE launch for small layers (the row-bits im2col + a CUDA-core xnor
// GEMM per block, weights in shared memory): returns 1 when it handled the call, 0 when the
// shape needs the im2col + GEMM path.
int conv_rowbits_fused(const float* x, size_t B, size_t C, size_t H, size_t W, const uint32_t* pw, size_t ldw,
                       const float* bias, const bnn_conv_geom* g, float* out, cudaStream_t s, int* handled) {
    *handled = 0;
    size_t oh, ow;
    BNN_TRY(bnn_output_dims(g, H, W, &oh, &ow));
    const size_t K = g->kernel_h * g->kernel_w * C, wpl = wpl_of(K), D = g->out_channels;
    const size_t kW = g->kernel_w, pW = g->pad_w, kH = g->kernel_h, sH = g->stride_h;
    if (!(W <= 32 && pW <= 16 && oh < 65536 && B < 65536 && (ow - 1) * g->stride_w + kW <= 48 + pW)) return BNN_OK;
    const size_t smem = (C * kH + ow * wpl + D * wpl) * sizeof(uint32_t);  // one output row per block
    if (smem > 48 * 1024 || D * ow * wpl > 4096 * 36) return BNN_OK;
    // channel slices: enough blocks for two per SM when the batch x rows grid is small
    const size_t dz = std::max<size_t>(1, std::min<size_t>(ceil_div(2 * size_t(num_sms()), oh * B), D / 4));
    im2col_rowbits_kernel<<<dim3(unsigned(oh), unsigned(B), unsigned(dz)), 256, smem, s>>>(
        x, int(C), int(H), int(W), int(kH), int(kW), int(sH), int(g->stride_w), int(g->pad_h), int(pW), int(oh),
        int(ow), int(K), int(wpl), 1, nullptr, 0, pw, ldw, int(D), bias, out);
    BNN_TRY(launch_check("im2col_rowbits_kernel (fused conv)"));
    set_last_gemm("conv_rowbits_popc");
    *handled = 1;
    return BNN_OK;
}

}  // namespace bnnk

extern "C" int bnn_im2col_sign_pack_f32(const float* x, size_t B, size_t C, size_t H, size_t W,
                                        const bnn_conv_geom* g, uint32_t* words, size_t ld,
                                        bnn_stream_t s) {
    BNN_TRY(bnnk::require_sm100());
    return bnnk::launch_im2col_sign_pack(x, B, C, H, W, g, words, ld, bnnk::S(s));
}
