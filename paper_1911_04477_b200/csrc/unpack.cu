// Packed bits -> signed int8 {-1,+1} operand rows for the tcgen05 kind::i8 GEMM.
//
// Line l of `words` (reference layout, LSB-first, bit 1 = +1) becomes row l of `out`: byte k
// is +1 / -1 for k < L and 0 for L <= k < ld_out, so the K padding contributes nothing to
// the int8 dot product. HBM-bound: 1 bit read per byte written.
#include "bnn_common.cuh"

namespace bnnk {
namespace {

// 4 bits -> 4 bytes of +1 (0x01) / -1 (0xFF): spread the nibble to byte lanes, then
// ~(t * 0xFE) maps a byte 1 -> 0x01 and 0 -> 0xFF without carries between bytes.
__device__ __forceinline__ uint32_t nib_pm1(uint32_t nib) {
    const uint32_t t = (nib * 0x00204081u) & 0x01010101u;
    return ~(t * 0xFEu);
}

__global__ void unpack_s8_kernel(const uint32_t* __restrict__ words, size_t ldw, size_t lines,
                                 int L, int ld_out, int8_t* __restrict__ out) {
    const int chunks = ld_out / 32;  // 32 output bytes per thread
    const size_t total = lines * size_t(chunks);
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t line = i / chunks;
        const int c = int(i % chunks);
        const int k0 = c * 32;
        uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
        if (k0 < L) {
            const uint32_t w = words[line * ldw + c];
            uint32_t v[8];
#pragma unroll
            for (int n = 0; n < 8; ++n) v[n] = nib_pm1((w >> (4 * n)) & 0xFu);
            if (k0 + 32 > L) {  // partial last word: bytes past L are 0
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    uint32_t keep = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (k0 + 4 * n + b < L) keep |= 0xFFu << (8 * b);
                    v[n] &= keep;
                }
            }
            lo = make_uint4(v[0], v[1], v[2], v[3]);
            hi = make_uint4(v[4], v[5], v[6], v[7]);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + line * size_t(ld_out) + k0);
        dst[0] = lo;
        dst[1] = hi;
    }
}

}  // namespace

// ld_out must be a multiple of 32 and >= L.
int launch_unpack_s8(const uint32_t* words, size_t ldw, size_t lines, size_t L, int8_t* out,
                     size_t ld_out, cudaStream_t s) {
    if (ld_out % 32 != 0 || ld_out < L) return fail(BNN_E_SHAPE, "unpack_s8: bad output stride");
    const size_t total = lines * (ld_out / 32);
    if (total == 0) return BNN_OK;
    size_t g = ceil_div(total, 256);
    g = std::min<size_t>(g, size_t(num_sms()) * 32);
    unpack_s8_kernel<<<unsigned(g), 256, 0, s>>>(words, ldw, lines, int(L), int(ld_out), out);
    return launch_check("unpack_s8_kernel");
}

}  // namespace bnnk
