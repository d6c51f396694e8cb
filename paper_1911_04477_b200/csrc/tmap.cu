// TMA tensor maps over byte matrices (the fused engine's int8 / e2m1 weight operands).
#include <cuda.h>

#include <mutex>

#include "bnn_common.cuh"

namespace bnnk {

namespace {

constexpr int kBK = 128;  // bytes of K per box row: one 128-byte swizzle atom row

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

}  // namespace bnnk
