// Shared helpers for the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "bnn_cuda.h"

namespace bnnk {

// Thread-local error state behind bnn_last_error().
int fail(int code, const std::string& msg);
void set_last_gemm(const char* name);

inline cudaStream_t S(bnn_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }
inline size_t wpl_of(size_t extent) { return (extent + 31) / 32; }

// Kernel launch check: launch errors are reported as BNN_E_CUDA with the kernel name.
int launch_check(const char* what);

// Number of SMs on the current device (cached per device).
int num_sms();

// The device must be sm_100 (B200). Checked once per device.
int require_sm100();

// Stream-ordered scratch allocation (cudaMallocAsync on the caller's stream).
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    int alloc(size_t bytes, cudaStream_t st) {
        s = st;
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, st);
        if (e != cudaSuccess) {
            p = nullptr;
            return fail(BNN_E_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
        }
        return BNN_OK;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// tensor.cpp:65-71 — counter-based splitmix64 (host + device).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// tensor.cpp:73-77 — top 24 bits -> [-1, 1), exact in f32.
__host__ __device__ __forceinline__ float unit_random(uint64_t seed, uint64_t index) {
    const uint32_t top = static_cast<uint32_t>(mix64(seed, index) >> 40);
    return static_cast<float>(top) * 0x1.0p-23f - 1.0f;
}

#ifdef __CUDACC__
// A value every lane of the (converged) warp holds, through a lane-0 shuffle: ptxas then treats it
// as warp-uniform, so role branches on the warp index are uniform branches and what is computed
// under them (UMMA descriptors, TMEM addresses) stays in uniform registers.
__device__ __forceinline__ int warp_uniform(int x) { return __shfl_sync(0xffffffffu, x, 0); }
__device__ __forceinline__ uint32_t warp_uniform(uint32_t x) { return __shfl_sync(0xffffffffu, x, 0); }
#endif

}  // namespace bnnk

#define BNN_TRY(expr)                 \
    do {                              \
        int rc_ = (expr);             \
        if (rc_ != BNN_OK) return rc_; \
    } while (0)

#define BNN_CUDA(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return ::bnnk::fail(BNN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)
