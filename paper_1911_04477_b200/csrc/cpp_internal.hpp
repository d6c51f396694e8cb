// Internal helpers shared by the C++ reference-signature API translation units (cpp_api.cpp,
// cpp_network.cpp, bench_api.cpp): C-ABI status -> reference exception, and a synchronous device
// buffer on the legacy default stream.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#include "bnn_b200.hpp"
#include "bnn_cuda.h"

namespace bnn {
namespace cppi {

[[noreturn]] inline void raise(int rc) {
    const std::string msg = bnn_last_error();
    switch (rc) {
        case BNN_E_SHAPE: throw ShapeError(msg);
        case BNN_E_ENCODING: throw EncodingError(msg);
        case BNN_E_CONFIG: throw ConfigError(msg);
        case BNN_E_IO: throw IoError(msg);
        default: throw CudaError(msg);
    }
}

inline void check(int rc) {
    if (rc != BNN_OK) raise(rc);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer; synchronous copies on the legacy default stream (the stream every call here uses).
class Dev {
public:
    explicit Dev(std::size_t bytes) { cuda(cudaMalloc(&p_, bytes ? bytes : 16), "cudaMalloc"); }
    ~Dev() { cudaFree(p_); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    void put(const void* src, std::size_t bytes) { cuda(cudaMemcpy(p_, src, bytes, cudaMemcpyHostToDevice), "H2D"); }
    void get(void* dst, std::size_t bytes) const { cuda(cudaMemcpy(dst, p_, bytes, cudaMemcpyDeviceToHost), "D2H"); }

private:
    void* p_ = nullptr;
};

inline void check_extent(std::size_t v, const char* name) {  // tensor.cpp:11-13
    if (v == 0) throw ShapeError(std::string("extent '") + name + "' must be >= 1");
}

inline bnn_conv_geom to_c(const ConvGeometry& g) {
    return bnn_conv_geom{g.kernel_h, g.kernel_w, g.stride_h, g.stride_w, g.pad_h, g.pad_w, g.in_channels,
                         g.out_channels};
}


}  // namespace cppi
}  // namespace bnn
