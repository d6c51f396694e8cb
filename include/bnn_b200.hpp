// bnn_b200.hpp — C++ drop-in for the reference operator API of the binarized-layer hot path.
//
// A program written against the reference library (namespace bnn, static lib bnncore,
// /root/reference/proj/include/bnn/*.hpp) switches to the B200 implementation by including
// this header instead of bnn/tensor.hpp, bnn/binarize.hpp, bnn/kernels.hpp, bnn/lowering.hpp
// and bnn/network.hpp, and linking libbnn_b200.so instead of bnncore. Types, function names,
// argument meaning, return-by-value ownership and exception types are the reference's; every
// compute call runs on the current CUDA device (sm_100a) through the C ABI of bnn_cuda.h
// (host buffers in and out, synchronous). There is no CPU fallback: without a B200 every
// compute call throws bnn::CudaError.
//
// Scope: encode (sign, htanh, pack_rows, pack_cols, unpack), lowering
// (binary im2col, flatten_weights, reshape_output), the xnor GEMM and its epilogue (xnor_gemm,
// to_float, bias_add), the two layer forwards, the network glue, and the seeded generator.
// Out of scope: the float control-group path (float_gemm,
// conv_forward_float, KernelChoice::Float), naive_conv, col2im, blob and JSON I/O, the CLI.
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

struct bnn_net;

namespace bnn {

// ---------------------------------------------------------------- errors (tensor.hpp:11-25)
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct EncodingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
// Not in the reference: a CUDA failure or a missing sm_100 device.
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- containers (tensor.hpp:27-114)
// [batch, channels, height, width], width fastest.
struct FloatTensor {
    std::size_t batch = 0, channels = 0, height = 0, width = 0;
    std::vector<float> data;
    FloatTensor() = default;
    FloatTensor(std::size_t n, std::size_t c, std::size_t h, std::size_t w);  // ShapeError on a 0 extent
    std::size_t size() const { return data.size(); }
    std::size_t index(std::size_t n, std::size_t c, std::size_t h, std::size_t w) const {
        return ((n * channels + c) * height + h) * width + w;
    }
    float at(std::size_t n, std::size_t c, std::size_t h, std::size_t w) const { return data[index(n, c, h, w)]; }
    float& at(std::size_t n, std::size_t c, std::size_t h, std::size_t w) { return data[index(n, c, h, w)]; }
};

// Row-major [rows, cols].
struct FloatMatrix {
    std::size_t rows = 0, cols = 0;
    std::vector<float> data;
    FloatMatrix() = default;
    FloatMatrix(std::size_t r, std::size_t c);  // ShapeError on a 0 extent
    float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    float& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
    const float* row(std::size_t r) const { return data.data() + r * cols; }
    float* row(std::size_t r) { return data.data() + r * cols; }
};

enum class PackOrientation : std::uint8_t { RowPacked = 0, ColPacked = 1 };
constexpr std::size_t kWordBits = 32;

// Packed {-1,+1} matrix: bit 1 = +1, logical index 32k+b of a line is bit b of word k,
// pad bits past the extent are 0 (the device kernels produce and rely on exactly this).
struct PackedBitMatrix {
    std::size_t logical_rows = 0, logical_cols = 0;
    PackOrientation orientation = PackOrientation::RowPacked;
    std::size_t words_per_line = 0;
    std::size_t pad_bits_per_line = 0;
    std::vector<std::uint32_t> words;

    static PackedBitMatrix make(std::size_t rows, std::size_t cols, PackOrientation o);
    std::size_t lines() const { return orientation == PackOrientation::RowPacked ? logical_rows : logical_cols; }
    std::size_t packed_extent() const {
        return orientation == PackOrientation::RowPacked ? logical_cols : logical_rows;
    }
    const std::uint32_t* line(std::size_t i) const { return words.data() + i * words_per_line; }
    std::uint32_t* line(std::size_t i) { return words.data() + i * words_per_line; }
    std::uint32_t pad_mask() const {
        return pad_bits_per_line ? ~std::uint32_t(0) << (kWordBits - pad_bits_per_line) : 0u;
    }
    std::size_t byte_size() const { return words.size() * sizeof(std::uint32_t); }
};

struct ConvGeometry {
    std::size_t kernel_h = 1, kernel_w = 1;
    std::size_t stride_h = 1, stride_w = 1;
    std::size_t pad_h = 0, pad_w = 0;
    std::size_t in_channels = 1;
    std::size_t out_channels = 1;
    std::size_t patch_len() const { return kernel_h * kernel_w * in_channels; }
};

// Exact xnor-popcount results, [rows, cols] row-major (kernels.hpp:13-22).
struct IntMatrix {
    std::size_t rows = 0, cols = 0;
    std::vector<std::int32_t> data;
    IntMatrix() = default;
    IntMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0) {}
    std::int32_t at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
    std::int32_t& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
};

// ---------------------------------------------------------------- geometry + generator
std::pair<std::size_t, std::size_t> output_dims(const ConvGeometry& geom, std::size_t in_h, std::size_t in_w);
std::uint64_t mix64(std::uint64_t seed, std::uint64_t counter);
float unit_random(std::uint64_t seed, std::uint64_t index);
// Generated on the device, bit-identical to the reference's counter-based generator.
FloatTensor fill_random(std::size_t n, std::size_t c, std::size_t h, std::size_t w, std::uint64_t seed);
FloatMatrix fill_random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed);
std::vector<float> fill_random_vector(std::size_t len, std::uint64_t seed);

// ---------------------------------------------------------------- encode (binarize.hpp)
FloatTensor sign(FloatTensor x);
FloatMatrix sign(FloatMatrix x);
FloatTensor htanh(FloatTensor x);
FloatMatrix htanh(FloatMatrix x);
// Strict packers: EncodingError naming the first non-+-1 entry in row-major order.
PackedBitMatrix pack_rows(const FloatMatrix& w);
PackedBitMatrix pack_cols(const FloatMatrix& x);
FloatMatrix unpack(const PackedBitMatrix& p);
// The fused encoder of the hot path: pack_rows(sign(w)) / pack_cols(sign(x)) in one kernel.
PackedBitMatrix sign_pack_rows(const FloatMatrix& w);
PackedBitMatrix sign_pack_cols(const FloatMatrix& x);

// ---------------------------------------------------------------- lowering (lowering.hpp)
// pack_cols(sign(im2col(x, batch_index, geom))) without the float patch matrix.
PackedBitMatrix im2col_sign_pack(const FloatTensor& x, std::size_t batch_index, const ConvGeometry& geom);
FloatTensor reshape_output(const FloatMatrix& m, std::size_t out_h, std::size_t out_w);
FloatMatrix flatten_weights(const FloatTensor& w);

// ---------------------------------------------------------------- GEMM (kernels.hpp)
// `threads` is accepted for source compatibility; the device grid replaces it.
IntMatrix xnor_gemm(const PackedBitMatrix& w, const PackedBitMatrix& x, std::size_t inner_len,
                    unsigned threads = 1);
FloatMatrix to_float(const IntMatrix& m);
FloatMatrix bias_add(FloatMatrix a, std::span<const float> bias);

// ---------------------------------------------------------------- layers (network.hpp)
enum class LayerKind { Conv, Linear, MaxPool, AffineNorm, SignAct, HtanhAct };
enum class KernelChoice { Float, Binary, Naive };

FloatTensor conv_forward_binary(const FloatTensor& x, const PackedBitMatrix& packed_w,
                                std::span<const float> bias, const ConvGeometry& geom, unsigned threads = 1);
// Only KernelChoice::Binary is on the device path; Float/Naive throw ConfigError.
FloatMatrix linear_forward(const FloatMatrix& x, const FloatMatrix& w, std::span<const float> bias,
                           KernelChoice kernel, unsigned threads = 1);
FloatMatrix linear_forward_packed(const FloatMatrix& x, const PackedBitMatrix& packed_w,
                                  std::span<const float> bias, unsigned threads = 1);
FloatTensor maxpool2(const FloatTensor& x);
FloatTensor affine_norm(FloatTensor x, std::span<const float> scale, std::span<const float> shift);
FloatMatrix affine_norm(FloatMatrix x, std::span<const float> scale, std::span<const float> shift);
FloatMatrix flatten_to_columns(const FloatTensor& x);

// ---------------------------------------------------------------- network (network.hpp)
struct LayerSpec {
    LayerKind kind = LayerKind::SignAct;
    std::size_t out_channels = 0;
    std::size_t kernel_h = 0, kernel_w = 0;
    std::size_t stride_h = 1, stride_w = 1;
    std::size_t pad_h = 0, pad_w = 0;
    std::size_t out_features = 0;
    KernelChoice kernel = KernelChoice::Float;
    std::optional<std::uint64_t> seed;
    std::string weights_blob;  // tensor blob path; empty -> seeded weights (network.hpp:36)
};

struct NetworkSpec {
    std::string name;
    std::array<std::size_t, 4> input_shape{1, 3, 32, 32};
    std::uint64_t seed = 1;
    bool binarize_weights = false;
    std::vector<LayerSpec> layers;
};

// The reference's VGG-small benchmark topology (network.cpp:422-465).
NetworkSpec build_default_network(KernelChoice kernel, std::uint64_t seed);

// build_network + network_forward(ExecKernel::Binary) on the current device: parameters are
// generated from the spec's seeds and packed once at construction (network.cpp:203-306).
class DeviceNetwork {
public:
    explicit DeviceNetwork(const NetworkSpec& spec);
    // load_network_spec (network.cpp:487-536) + build_network: a NetworkSpec JSON file.
    static DeviceNetwork from_spec_file(const std::string& path);
    ~DeviceNetwork();
    DeviceNetwork(const DeviceNetwork&) = delete;
    DeviceNetwork& operator=(const DeviceNetwork&) = delete;
    // [batch, C, H, W] -> logits [features, batch] (network.hpp:104-105).
    FloatMatrix forward(const FloatTensor& x);
    std::size_t logits() const;
    bnn_net* handle() const { return net_; }

private:
    DeviceNetwork() = default;
    bnn_net* net_ = nullptr;
    std::array<std::size_t, 3> in_chw_{};

public:
    DeviceNetwork(DeviceNetwork&& o) noexcept : net_(o.net_), in_chw_(o.in_chw_) { o.net_ = nullptr; }
};

// ------------------------------------------------------- on-disk formats (binarize.hpp:28-32,
// tensor.hpp:129-133): byte-identical to the reference's files, same IoError messages.
void save_packed_blob(const PackedBitMatrix& p, const std::string& path);
PackedBitMatrix load_packed_blob(const std::string& path);
void save_tensor_blob(const FloatTensor& t, const std::string& path);
FloatTensor load_tensor_blob(const std::string& path);

FloatMatrix network_forward(DeviceNetwork& net, const FloatTensor& x);

// FNV-1a over the float bytes (bench.cpp:23-33): cheap whole-output bit-exactness checks.
std::uint64_t fnv1a_hash(std::span<const float> values);

}  // namespace bnn

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
