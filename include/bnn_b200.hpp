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
// Scope: the reference's tensor.hpp, binarize.hpp, lowering.hpp, kernels.hpp, network.hpp and
// bench.hpp declarations: encode, lowering (im2col, col2im,
// reshape_output, flatten_weights), the xnor GEMM and its epilogue, the float control group
// (float_gemm, conv_forward_float), the BinaryReference and naive forwards, the network
// (build_network, network_forward with ExecKernel / ForwardOptions, the JSON spec), the
// bench/verify harness (run_benchmark, run_verify, verify_network, the report JSON) and the
// blob formats. Additions beyond the reference are marked "B200:". Not provided: the bnnbench
// CLI (out of scope).
#pragma once

#include <array>
#include <bit>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <iosfwd>
#include <memory>
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
// [K*K*C, outH*outW] float patch matrix of one batch slice (lowering.hpp:11), on the device.
FloatMatrix im2col(const FloatTensor& x, std::size_t batch_index, const ConvGeometry& geom);
// Adjoint of im2col (lowering.hpp:17-18), on the device, bit-identical sums.
FloatTensor col2im(const FloatMatrix& m, const ConvGeometry& geom, std::size_t out_h, std::size_t out_w);
// B200: pack_cols(sign(im2col(x, batch_index, geom))) without the float patch matrix.
PackedBitMatrix im2col_sign_pack(const FloatTensor& x, std::size_t batch_index, const ConvGeometry& geom);
FloatTensor reshape_output(const FloatMatrix& m, std::size_t out_h, std::size_t out_w);
FloatMatrix flatten_weights(const FloatTensor& w);

// ---------------------------------------------------------------- GEMM (kernels.hpp)
// Word primitives (kernels.hpp:25-39): host inline like the reference's; the device kernels use
// the POPC / LOP3 instructions and the tensor cores instead.
constexpr int popcount32_portable(std::uint32_t x) noexcept {
    x = x - ((x >> 1) & 0x55555555u);
    x = (x & 0x33333333u) + ((x >> 2) & 0x33333333u);
    x = (x + (x >> 4)) & 0x0F0F0F0Fu;
    return static_cast<int>((x * 0x01010101u) >> 24);
}
inline int popcount32(std::uint32_t x) noexcept { return std::popcount(x); }
inline int word_dot(std::uint32_t w, std::uint32_t x) noexcept { return 2 * popcount32(~(w ^ x)) - 32; }

// Control-group float GEMM (kernels.hpp:44), on the CUDA cores with the reference's k-ascending
// FMA chain per output: bit-identical. `threads` is accepted for source compatibility.
FloatMatrix float_gemm(const FloatMatrix& w, const FloatMatrix& x, unsigned threads = 1);
// Direct convolution of one batch slice (kernels.hpp:63-64), bit-identical.
FloatTensor naive_conv(const FloatTensor& x, std::size_t batch_index, const FloatTensor& w, const ConvGeometry& geom);
// `threads` is accepted for source compatibility; the device grid replaces it. The kernel
// follows the product size (bnn_set_gemm_policy, include/bnn_cuda.h): LOP3 + POPC below 2^26
// bit-MACs, FP4 tensor cores with in-CTA operand expansion up to 2^32, TMA-fed FP4 CTA pairs
// over operands expanded once in HBM above; every choice is bit-exact.
IntMatrix xnor_gemm(const PackedBitMatrix& w, const PackedBitMatrix& x, std::size_t inner_len,
                    unsigned threads = 1);
FloatMatrix to_float(const IntMatrix& m);
FloatMatrix bias_add(FloatMatrix a, std::span<const float> bias);

// ---------------------------------------------------------------- layers (network.hpp)
enum class LayerKind { Conv, Linear, MaxPool, AffineNorm, SignAct, HtanhAct };
enum class KernelChoice { Float, Binary, Naive };

const char* to_string(LayerKind k);
const char* to_string(KernelChoice k);
LayerKind parse_layer_kind(const std::string& s);
KernelChoice parse_kernel_choice(const std::string& s);

FloatTensor conv_forward_float(const FloatTensor& x, const FloatMatrix& w_flat, std::span<const float> bias,
                               const ConvGeometry& geom, unsigned threads = 1);
FloatTensor conv_forward_binary(const FloatTensor& x, const PackedBitMatrix& packed_w,
                                std::span<const float> bias, const ConvGeometry& geom, unsigned threads = 1);
FloatTensor conv_forward_binary_reference(const FloatTensor& x, const FloatMatrix& w_pm1, std::span<const float> bias,
                                          const ConvGeometry& geom, unsigned threads = 1);
FloatTensor conv_forward_naive(const FloatTensor& x, const FloatTensor& w, std::span<const float> bias,
                               const ConvGeometry& geom);
FloatMatrix linear_forward(const FloatMatrix& x, const FloatMatrix& w, std::span<const float> bias,
                           KernelChoice kernel, unsigned threads = 1);
FloatMatrix linear_forward_packed(const FloatMatrix& x, const PackedBitMatrix& packed_w,
                                  std::span<const float> bias, unsigned threads = 1);
FloatMatrix linear_forward_binary_reference(const FloatMatrix& x, const FloatMatrix& w_pm1,
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
    bool operator==(const LayerSpec&) const = default;
};

struct NetworkSpec {
    std::string name;
    std::array<std::size_t, 4> input_shape{1, 3, 32, 32};
    std::uint64_t seed = 1;
    bool binarize_weights = false;
    std::vector<LayerSpec> layers;
    bool operator==(const NetworkSpec&) const = default;
};

// A layer with resolved shapes and its parameters (network.hpp:57-77). The host copies mirror
// the device engine's; network_forward re-uploads any the caller changed.
struct BuiltLayer {
    LayerSpec spec;
    ConvGeometry geom;
    std::size_t in_features = 0, out_features = 0;
    FloatTensor weight_tensor;       // conv, [D, C, kH, kW]
    FloatMatrix weights;             // conv [D, K2C] / linear [out, in]
    PackedBitMatrix packed_weights;  // row-packed sign(weights)
    std::vector<float> bias;
    std::vector<float> scale, shift;
    std::size_t out_channels = 0, out_h = 0, out_w = 0;
    bool out_flat = false;
    bool has_weights() const { return spec.kind == LayerKind::Conv || spec.kind == LayerKind::Linear; }
    std::size_t float_weight_bytes() const { return weights.data.size() * sizeof(float); }
    std::size_t packed_weight_bytes() const { return packed_weights.byte_size(); }
};

namespace detail {
struct DeviceEngine;  // the device network (bnn_net) + the parameter snapshot it was built from
}

struct Network {
    NetworkSpec spec;
    std::vector<BuiltLayer> layers;
    std::size_t in_channels = 0, in_h = 0, in_w = 0;
    std::size_t logits = 0;
    std::size_t parameter_count = 0;
    // B200: the device engine build_network created (parameters generated and packed on the
    // device once). Copies of a Network share it.
    std::shared_ptr<detail::DeviceEngine> device;
};

// Validate the shape chain and materialize the parameters (network.cpp:203-306), on the device.
Network build_network(const NetworkSpec& spec);

enum class ExecKernel { PerLayer, Float, Binary, Naive, BinaryReference };

struct ForwardOptions {
    ExecKernel kernel = ExecKernel::PerLayer;
    unsigned threads = 1;                          // accepted; the device grid replaces it
    std::vector<double>* layer_seconds = nullptr;  // per-layer device time (CUDA events), accumulated
};

// network_forward (network.hpp:104-105): [batch, C, H, W] -> logits [features, batch].
// ExecKernel::Binary (and PerLayer over an all-Binary network) runs the fused tcgen05 engine;
// the others run their layer-by-layer device graphs. Bit-identical to the reference for every
// ExecKernel. layer_seconds: the fused engine folds each weighted layer's glue into its launch,
// so the glue layers' entries stay 0.
FloatMatrix network_forward(const Network& net, const FloatTensor& x, const ForwardOptions& opts = {});

// The reference's VGG-small benchmark topology (network.cpp:422-465).
NetworkSpec build_default_network(KernelChoice kernel, std::uint64_t seed);
NetworkSpec load_network_spec(const std::string& path);
void save_network_spec(const NetworkSpec& spec, const std::string& path);

// B200: the device network as an owning handle (build_network + network_forward(Binary)), for
// callers that keep one network resident; Network above is the reference-shaped entry point.
class DeviceNetwork {
public:
    explicit DeviceNetwork(const NetworkSpec& spec);
    static DeviceNetwork from_spec_file(const std::string& path);
    ~DeviceNetwork();
    DeviceNetwork(const DeviceNetwork&) = delete;
    DeviceNetwork& operator=(const DeviceNetwork&) = delete;
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

// ---------------------------------------------------------------- harness (bench.hpp)
constexpr double kVerifyTolerance = 1e-4;

struct BenchConfig {
    std::string spec_path;  // empty: built-in default network
    std::vector<KernelChoice> kernels{KernelChoice::Binary, KernelChoice::Float};
    std::size_t batch = 64;
    std::size_t iterations = 20;
    std::size_t warmup = 3;
    unsigned threads = 1;
    std::uint64_t seed = 1;
    std::string out_path;
    std::string input_blob;
    bool layer_times = true;
};

struct KernelStats {
    KernelChoice kernel = KernelChoice::Binary;
    std::vector<double> samples_s;  // wall-clock seconds per timed network_forward
    double median_s = 0, min_s = 0, mean_s = 0;
    std::vector<double> layer_seconds;
    std::uint64_t logits_hash = 0;
};

struct SpeedupEntry {
    std::string baseline;
    std::string target;
    double ratio = 0;
};

struct LayerMemory {
    std::size_t layer_index = 0;
    std::string label;
    std::size_t float_bytes = 0;
    std::size_t packed_bytes = 0;
};

struct BenchReport {
    std::string network_name;
    std::string spec_path;
    std::size_t batch = 0, iterations = 0, warmup = 0;
    unsigned threads = 1;
    std::uint64_t seed = 0;
    std::string environment;
    double timer_resolution_ns = 0;
    std::vector<KernelStats> kernels;
    std::vector<LayerMemory> weight_memory;
    std::size_t total_float_bytes = 0, total_packed_bytes = 0;
    std::vector<SpeedupEntry> speedups;
};

struct VerifySummary {
    std::string network_name;
    std::size_t batch = 0;
    std::size_t compared = 0;
    double max_abs_deviation = 0;
    double tolerance = kVerifyTolerance;
    bool pass = false;
    bool pad_correction_exercised = false;
};

double median(std::vector<double> samples);
// FNV-1a over the float bytes (bench.cpp:23-33).
std::uint64_t fnv1a_hash(const FloatMatrix& m);
// B200: the same hash of any float span.
std::uint64_t fnv1a_hash(std::span<const float> values);
BenchReport run_benchmark(const BenchConfig& cfg);
VerifySummary run_verify(const BenchConfig& cfg);
// Binary vs BinaryReference on the device (bench.cpp:172-191); the max deviation is reduced on
// the device. Callers may perturb net.layers[i] first (test hook, test_bench.cpp:159-173).
VerifySummary verify_network(const Network& net, const FloatTensor& input, unsigned threads = 1);
void emit_report(const BenchReport& r, const std::string& path);
BenchReport parse_report(const std::string& path);
void print_report(const BenchReport& r, std::ostream& os);

}  // namespace bnn

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
