// On-disk formats of the reference, loaded onto / written from the B200 path (SURVEY.md §8(f)
// row f2). Host code only: file bytes <-> caller buffers; the network builder copies the
// loaded weights to the device and packs them there.
//
//   packed blob  binarize.cpp:116-148 / binarize.hpp:28-32: orientation byte (0 row-packed,
//                1 col-packed), logical rows and cols as little-endian u64, then the words as
//                little-endian u32 (lines x ceil(extent / 32)); pad bits must be 0.
//   tensor blob  tensor.cpp:123-150 / tensor.hpp:129-133: batch, channels, height, width as
//                little-endian u64, then the floats as little-endian f32 (NCHW).
//   NetworkSpec  network.cpp:487-567: JSON {name, input_shape[4], seed, binarize_weights,
//                kernel, layers[{kind, out_channels, kernel_size, stride, pad, out_features,
//                kernel, seed, weights_blob}]}; kernel_size/stride/pad are a number or a pair.
//
// Error behaviour follows the reference: IoError (BNN_E_IO) for file problems with the same
// messages, ConfigError (BNN_E_CONFIG) for malformed specs.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "bnn_b200.hpp"
#include "bnn_cuda.h"

namespace bnnk {
int fail(int code, const std::string& msg);
}

namespace {

using json = nlohmann::json;

void put_u64le(std::string& b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back(char((v >> (8 * i)) & 0xff));
}
void put_u32le(std::string& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(char((v >> (8 * i)) & 0xff));
}
uint64_t get_u64le(const unsigned char* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
    return v;
}
uint32_t get_u32le(const unsigned char* p) {
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= uint32_t(p[i]) << (8 * i);
    return v;
}

int read_file(const char* path, std::string& buf) {
    std::ifstream is(path, std::ios::binary);
    if (!is) return bnnk::fail(BNN_E_IO, std::string("cannot open for reading: ") + path);
    buf.assign(std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>());
    return BNN_OK;
}

int write_file(const char* path, const std::string& buf) {
    std::ofstream os(path, std::ios::binary);
    if (!os) return bnnk::fail(BNN_E_IO, std::string("cannot open for writing: ") + path);
    os.write(buf.data(), std::streamsize(buf.size()));
    if (!os) return bnnk::fail(BNN_E_IO, std::string("write failed: ") + path);
    return BNN_OK;
}

struct ParsedSpec {
    bnn::NetworkSpec spec;
    std::vector<bnn_layer_spec> layers;
};

// load_network_spec with its exceptions mapped onto the C ABI's status codes.
int parse_spec(const char* path, ParsedSpec& out) {
    try {
        out.spec = bnn::load_network_spec(path);
    } catch (const bnn::ConfigError& e) {
        return bnnk::fail(BNN_E_CONFIG, e.what());
    } catch (const bnn::ShapeError& e) {
        return bnnk::fail(BNN_E_SHAPE, e.what());
    } catch (const bnn::IoError& e) {
        return bnnk::fail(BNN_E_IO, e.what());
    } catch (const std::exception& e) {
        return bnnk::fail(BNN_E_CONFIG, e.what());
    }
    for (const bnn::LayerSpec& l : out.spec.layers) {
        bnn_layer_spec c{};
        c.kind = uint32_t(l.kind);
        c.has_seed = l.seed ? 1 : 0;
        c.seed = l.seed.value_or(0);
        c.out_channels = l.out_channels;
        c.kernel_h = l.kernel_h, c.kernel_w = l.kernel_w;
        c.stride_h = l.stride_h, c.stride_w = l.stride_w;
        c.pad_h = l.pad_h, c.pad_w = l.pad_w;
        c.out_features = l.out_features;
        c.kernel = uint32_t(l.kernel);
        out.layers.push_back(c);
    }
    for (size_t i = 0; i < out.layers.size(); ++i)  // pointers into out.spec, which outlives the calls below
        out.layers[i].weights_blob = out.spec.layers[i].weights_blob.empty() ? nullptr : out.spec.layers[i].weights_blob.c_str();
    return BNN_OK;
}

// kernel_size / stride / pad: a number or a [h, w] pair (network.cpp:470-482). A malformed
// pair is a ConfigError with the reference's own text (not wrapped: it is not a json error).
std::pair<size_t, size_t> pair_field(const json& lj, const char* key, size_t dflt) {
    if (!lj.contains(key)) return {dflt, dflt};
    const json& v = lj.at(key);
    if (!v.is_array()) {
        const size_t s = v.get<size_t>();
        return {s, s};
    }
    if (v.size() != 2) throw bnn::ConfigError(std::string(key) + " must be a scalar or [h, w]");
    return {v[0].get<size_t>(), v[1].get<size_t>()};
}

}  // namespace

extern "C" {

// save_packed_blob (binarize.cpp:116-127)
int bnn_save_packed_blob(const char* path, int orientation, uint64_t rows, uint64_t cols, const uint32_t* words) {
    if (orientation != 0 && orientation != 1) return bnnk::fail(BNN_E_CONFIG, "orientation must be 0 or 1");
    const uint64_t lines = orientation == 0 ? rows : cols, extent = orientation == 0 ? cols : rows;
    const uint64_t n = lines * bnn_words_per_line(extent);
    std::string buf;
    buf.reserve(17 + 4 * n);
    buf.push_back(char(orientation));
    put_u64le(buf, rows);
    put_u64le(buf, cols);
    for (uint64_t i = 0; i < n; ++i) put_u32le(buf, words[i]);
    return write_file(path, buf);
}

// load_packed_blob (binarize.cpp:129-148): words == NULL queries the header only.
int bnn_load_packed_blob(const char* path, int* orientation, uint64_t* rows, uint64_t* cols, uint32_t* words,
                         size_t cap_words) {
    std::string buf;
    if (int rc = read_file(path, buf)) return rc;
    if (buf.size() < 17) return bnnk::fail(BNN_E_IO, std::string("packed blob truncated: ") + path);
    const auto* raw = reinterpret_cast<const unsigned char*>(buf.data());
    const uint8_t ob = raw[0];
    if (ob > 1) return bnnk::fail(BNN_E_IO, std::string("packed blob has bad orientation byte: ") + path);
    const uint64_t r = get_u64le(raw + 1), c = get_u64le(raw + 9);
    if (r == 0) return bnnk::fail(BNN_E_SHAPE, "extent 'rows' must be >= 1");  // PackedBitMatrix::make
    if (c == 0) return bnnk::fail(BNN_E_SHAPE, "extent 'cols' must be >= 1");
    const uint64_t lines = ob == 0 ? r : c, extent = ob == 0 ? c : r, wpl = bnn_words_per_line(extent);
    const uint64_t n = lines * wpl;
    if (buf.size() != 17 + 4 * n) return bnnk::fail(BNN_E_IO, std::string("packed blob size mismatch: ") + path);
    const uint32_t pad = uint32_t(wpl * 32 - extent);
    const uint32_t mask = pad ? ~((~0u) >> pad) : 0u;  // PackedBitMatrix::pad_mask (tensor.cpp:39-44)
    for (uint64_t li = 0; mask && li < lines; ++li)
        if (get_u32le(raw + 17 + 4 * (li * wpl + wpl - 1)) & mask)
            return bnnk::fail(BNN_E_IO, std::string("packed blob has nonzero pad bits: ") + path);
    if (orientation) *orientation = ob;
    if (rows) *rows = r;
    if (cols) *cols = c;
    if (!words) return BNN_OK;
    if (cap_words < n) return bnnk::fail(BNN_E_SHAPE, "packed blob: output buffer too small");
    for (uint64_t i = 0; i < n; ++i) words[i] = get_u32le(raw + 17 + 4 * i);
    return BNN_OK;
}

// save_tensor_blob (tensor.cpp:123-134)
int bnn_save_tensor_blob(const char* path, const uint64_t shape[4], const float* data) {
    const uint64_t n = shape[0] * shape[1] * shape[2] * shape[3];
    std::string buf;
    buf.reserve(32 + 4 * n);
    for (int i = 0; i < 4; ++i) put_u64le(buf, shape[i]);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t v;
        std::memcpy(&v, data + i, 4);
        put_u32le(buf, v);
    }
    return write_file(path, buf);
}

// load_tensor_blob (tensor.cpp:136-150): data == NULL queries the shape only.
int bnn_load_tensor_blob(const char* path, uint64_t shape[4], float* data, size_t cap) {
    std::string buf;
    if (int rc = read_file(path, buf)) return rc;
    if (buf.size() < 32) return bnnk::fail(BNN_E_IO, std::string("tensor blob truncated: ") + path);
    const auto* p = reinterpret_cast<const unsigned char*>(buf.data());
    uint64_t s[4];
    static const char* names[4] = {"batch", "channels", "height", "width"};
    for (int i = 0; i < 4; ++i) {
        s[i] = get_u64le(p + 8 * i);
        if (s[i] == 0) return bnnk::fail(BNN_E_SHAPE, std::string("extent '") + names[i] + "' must be >= 1");
    }
    const uint64_t n = s[0] * s[1] * s[2] * s[3];
    if (buf.size() != 32 + 4 * n) return bnnk::fail(BNN_E_IO, std::string("tensor blob size mismatch: ") + path);
    for (int i = 0; i < 4; ++i) shape[i] = s[i];
    if (!data) return BNN_OK;
    if (cap < n) return bnnk::fail(BNN_E_SHAPE, "tensor blob: output buffer too small");
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t v = get_u32le(p + 32 + 4 * i);
        std::memcpy(data + i, &v, 4);
    }
    return BNN_OK;
}

// load_network_spec (network.cpp:487-536) + build_network (network.cpp:203-306): layers with a
// weights_blob take their float weights from that tensor blob, the rest from the seeds.
// binarize_override: -1 keeps the spec's binarize_weights (packed bits do not depend on it).
int bnn_net_create_from_spec(const char* path, int binarize_override, bnn_net** out) {
    ParsedSpec sp;
    if (int rc = parse_spec(path, sp)) return rc;
    const int bin = binarize_override >= 0 ? binarize_override : (sp.spec.binarize_weights ? 1 : 0);
    const auto& s = sp.spec.input_shape;
    return bnn_net_create(sp.layers.data(), sp.layers.size(), s[1], s[2], s[3], sp.spec.seed, bin, out);
}

// Spec header for callers that build their own inputs: input_shape and layer count.
int bnn_spec_info(const char* path, uint64_t input_shape[4], size_t* n_layers) {
    ParsedSpec sp;
    if (int rc = parse_spec(path, sp)) return rc;
    for (int i = 0; i < 4; ++i) input_shape[i] = sp.spec.input_shape[i];
    if (n_layers) *n_layers = sp.layers.size();
    return BNN_OK;
}

}  // extern "C"

// ------------------------------------------------------------ C++ API: the NetworkSpec schema
namespace bnn {

const char* to_string(LayerKind k) {  // network.cpp:10-20
    static const char* names[] = {"conv", "linear", "maxpool", "affine_norm", "sign", "htanh"};
    const unsigned i = unsigned(k);
    return i < 6 ? names[i] : "?";
}

const char* to_string(KernelChoice k) {  // network.cpp:22-29
    static const char* names[] = {"float", "binary", "naive"};
    const unsigned i = unsigned(k);
    return i < 3 ? names[i] : "?";
}

LayerKind parse_layer_kind(const std::string& s) {  // network.cpp:31-39
    for (unsigned i = 0; i < 6; ++i)
        if (s == to_string(LayerKind(i))) return LayerKind(i);
    throw ConfigError("unknown layer kind '" + s + "'");
}

KernelChoice parse_kernel_choice(const std::string& s) {  // network.cpp:41-46
    for (unsigned i = 0; i < 3; ++i)
        if (s == to_string(KernelChoice(i))) return KernelChoice(i);
    throw ConfigError("unknown kernel choice '" + s + "', expected binary|float|naive");
}

// load_network_spec (network.cpp:487-536): the same schema, defaults and error behaviour -- json
// type / missing-key errors become ConfigError("bad network spec <path>: ..."), the schema's own
// ConfigErrors (bad shape, unknown kind or kernel, malformed pair) pass through unwrapped.
NetworkSpec load_network_spec(const std::string& path) {
    std::ifstream is(path);
    if (!is) throw ConfigError("cannot open network spec: " + path);
    json j;
    try {
        j = json::parse(is);
    } catch (const json::parse_error& e) {
        throw ConfigError("parse error in " + path + ": " + e.what());
    }
    try {
        NetworkSpec spec;
        spec.name = j.value("name", std::string("unnamed"));
        if (j.contains("input_shape")) {
            const json& sh = j.at("input_shape");
            if (!sh.is_array() || sh.size() != 4) throw ConfigError("input_shape must be [batch, channels, height, width]");
            for (size_t i = 0; i < 4; ++i) spec.input_shape[i] = sh[i].get<size_t>();
        }
        spec.seed = j.value("seed", uint64_t{1});
        spec.binarize_weights = j.value("binarize_weights", false);
        const KernelChoice fallback = parse_kernel_choice(j.value("kernel", std::string("float")));
        if (!j.contains("layers") || !j.at("layers").is_array()) throw ConfigError("spec needs a 'layers' array");
        for (const json& lj : j.at("layers")) {
            LayerSpec l;
            l.kind = parse_layer_kind(lj.at("kind").get<std::string>());
            const bool weighted = l.kind == LayerKind::Conv || l.kind == LayerKind::Linear;
            if (l.kind == LayerKind::Conv) {
                l.out_channels = lj.at("out_channels").get<size_t>();
                std::tie(l.kernel_h, l.kernel_w) = pair_field(lj, "kernel_size", 0);
                if (l.kernel_h == 0) throw ConfigError("conv layer needs kernel_size");
                std::tie(l.stride_h, l.stride_w) = pair_field(lj, "stride", 1);
                std::tie(l.pad_h, l.pad_w) = pair_field(lj, "pad", 0);
            } else if (l.kind == LayerKind::Linear) {
                l.out_features = lj.at("out_features").get<size_t>();
            }
            if (weighted) {
                l.kernel = lj.contains("kernel") ? parse_kernel_choice(lj.at("kernel").get<std::string>()) : fallback;
                l.weights_blob = lj.value("weights_blob", std::string{});
            }
            if (lj.contains("seed")) l.seed = lj.at("seed").get<uint64_t>();
            spec.layers.push_back(std::move(l));
        }
        return spec;
    } catch (const json::exception& e) {
        throw ConfigError("bad network spec " + path + ": " + e.what());
    }
}

void save_network_spec(const NetworkSpec& spec, const std::string& path) {  // network.cpp:538-567
    json j;
    j["name"] = spec.name;
    j["input_shape"] = spec.input_shape;
    j["seed"] = spec.seed;
    j["binarize_weights"] = spec.binarize_weights;
    json layers = json::array();
    for (const LayerSpec& l : spec.layers) {
        json lj;
        lj["kind"] = to_string(l.kind);
        if (l.kind == LayerKind::Conv) {
            lj["out_channels"] = l.out_channels;
            lj["kernel_size"] = json::array({l.kernel_h, l.kernel_w});
            lj["stride"] = json::array({l.stride_h, l.stride_w});
            lj["pad"] = json::array({l.pad_h, l.pad_w});
        } else if (l.kind == LayerKind::Linear) {
            lj["out_features"] = l.out_features;
        }
        if (l.kind == LayerKind::Conv || l.kind == LayerKind::Linear) {
            lj["kernel"] = to_string(l.kernel);
            if (!l.weights_blob.empty()) lj["weights_blob"] = l.weights_blob;
        }
        if (l.seed) lj["seed"] = *l.seed;
        layers.push_back(std::move(lj));
    }
    j["layers"] = std::move(layers);
    std::ofstream os(path);
    if (!os) throw IoError("cannot open for writing: " + path);
    os << j.dump(2) << '\n';
}

}  // namespace bnn
