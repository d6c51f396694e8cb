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

// kernel_size / stride / pad: a number or a [h, w] pair (network.cpp pair_field)
std::pair<uint64_t, uint64_t> pair_field(const json& lj, const char* key, uint64_t dflt) {
    if (!lj.contains(key)) return {dflt, dflt};
    const json& v = lj.at(key);
    if (v.is_array()) {
        if (v.size() != 2) throw std::runtime_error(std::string(key) + " must be a number or a pair");
        return {v[0].get<uint64_t>(), v[1].get<uint64_t>()};
    }
    const uint64_t s = v.get<uint64_t>();
    return {s, s};
}

struct ParsedSpec {
    std::string name;
    uint64_t shape[4] = {1, 3, 32, 32};
    uint64_t seed = 1;
    int binarize = 0;
    std::vector<bnn_layer_spec> layers;
    std::vector<std::string> blobs;  // per layer ("" = seeded weights)
};

int parse_spec(const char* path, ParsedSpec& out) {
    std::ifstream is(path);
    if (!is) return bnnk::fail(BNN_E_CONFIG, std::string("cannot open network spec: ") + path);
    json j;
    try {
        j = json::parse(is);
    } catch (const json::parse_error& e) {
        return bnnk::fail(BNN_E_CONFIG, std::string("parse error in ") + path + ": " + e.what());
    }
    try {
        out.name = j.value("name", std::string("unnamed"));
        if (j.contains("input_shape")) {
            const json& s = j.at("input_shape");
            if (!s.is_array() || s.size() != 4)
                return bnnk::fail(BNN_E_CONFIG, "input_shape must be [batch, channels, height, width]");
            for (int i = 0; i < 4; ++i) out.shape[i] = s[i].get<uint64_t>();
        }
        out.seed = j.value("seed", uint64_t{1});
        out.binarize = j.value("binarize_weights", false) ? 1 : 0;
        if (!j.contains("layers") || !j.at("layers").is_array())
            return bnnk::fail(BNN_E_CONFIG, "spec needs a 'layers' array");
        static const char* kinds[] = {"conv", "linear", "maxpool", "affine_norm", "sign", "htanh"};
        for (const json& lj : j.at("layers")) {
            bnn_layer_spec l{};
            l.stride_h = l.stride_w = 1;
            const std::string k = lj.at("kind").get<std::string>();
            int kind = -1;
            for (int i = 0; i < 6; ++i)
                if (k == kinds[i]) kind = i;
            if (kind < 0) return bnnk::fail(BNN_E_CONFIG, "unknown layer kind '" + k + "'");
            l.kind = uint32_t(kind);
            if (kind == BNN_LAYER_CONV) {
                l.out_channels = lj.at("out_channels").get<uint64_t>();
                std::tie(l.kernel_h, l.kernel_w) = pair_field(lj, "kernel_size", 0);
                if (l.kernel_h == 0) return bnnk::fail(BNN_E_CONFIG, "conv layer needs kernel_size");
                std::tie(l.stride_h, l.stride_w) = pair_field(lj, "stride", 1);
                std::tie(l.pad_h, l.pad_w) = pair_field(lj, "pad", 0);
            } else if (kind == BNN_LAYER_LINEAR) {
                l.out_features = lj.at("out_features").get<uint64_t>();
            }
            std::string blob;
            if (kind == BNN_LAYER_CONV || kind == BNN_LAYER_LINEAR) blob = lj.value("weights_blob", std::string{});
            if (lj.contains("seed")) l.has_seed = 1, l.seed = lj.at("seed").get<uint64_t>();
            out.layers.push_back(l);
            out.blobs.push_back(blob);
        }
    } catch (const std::exception& e) {
        return bnnk::fail(BNN_E_CONFIG, std::string("bad network spec ") + path + ": " + e.what());
    }
    return BNN_OK;
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
    for (size_t i = 0; i < sp.layers.size(); ++i) sp.layers[i].weights_blob = sp.blobs[i].empty() ? nullptr : sp.blobs[i].c_str();
    const int bin = binarize_override >= 0 ? binarize_override : sp.binarize;
    return bnn_net_create(sp.layers.data(), sp.layers.size(), sp.shape[1], sp.shape[2], sp.shape[3], sp.seed, bin, out);
}

// Spec header for callers that build their own inputs: input_shape and layer count.
int bnn_spec_info(const char* path, uint64_t input_shape[4], size_t* n_layers) {
    ParsedSpec sp;
    if (int rc = parse_spec(path, sp)) return rc;
    for (int i = 0; i < 4; ++i) input_shape[i] = sp.shape[i];
    if (n_layers) *n_layers = sp.layers.size();
    return BNN_OK;
}

}  // extern "C"
