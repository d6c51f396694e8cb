// C++ drop-in parity tests: the reference's own unit-test cases (proj/tests/test_*.cpp),
// re-expressed against include/bnn_b200.hpp (namespace bnn, running on the B200) and checked
// against the C oracle (oracle/bnn_oracle.h, TEST INFRASTRUCTURE) or the known answers.
// Built by __graft_entry__.build(); run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <unistd.h>
#include <functional>
#include <string>

#include "bnn_b200.hpp"

extern "C" {
#include "../../oracle/bnn_oracle.h"
}

namespace {
int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++g_fail;                                                            \
        } else {                                                                 \
            ++g_pass;                                                            \
        }                                                                        \
    } while (0)

template <class E>
bool throws_with(const std::function<void()>& f, const char* needle) {
    try {
        f();
    } catch (const E& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

bnn::FloatMatrix pm1(std::size_t r, std::size_t c, std::uint64_t seed) {
    return bnn::sign(bnn::fill_random_matrix(r, c, seed));
}

// --- tensor.cpp / test_tensor.cpp
void test_tensor() {
    bnn::ConvGeometry g;
    g.kernel_h = g.kernel_w = 3, g.pad_h = g.pad_w = 1, g.in_channels = 3, g.out_channels = 8;
    CHECK(bnn::output_dims(g, 32, 32) == std::make_pair(std::size_t(32), std::size_t(32)));
    g.stride_h = 2, g.pad_h = 0;
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::output_dims(g, 32, 32); }, "height"));
    g.stride_h = 1, g.stride_w = 2, g.pad_w = 0;
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::output_dims(g, 32, 32); }, "width"));
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::FloatMatrix(0, 3); }, "rows"));
    // the device generator is bit-identical to the reference's
    std::vector<float> want(4096);
    orc_fill_random(want.size(), 77, 0, want.data());
    const auto got = bnn::fill_random_vector(4096, 77);
    CHECK(std::memcmp(got.data(), want.data(), 4096 * 4) == 0);
    CHECK(bnn::unit_random(5, 9) == orc_unit_random(5, 9));
    auto p = bnn::PackedBitMatrix::make(3, 40, bnn::PackOrientation::RowPacked);
    CHECK(p.words_per_line == 2 && p.pad_bits_per_line == 24 && p.words.size() == 6);
}

// --- binarize.cpp / test_binarize.cpp
void test_binarize() {
    bnn::FloatMatrix m(1, 3);
    m.data = {-0.3f, 0.7f, 0.0f};
    CHECK((bnn::sign(m).data == std::vector<float>{-1.0f, 1.0f, 1.0f}));
    m.data = {-0.0f, NAN, 2.5f};
    CHECK((bnn::sign(m).data == std::vector<float>{1.0f, -1.0f, 1.0f}));
    m.data = {-3.0f, 0.25f, 7.0f};
    CHECK((bnn::htanh(m).data == std::vector<float>{-1.0f, 0.25f, 1.0f}));
    bnn::FloatMatrix ones(1, 32), alt(1, 32);
    for (int j = 0; j < 32; ++j) ones.data[j] = 1.0f, alt.data[j] = (j % 2 == 0) ? 1.0f : -1.0f;
    CHECK(bnn::pack_rows(ones).words[0] == 0xFFFFFFFFu);
    CHECK(bnn::pack_rows(alt).words[0] == 0x55555555u);
    bnn::FloatMatrix col(33, 1);
    for (int r = 0; r < 33; ++r) col.data[r] = r < 32 ? 1.0f : -1.0f;
    const auto pc = bnn::pack_cols(col);
    CHECK(pc.words.size() == 2 && pc.words[0] == 0xFFFFFFFFu && pc.words[1] == 0u);
    auto bad = pm1(2, 4, 3);
    bad.at(1, 2) = 0.5f;
    CHECK(throws_with<bnn::EncodingError>([&] { bnn::pack_rows(bad); }, "(1,2)"));
    // pack_cols(M^T) == pack_rows(M), and round trips, against the oracle
    const auto w = pm1(37, 70, 11);
    bnn::FloatMatrix wt(70, 37);
    for (std::size_t i = 0; i < 37; ++i)
        for (std::size_t j = 0; j < 70; ++j) wt.at(j, i) = w.at(i, j);
    CHECK(bnn::pack_cols(wt).words == bnn::pack_rows(w).words);
    CHECK(bnn::unpack(bnn::pack_rows(w)).data == w.data);
    const auto x = bnn::fill_random_matrix(100, 29, 12);
    std::vector<std::uint32_t> want(29 * 4);
    std::size_t br = 0, bc = 0;
    orc_pack(x.data.data(), 100, 29, 1, 1, want.data(), &br, &bc);
    CHECK(bnn::sign_pack_cols(x).words == want);
}

// --- kernels.cpp / test_kernels.cpp + acceptance.cpp:61-79
void test_gemm() {
    const std::size_t Ls[] = {1, 31, 32, 33, 40, 64, 96, 100, 576, 9216};
    for (std::size_t L : Ls) {
        const std::size_t M = 1 + L % 17, N = 3 + L % 13;
        const auto pw = bnn::pack_rows(pm1(M, L, 100 + L));
        const auto px = bnn::pack_cols(pm1(L, N, 200 + L));
        const auto got = bnn::xnor_gemm(pw, px, L);
        std::vector<std::int32_t> want(M * N);
        orc_xnor_gemm(pw.words.data(), M, px.words.data(), N, L, want.data());
        CHECK(got.data == want);
        bool range = true;
        for (auto v : got.data) range = range && std::abs(v) <= int(L) && ((v - int(L)) % 2 == 0);
        CHECK(range);
    }
    const auto a = bnn::pack_rows(pm1(4, 40, 1));
    const auto b = bnn::pack_cols(pm1(33, 5, 2));
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::xnor_gemm(a, b, 40); }, "inner extents"));
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::xnor_gemm(b, b, 33); }, "row-packed"));
    // to_float + bias_add
    bnn::IntMatrix im(2, 3);
    im.data = {1, -3, 5, 7, 0, -9};
    const float bias[2] = {0.5f, -1.25f};
    const auto f = bnn::bias_add(bnn::to_float(im), bias);
    CHECK((f.data == std::vector<float>{1.5f, -2.5f, 5.5f, 5.75f, -1.25f, -10.25f}));
}

// --- network.cpp layer forwards / test_network.cpp
void test_layers() {
    bnn::ConvGeometry g;
    g.kernel_h = g.kernel_w = 3, g.pad_h = g.pad_w = 1, g.in_channels = 3, g.out_channels = 5;
    const auto x = bnn::fill_random(2, 3, 7, 9, 21);
    const auto pw = bnn::sign_pack_rows(bnn::fill_random_matrix(5, 27, 22));
    const auto bias = bnn::fill_random_vector(5, 23);
    const auto y = bnn::conv_forward_binary(x, pw, bias, g);
    std::vector<float> want(y.size());
    const std::uint64_t gg[8] = {3, 3, 1, 1, 1, 1, 3, 5};
    orc_conv_forward_binary(x.data.data(), 2, 3, 7, 9, pw.words.data(), bias.data(), gg, want.data());
    CHECK(y.data == want);
    // all-ones input and weights: every output = 27 + bias (test_network.cpp:64-76)
    bnn::FloatTensor ones(1, 3, 4, 4);
    for (auto& v : ones.data) v = 1.0f;
    bnn::FloatMatrix wones(5, 27);
    for (auto& v : wones.data) v = 1.0f;
    const std::vector<float> zero(5, 0.0f);
    bnn::ConvGeometry g0 = g;
    g0.pad_h = g0.pad_w = 0;
    const auto y1 = bnn::conv_forward_binary(ones, bnn::pack_rows(wones), zero, g0);
    bool all27 = true;
    for (float v : y1.data) all27 = all27 && v == 27.0f;
    CHECK(all27);
    // linear, L = 33 (pad correction), binary == float on +-1 operands
    const auto xin = pm1(33, 6, 31);
    const auto w = pm1(4, 33, 32);
    const auto lb = bnn::fill_random_vector(4, 33);
    const auto lo = bnn::linear_forward(xin, w, lb, bnn::KernelChoice::Binary);
    bool ok = true;
    for (std::size_t i = 0; i < 4; ++i)
        for (std::size_t j = 0; j < 6; ++j) {
            float acc = 0.0f;
            for (std::size_t k = 0; k < 33; ++k) acc += w.at(i, k) * xin.at(k, j);
            ok = ok && lo.at(i, j) == acc + lb[i];
        }
    CHECK(ok);
    CHECK(throws_with<bnn::ConfigError>([&] { bnn::linear_forward(xin, w, lb, bnn::KernelChoice::Float); },
                                        "Binary"));
    // glue
    const auto t = bnn::fill_random(2, 3, 4, 6, 41);
    std::vector<float> mp(2 * 3 * 2 * 3);
    orc_maxpool2(t.data.data(), 2, 3, 4, 6, mp.data());
    CHECK(bnn::maxpool2(t).data == mp);
    const auto sc = bnn::fill_random_vector(3, 42), sh = bnn::fill_random_vector(3, 43);
    std::vector<float> af(t.size());
    orc_affine_tensor(t.data.data(), 2, 3, 24, sc.data(), sh.data(), af.data());
    CHECK(bnn::affine_norm(t, sc, sh).data == af);
    const auto cols = bnn::flatten_to_columns(t);
    CHECK(cols.rows == 72 && cols.cols == 2 && cols.at(5, 1) == t.data[72 + 5]);
}

// --- whole network (network.cpp:330-420) vs the oracle, FNV-1a of the logits
void test_network() {
    auto spec = bnn::build_default_network(bnn::KernelChoice::Binary, 1);
    bnn::DeviceNetwork net(spec);
    const auto x = bnn::fill_random(3, 3, 32, 32, bnn::mix64(1, 0x696E707574ull));
    const auto logits = bnn::network_forward(net, x);
    orc_layer_spec layers[64];
    const std::size_t n = orc_default_spec(layers, 64);
    void* on = orc_net_build(layers, n, 3, 32, 32, 1, 0);
    std::vector<float> want(10 * 3);
    orc_net_forward(on, x.data.data(), 3, want.data());
    orc_net_free(on);
    CHECK(logits.rows == 10 && logits.cols == 3);
    CHECK(logits.data == want);
    CHECK(bnn::fnv1a_hash(logits.data) == orc_fnv1a(want.data(), want.size()));
    const auto wrong = bnn::fill_random(1, 3, 16, 16, 1);
    CHECK(throws_with<bnn::ShapeError>([&] { net.forward(wrong); }, "network expects"));
}
void test_io() {  // on-disk formats: round trips and the reference's IoError messages
    const std::string dir = "/tmp/bnn_cpp_io_" + std::to_string(::getpid());
    std::system(("mkdir -p " + dir).c_str());
    bnn::FloatMatrix w = bnn::fill_random_matrix(5, 40, 3);
    const auto p = bnn::sign_pack_rows(w);
    bnn::save_packed_blob(p, dir + "/w.pbm");
    const auto q = bnn::load_packed_blob(dir + "/w.pbm");
    CHECK(q.logical_rows == 5 && q.logical_cols == 40 && q.orientation == p.orientation && q.words == p.words);
    const auto t = bnn::fill_random(2, 3, 4, 5, 9);
    bnn::save_tensor_blob(t, dir + "/t.tb");
    const auto u = bnn::load_tensor_blob(dir + "/t.tb");
    CHECK(u.batch == 2 && u.channels == 3 && u.height == 4 && u.width == 5 && u.data == t.data);
    CHECK(throws_with<bnn::IoError>([&] { bnn::load_tensor_blob(dir + "/missing.tb"); }, "cannot open for reading"));
    std::system(("rm -rf " + dir).c_str());
}
}  // namespace

int main() {
    const std::pair<const char*, void (*)()> suites[] = {{"tensor", test_tensor},   {"binarize", test_binarize},
                                                        {"gemm", test_gemm},       {"layers", test_layers},
                                                        {"network", test_network}, {"io", test_io}};
    for (const auto& [name, fn] : suites) {
        try {
            fn();
        } catch (const std::exception& e) {
            std::fprintf(stderr, "FAIL suite %s threw: %s\n", name, e.what());
            ++g_fail;
        }
    }
    std::printf("cpp api: %d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
