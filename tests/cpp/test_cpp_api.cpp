// C++ drop-in parity tests: the reference's own unit-test cases (proj/tests/test_*.cpp),
// re-expressed against include/bnn_b200.hpp (namespace bnn, running on the B200) and checked
// against the C oracle (oracle/bnn_oracle.h, TEST INFRASTRUCTURE) or the known answers.
// Built by __graft_entry__.build(); run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
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
std::string g_root = ".";  // repository root (argv[1]): the spec fixtures live in tests/golden
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
    // linear_forward(Float): float_gemm (k-ascending FMA chain, kernels.cpp:33-51) + bias
    const auto lf = bnn::linear_forward(xin, w, lb, bnn::KernelChoice::Float);
    bool okf = true;
    for (std::size_t i = 0; i < 4; ++i)
        for (std::size_t j = 0; j < 6; ++j) {
            float acc = 0.0f;
            for (std::size_t k = 0; k < 33; ++k) acc = std::fma(w.at(i, k), xin.at(k, j), acc);
            okf = okf && lf.at(i, j) == acc + lb[i];
        }
    CHECK(okf);
    CHECK(bnn::linear_forward_binary_reference(xin, w, lb).data == lo.data);
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

// --- kernels.hpp word primitives, float_gemm, naive_conv (test_kernels.cpp:11-102)
void test_kernels_extra() {
    std::mt19937 rng(7);
    bool pc = true;
    for (int i = 0; i < 4096; ++i) {
        const std::uint32_t v = rng();
        int bits = 0;
        for (int b = 0; b < 32; ++b) bits += (v >> b) & 1u;
        pc = pc && bnn::popcount32(v) == bits && bnn::popcount32_portable(v) == bits;
    }
    CHECK(pc);
    CHECK(bnn::word_dot(0xF0F0F0F0u, 0xFF00FF00u) == 0);
    CHECK(bnn::word_dot(0u, 0u) == 32 && bnn::word_dot(0xFFFFFFFFu, 0u) == -32);
    const auto w = bnn::fill_random_matrix(7, 45, 51), x = bnn::fill_random_matrix(45, 13, 52);
    const auto y = bnn::float_gemm(w, x);
    bool ok = y.rows == 7 && y.cols == 13;
    for (std::size_t i = 0; i < 7; ++i)
        for (std::size_t j = 0; j < 13; ++j) {
            float acc = 0.0f;
            for (std::size_t k = 0; k < 45; ++k) acc = std::fma(w.at(i, k), x.at(k, j), acc);
            ok = ok && y.at(i, j) == acc;
        }
    CHECK(ok);
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::float_gemm(w, w); }, "inner extents differ"));
    // naive_conv (kernels.cpp:109-147): kh, kw, c loop order, out-of-image taps skipped
    bnn::ConvGeometry g;
    g.kernel_h = 3, g.kernel_w = 2, g.stride_h = 2, g.pad_h = g.pad_w = 1, g.in_channels = 4, g.out_channels = 3;
    const auto xt = bnn::fill_random(2, 4, 7, 6, 53);
    const auto wt = bnn::fill_random(3, 4, 3, 2, 54);
    const auto yt = bnn::naive_conv(xt, 1, wt, g);
    const auto [oh, ow] = bnn::output_dims(g, 7, 6);
    bool okn = yt.batch == 1 && yt.channels == 3 && yt.height == oh && yt.width == ow;
    for (std::size_t d = 0; d < 3; ++d)
        for (std::size_t a = 0; a < oh; ++a)
            for (std::size_t b = 0; b < ow; ++b) {
                float acc = 0.0f;
                for (std::size_t kh = 0; kh < 3; ++kh) {
                    const long ih = long(a * 2 + kh) - 1;
                    if (ih < 0 || ih >= 7) continue;
                    for (std::size_t kw = 0; kw < 2; ++kw) {
                        const long iw = long(b + kw) - 1;
                        if (iw < 0 || iw >= 6) continue;
                        for (std::size_t c = 0; c < 4; ++c) acc = std::fma(wt.at(d, c, kh, kw), xt.at(1, c, ih, iw), acc);
                    }
                }
                okn = okn && yt.at(0, d, a, b) == acc;
            }
    CHECK(okn);
}

// --- lowering.hpp: im2col / col2im (test_lowering.cpp:55-102)
void test_lowering() {
    bnn::FloatTensor x(1, 1, 3, 3);
    for (int i = 0; i < 9; ++i) x.data[i] = float(i + 1);
    bnn::ConvGeometry g;
    g.kernel_h = g.kernel_w = 2;
    const auto m = bnn::im2col(x, 0, g);
    CHECK(m.rows == 4 && m.cols == 4);
    // columns [1,2,4,5], [2,3,5,6], [4,5,7,8], [5,6,8,9]
    CHECK((std::vector<float>{m.at(0, 0), m.at(1, 0), m.at(2, 0), m.at(3, 0)} == std::vector<float>{1, 2, 4, 5}));
    CHECK((std::vector<float>{m.at(0, 3), m.at(1, 3), m.at(2, 3), m.at(3, 3)} == std::vector<float>{5, 6, 8, 9}));
    bnn::ConvGeometry g2;
    g2.kernel_h = 3, g2.kernel_w = 3, g2.stride_h = 2, g2.stride_w = 1, g2.pad_h = 1, g2.pad_w = 1, g2.in_channels = 5;
    const auto xt = bnn::fill_random(3, 5, 9, 7, 61);
    const auto mt = bnn::im2col(xt, 2, g2);
    std::vector<float> want(mt.data.size());
    const std::uint64_t gg[8] = {3, 3, 2, 1, 1, 1, 5, 1};
    orc_im2col(xt.data.data(), 3, 5, 9, 7, 2, gg, want.data());
    CHECK(mt.data == want);
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::im2col(xt, 3, g2); }, "out of range"));
    // col2im: the reference's scatter order, reproduced on the host here
    const auto [oh, ow] = bnn::output_dims(g2, 9, 7);
    const auto cm = bnn::fill_random_matrix(45, oh * ow, 62);
    const auto back = bnn::col2im(cm, g2, oh, ow);
    bnn::FloatTensor ref(1, 5, 9, 7);
    for (std::size_t c = 0; c < 5; ++c)
        for (std::size_t kh = 0; kh < 3; ++kh)
            for (std::size_t kw = 0; kw < 3; ++kw)
                for (std::size_t a = 0; a < oh; ++a)
                    for (std::size_t b = 0; b < ow; ++b) {
                        const long ih = long(a * 2 + kh) - 1, iw = long(b + kw) - 1;
                        if (ih < 0 || ih >= 9 || iw < 0 || iw >= 7) continue;
                        ref.at(0, c, ih, iw) += cm.at((c * 3 + kh) * 3 + kw, a * ow + b);
                    }
    CHECK(back.height == 9 && back.width == 7 && back.data == ref.data);
}

// --- the reference's call chains through namespace bnn
void test_network() {
    // (1) bnnbench bench: build_default_network -> build_network -> make_input -> network_forward
    const bnn::NetworkSpec spec = bnn::build_default_network(bnn::KernelChoice::Binary, 1);
    const bnn::Network net = bnn::build_network(spec);
    const bnn::FloatTensor input =
        bnn::fill_random(3, net.in_channels, net.in_h, net.in_w, bnn::mix64(1, 0x696e707574));
    std::vector<double> layer_seconds;
    const bnn::FloatMatrix logits =
        bnn::network_forward(net, input, bnn::ForwardOptions{bnn::ExecKernel::Binary, 1, &layer_seconds});
    orc_layer_spec layers[64];
    const std::size_t n = orc_default_spec(layers, 64);
    void* on = orc_net_build(layers, n, 3, 32, 32, 1, 0);
    std::vector<float> want(10 * 3);
    orc_net_forward(on, input.data.data(), 3, want.data());
    CHECK(logits.rows == 10 && logits.cols == 3);
    CHECK(logits.data == want);
    CHECK(bnn::fnv1a_hash(logits) == orc_fnv1a(want.data(), want.size()));
    CHECK(layer_seconds.size() == net.layers.size() && layer_seconds[0] > 0.0);
    CHECK(net.layers.size() == n && net.logits == 10 && net.parameter_count > 14000000);
    // the host mirror holds the reference's parameters
    std::vector<std::uint32_t> pw(net.layers[0].packed_weights.words.size());
    std::vector<float> pb(128), ps(128), psh(128);
    orc_net_layer_params(on, 0, pw.data(), pb.data(), nullptr, nullptr);
    CHECK(net.layers[0].packed_weights.words == pw && net.layers[0].bias == pb);
    orc_net_layer_params(on, 1, nullptr, nullptr, ps.data(), psh.data());
    CHECK(net.layers[1].scale == ps && net.layers[1].shift == psh);
    orc_net_free(on);
    // the other ExecKernels: BinaryReference equals Binary exactly here (+-1 float GEMMs are exact)
    const auto lref = bnn::network_forward(net, input, bnn::ForwardOptions{bnn::ExecKernel::BinaryReference});
    CHECK(lref.data == logits.data);
    const auto lper = bnn::network_forward(net, input);  // PerLayer: every layer Binary
    CHECK(lper.data == logits.data);
    const auto wrong = bnn::fill_random(1, 3, 16, 16, 1);
    CHECK(throws_with<bnn::ShapeError>([&] { bnn::network_forward(net, wrong); }, "network expects"));
    // the owning device handle
    bnn::DeviceNetwork dnet(spec);
    CHECK(bnn::network_forward(dnet, input).data == logits.data);
}

// --- bench.hpp: verify + corrupted-bit hook (test_bench.cpp:150-173), reports, spec JSON
void test_harness() {
    const std::string tiny = g_root + "/tests/golden/tiny_spec.json";
    bnn::BenchConfig cfg;
    cfg.spec_path = tiny;
    cfg.batch = 4;
    const bnn::VerifySummary s = bnn::run_verify(cfg);
    CHECK(s.pass && s.max_abs_deviation <= 1e-4 && s.pad_correction_exercised);
    bnn::NetworkSpec spec = bnn::load_network_spec(tiny);
    spec.binarize_weights = true;
    bnn::Network net = bnn::build_network(spec);
    const bnn::FloatTensor input = bnn::fill_random(4, net.in_channels, net.in_h, net.in_w, 9);
    CHECK(bnn::verify_network(net, input).pass);
    bnn::BuiltLayer& last = net.layers.back();
    CHECK(last.spec.kind == bnn::LayerKind::Linear);
    last.packed_weights.words[0] ^= 1u;  // flip one real (non-pad) bit in the logits layer
    const bnn::VerifySummary bad = bnn::verify_network(net, input);
    CHECK(!bad.pass && bad.max_abs_deviation >= 1.9);
    last.packed_weights.words[0] ^= 1u;  // restored: the engine follows the host copy again
    CHECK(bnn::verify_network(net, input).pass);
    // spec JSON round trip and the reference's error texts
    const std::string dir = "/tmp/bnn_cpp_h_" + std::to_string(::getpid());
    std::system(("mkdir -p " + dir).c_str());
    bnn::save_network_spec(spec, dir + "/s.json");
    CHECK(bnn::load_network_spec(dir + "/s.json") == spec);
    {
        std::FILE* f = std::fopen((dir + "/bad.json").c_str(), "w");
        std::fputs("{\"kernel\": \"fast\", \"layers\": []}", f);
        std::fclose(f);
    }
    CHECK(throws_with<bnn::ConfigError>([&] { bnn::load_network_spec(dir + "/bad.json"); }, "unknown kernel choice 'fast'"));
    {
        std::FILE* f = std::fopen((dir + "/pair.json").c_str(), "w");
        std::fputs("{\"layers\": [{\"kind\": \"conv\", \"out_channels\": 4, \"kernel_size\": [3, 3, 3]}]}", f);
        std::fclose(f);
    }
    CHECK(throws_with<bnn::ConfigError>([&] { bnn::load_network_spec(dir + "/pair.json"); },
                                        "kernel_size must be a scalar or [h, w]"));
    // run_benchmark -> emit_report -> parse_report round trip, and the text summary
    bnn::BenchConfig bc;
    bc.spec_path = tiny;
    bc.batch = 4;
    bc.iterations = 3;
    bc.warmup = 1;
    const bnn::BenchReport r = bnn::run_benchmark(bc);
    CHECK(r.kernels.size() == 2 && r.kernels[0].samples_s.size() == 3 && r.speedups.size() == 1);
    bnn::emit_report(r, dir + "/r.json");
    const bnn::BenchReport p = bnn::parse_report(dir + "/r.json");
    CHECK(p.network_name == r.network_name && p.kernels.size() == 2 &&
          p.kernels[0].logits_hash == r.kernels[0].logits_hash && p.total_packed_bytes == r.total_packed_bytes);
    std::ostringstream os;
    bnn::print_report(r, os);
    CHECK(os.str().find("speedup float/binary") != std::string::npos && os.str().find("packed/float") != std::string::npos);
    CHECK(bnn::median({3.0, 1.0, 2.0}) == 2.0 && bnn::median({4.0, 1.0, 2.0, 3.0}) == 2.5);
    std::system(("rm -rf " + dir).c_str());
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

int main(int argc, char** argv) {
    if (argc > 1) g_root = argv[1];
    const std::pair<const char*, void (*)()> suites[] = {
        {"tensor", test_tensor},   {"binarize", test_binarize}, {"gemm", test_gemm},
        {"kernels", test_kernels_extra}, {"lowering", test_lowering}, {"layers", test_layers},
        {"network", test_network}, {"harness", test_harness},   {"io", test_io}};
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
