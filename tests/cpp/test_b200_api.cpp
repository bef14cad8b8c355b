// The C++ host API (include/ouro_b200.hpp) against the reference's own
// implementation of the same operators, linked from the reference sources
// compiled in place (oracle/_ref objects): the cases read like the reference's
// test_gemm.cpp / test_quant.cpp, with the expected values produced by ouro::.
// Test infrastructure only; built by `make -C oracle cpp-api-test` (needs the
// reference headers) and run on a GPU by tests/test_gpu_cpp_api.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <cstring>
#include <random>

#include "ouro/gemm.hpp"
#include "ouro/quant.hpp"
#include "ouro/rng.hpp"
#include "ouro/ssm.hpp"
#include "ouro_b200.hpp"

namespace {

struct Plane {
    std::vector<int8_t> codes;
    size_t rows, cols;
};

Plane random_codes(std::mt19937& g, size_t rows, size_t cols, int lim) {
    std::uniform_int_distribution<int> d(-lim, lim);
    Plane p{std::vector<int8_t>(rows * cols), rows, cols};
    for (auto& v : p.codes) v = static_cast<int8_t>(d(g));
    return p;
}

template <class P>
P to_packed(const Plane& p);
template <>
ouro::PackedInt4 to_packed<ouro::PackedInt4>(const Plane& p) {
    return ouro::pack_int4(p.codes.data(), p.rows, p.cols);
}
template <>
ouro_b200::PackedInt4 to_packed<ouro_b200::PackedInt4>(const Plane& p) {
    return ouro_b200::pack_int4(p.codes.data(), p.rows, p.cols);
}

struct Outliers {
    std::vector<size_t> channels;
    std::vector<int8_t> codes;
    std::vector<double> scales;
};

Outliers random_outliers(std::mt19937& g, size_t k, size_t c, size_t n_o) {
    std::vector<size_t> all(k);
    for (size_t i = 0; i < k; ++i) all[i] = i;
    std::shuffle(all.begin(), all.end(), g);
    Outliers o;
    o.channels.assign(all.begin(), all.begin() + static_cast<std::ptrdiff_t>(n_o));
    std::sort(o.channels.begin(), o.channels.end());
    std::uniform_int_distribution<int> d(-127, 127);
    std::uniform_real_distribution<double> s(0.005, 0.02);
    o.codes.resize(n_o * c);
    for (auto& v : o.codes) v = static_cast<int8_t>(d(g));
    for (size_t j = 0; j < n_o; ++j) o.scales.push_back(s(g));
    return o;
}

template <class B>
B to_buffer(const Outliers& o, size_t c) {
    B b;
    b.channels = o.channels;
    b.codes = o.codes;
    b.scales = o.scales;
    b.cols = c;
    return b;
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

double rel_err(const std::vector<double>& a, const std::vector<double>& b) {
    double num = 0.0, den = 1e-300;
    for (size_t i = 0; i < a.size(); ++i) {
        num = std::max(num, std::fabs(a[i] - b[i]));
        den = std::max(den, std::fabs(b[i]));
    }
    return num / den;
}

ouro::ModelDims ref_dims() {
    ouro::ModelDims d;
    d.image = 32;
    d.channels = 3;
    d.patch = 8;
    d.embed = 64;
    d.state = 16;
    d.blocks = 2;
    d.classes = 10;
    d.conv_width = 4;
    return d;
}

ouro_b200::ModelDims gpu_dims() {
    ouro_b200::ModelDims d;
    d.image = 32;
    d.channels = 3;
    d.patch = 8;
    d.embed = 64;
    d.state = 16;
    d.blocks = 2;
    d.classes = 10;
    d.conv_width = 4;
    return d;
}

std::vector<double> images(uint64_t seed, size_t batch) {
    ouro::SeededRng rng(seed);
    std::vector<double> v(batch * 32 * 32 * 3);
    for (double& x : v) x = rng.normal();
    return v;
}

ouro_b200::CalibrationResult to_gpu(const ouro::CalibrationResult& c) {
    ouro_b200::CalibrationResult g;
    g.spec.weight_bits = c.spec.weight_bits;
    g.spec.act_bits = c.spec.act_bits;
    g.spec.outlier_bits = c.spec.outlier_bits;
    g.spec.n_refresh = c.spec.n_refresh;
    g.spec.rho = c.spec.rho;
    g.tokens = c.tokens;
    g.embed = c.embed;
    g.state = c.state;
    g.blocks = c.blocks;
    g.ndirs = c.ndirs;
    for (const auto& t : c.tensors)
        g.tensors.push_back({t.name, t.theta, t.scale_inlier, t.scale_full, t.excluded});
    return g;
}

}  // namespace

TEST_CASE("hybrid_gemm == reference hybrid_gemm, bit for bit (planes and output)") {
    std::mt19937 g(11);
    const size_t shapes[][4] = {{5, 7, 3, 0}, {64, 96, 40, 3}, {33, 129, 77, 9}, {200, 768, 300, 20}, {1, 16, 1, 1}};
    for (const auto& sh : shapes) {
        const size_t m = sh[0], k = sh[1], c = sh[2], n_o = sh[3];
        Plane w = random_codes(g, m, k, 7), x = random_codes(g, k, c, 7);
        Outliers o = random_outliers(g, k, c, n_o);
        std::uniform_real_distribution<double> s(0.005, 0.02);
        std::vector<double> ws(m);
        for (double& v : ws) v = s(g);
        for (bool f16 : {false, true}) {
            ouro::GemmResult want = ouro::hybrid_gemm(to_packed<ouro::PackedInt4>(w), ws, to_packed<ouro::PackedInt4>(x),
                                                      0.0123, to_buffer<ouro::OutlierBuffer>(o, c), 1, f16);
            ouro_b200::GemmResult got =
                ouro_b200::hybrid_gemm(to_packed<ouro_b200::PackedInt4>(w), ws, to_packed<ouro_b200::PackedInt4>(x),
                                       0.0123, to_buffer<ouro_b200::OutlierBuffer>(o, c), 1, f16);
            CHECK(got.rows == want.rows);
            CHECK(got.cols == want.cols);
            CHECK(got.acc_inlier == want.acc_inlier);
            CHECK(got.acc_outlier == want.acc_outlier);
            CHECK(same_bits(got.output, want.output));
        }
    }
}

TEST_CASE("gemm_i4 and gemm_i4xi8 == reference") {
    std::mt19937 g(12);
    Plane w = random_codes(g, 48, 80, 7), x = random_codes(g, 80, 33, 7);
    Outliers o = random_outliers(g, 80, 33, 6);
    CHECK(ouro_b200::gemm_i4(to_packed<ouro_b200::PackedInt4>(w), to_packed<ouro_b200::PackedInt4>(x)) ==
          ouro::gemm_i4(to_packed<ouro::PackedInt4>(w), to_packed<ouro::PackedInt4>(x)));
    CHECK(ouro_b200::gemm_i4xi8(to_packed<ouro_b200::PackedInt4>(w), to_buffer<ouro_b200::OutlierBuffer>(o, 33)) ==
          ouro::gemm_i4xi8(to_packed<ouro::PackedInt4>(w), to_buffer<ouro::OutlierBuffer>(o, 33)));
}

TEST_CASE("pack_int4 layout and validation match the reference") {
    std::mt19937 g(13);
    Plane p = random_codes(g, 9, 13, 7);
    ouro::PackedInt4 a = to_packed<ouro::PackedInt4>(p);
    ouro_b200::PackedInt4 b = to_packed<ouro_b200::PackedInt4>(p);
    CHECK(a.bytes == b.bytes);
    CHECK(a.stride == b.stride);
    CHECK(ouro_b200::unpack_int4(b) == ouro::unpack_int4(a));
    const int8_t bad[2] = {3, 8};
    CHECK_THROWS_AS(ouro_b200::pack_int4(bad, 1, 2), ouro_b200::ValidationError);
    std::vector<double> one{1.0};
    Plane w = random_codes(g, 2, 4, 7), x = random_codes(g, 4, 3, 7);
    CHECK_THROWS_AS(ouro_b200::hybrid_gemm(to_packed<ouro_b200::PackedInt4>(w), one, to_packed<ouro_b200::PackedInt4>(x),
                                           1.0, ouro_b200::OutlierBuffer{}),
                    ouro_b200::ValidationError);  // one scale per output row
    Plane x5 = random_codes(g, 5, 3, 7);
    CHECK_THROWS_AS(ouro_b200::gemm_i4(to_packed<ouro_b200::PackedInt4>(w), to_packed<ouro_b200::PackedInt4>(x5)),
                    ouro_b200::ValidationError);  // inner dimensions disagree
}

TEST_CASE("round_f16 == reference round_f16") {
    const double vals[] = {0.0, -0.0, 1.0, 1.0 + 1e-4, 65504.0, 65519.0, 65520.0, -70000.0, 6e-8, 3e-8, 1e-9, 0.1};
    for (double v : vals) {
        const double a = ouro::round_f16(v), b = ouro_b200::round_f16(v);
        CHECK(std::memcmp(&a, &b, sizeof a) == 0);
    }
}

TEST_CASE("calibrate on the GPU == reference calibrate") {
    ouro::ToyVmmModel rm = ouro::make_toy_model(ref_dims(), {ouro::ScanOrder::RowForward, ouro::ScanOrder::RowBackward}, 7);
    auto gm = ouro_b200::make_toy_model(
        gpu_dims(), {ouro_b200::ScanOrder::RowForward, ouro_b200::ScanOrder::RowBackward}, 7);
    const std::vector<double> img = images(21, 3);
    ouro::QuantSpec rs;
    rs.act_bits = 4;
    rs.n_refresh = 4;
    rs.rho = 0.05;
    ouro_b200::QuantSpec gs;
    gs.act_bits = 4;
    gs.n_refresh = 4;
    gs.rho = 0.05;
    ouro::CalibrationResult want = ouro::calibrate(rm, img, 3, rs);
    ouro_b200::CalibrationResult got = ouro_b200::calibrate(*gm, img, 3, gs);
    REQUIRE(got.tensors.size() == want.tensors.size());
    for (size_t i = 0; i < want.tensors.size(); ++i) {
        CHECK(got.tensors[i].name == want.tensors[i].name);
        // peaks and thresholds of bit-identical activations: bit-identical
        CHECK(std::memcmp(&got.tensors[i].theta, &want.tensors[i].theta, sizeof(double)) == 0);
        CHECK(same_bits(got.tensors[i].scale_inlier, want.tensors[i].scale_inlier));
        CHECK(same_bits(got.tensors[i].scale_full, want.tensors[i].scale_full));
        CHECK(got.tensors[i].excluded == want.tensors[i].excluded);
    }
}

TEST_CASE("quantized_forward on the GPU == reference quantized_forward (logits and metrics)") {
    ouro::ToyVmmModel rm = ouro::make_toy_model(ref_dims(), {ouro::ScanOrder::RowForward, ouro::ScanOrder::RowBackward}, 9);
    auto gm = ouro_b200::make_toy_model(
        gpu_dims(), {ouro_b200::ScanOrder::RowForward, ouro_b200::ScanOrder::RowBackward}, 9);
    ouro::QuantSpec rs;
    rs.act_bits = 4;
    rs.n_refresh = 5;
    rs.rho = 0.05;
    const ouro::CalibrationResult cal = ouro::calibrate(rm, images(31, 3), 3, rs);
    const std::vector<double> img = images(32, 4);
    const ouro::QuantMode rmodes[] = {ouro::QuantMode::Dynamic, ouro::QuantMode::Static, ouro::QuantMode::Bypass};
    const ouro_b200::QuantMode gmodes[] = {ouro_b200::QuantMode::Dynamic, ouro_b200::QuantMode::Static,
                                           ouro_b200::QuantMode::Bypass};
    // The device exp/log1p restate glibc's (glibc_math.cuh), so both passes equal the
    // reference's logits bit for bit; the MSEs differ only by reduction order.
    for (int i = 0; i < 3; ++i) {
        ouro::QuantEvalResult want = ouro::quantized_forward(rm, img, 4, cal, rmodes[i], ouro::SpikeSettings{});
        ouro_b200::QuantEvalResult got = ouro_b200::quantized_forward(*gm, img, 4, to_gpu(cal), gmodes[i]);
        CHECK(same_bits(got.logits_fp, want.logits_fp));
        CHECK(same_bits(got.logits_q, want.logits_q));
        CHECK(got.argmax_agree == want.argmax_agree);
        CHECK(std::fabs(got.logits_mse - want.logits_mse) <= 1e-12 * want.logits_mse + 1e-300);
        REQUIRE(got.layer_mse.size() == want.layer_mse.size());
        for (size_t l = 0; l < want.layer_mse.size(); ++l) {
            CHECK(got.layer_mse[l].first == want.layer_mse[l].first);
            CHECK(std::fabs(got.layer_mse[l].second - want.layer_mse[l].second) <=
                  1e-12 * want.layer_mse[l].second + 1e-300);
        }
    }
    // SpikeHook in every pass (FP, quantized, teacher-forced), bit for bit
    const double rates[] = {0.2, 0.5};
    const size_t chans[] = {1, 3};
    for (int j = 0; j < 2; ++j) {
        ouro::SpikeSettings rsp;
        rsp.rate = rates[j];
        rsp.gain = 50.0;
        rsp.channels = chans[j];
        rsp.salt = 11;
        ouro_b200::SpikeSettings gsp;
        gsp.rate = rates[j];
        gsp.gain = 50.0;
        gsp.channels = chans[j];
        gsp.salt = 11;
        for (int i = 0; i < 3; ++i) {
            ouro::QuantEvalResult want = ouro::quantized_forward(rm, img, 4, cal, rmodes[i], rsp);
            ouro_b200::QuantEvalResult got = ouro_b200::quantized_forward(*gm, img, 4, to_gpu(cal), gmodes[i], gsp);
            CHECK(same_bits(got.logits_fp, want.logits_fp));
            CHECK(same_bits(got.logits_q, want.logits_q));
            CHECK(got.argmax_agree == want.argmax_agree);
            REQUIRE(got.layer_mse.size() == want.layer_mse.size());
            for (size_t l = 0; l < want.layer_mse.size(); ++l)
                CHECK(std::fabs(got.layer_mse[l].second - want.layer_mse[l].second) <=
                      1e-12 * want.layer_mse[l].second + 1e-300);
        }
    }
    ouro_b200::SpikeSettings bad;
    bad.rate = 0.1;
    bad.channels = 65;
    CHECK_THROWS_AS(ouro_b200::quantized_forward(*gm, img, 4, to_gpu(cal), ouro_b200::QuantMode::Dynamic, bad),
                    ouro_b200::ValidationError);
}

TEST_CASE("bench_refresh_sweep and bench_gemm on the GPU == reference records") {
    ouro::SweepSettings rs;
    rs.steps = 120;
    rs.k = 256;
    rs.c = 16;
    rs.trials = 1;
    rs.seed = 4;
    ouro_b200::SweepSettings gs;
    gs.steps = 120;
    gs.k = 256;
    gs.c = 16;
    gs.trials = 2;
    gs.seed = 4;
    const auto want = ouro::bench_refresh_sweep(rs);
    const auto got = ouro_b200::bench_refresh_sweep(gs);
    REQUIRE(got.size() == want.size());
    for (size_t i = 0; i < want.size(); ++i) {
        CHECK(got[i].period == want[i].period);
        CHECK(got[i].mean_o_list == want[i].mean_o_list);
        CHECK(got[i].scans_per_step == want[i].scans_per_step);
        CHECK(got[i].median_total_ns > 0.0);
    }
    ouro::BenchSettings rb;
    rb.sizes = {48, 160};
    rb.trials = 1;
    ouro_b200::BenchSettings gb;
    gb.sizes = {48, 160};
    gb.trials = 2;
    const auto wb = ouro::bench_gemm(rb);
    const auto gbr = ouro_b200::bench_gemm(gb);
    REQUIRE(gbr.size() == wb.size());
    for (size_t i = 0; i < wb.size(); ++i) {
        CHECK(gbr[i].path == wb[i].path);
        CHECK(gbr[i].size == wb[i].size);
        CHECK(gbr[i].median_ns > 0.0);
    }
    gs.spike_gain = 1.0;
    CHECK_THROWS_AS(ouro_b200::bench_refresh_sweep(gs), ouro_b200::ValidationError);
}
