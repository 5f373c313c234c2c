// C++ API tests of the B200 detector, written like the reference's doctest
// suites (proj/tests/test_lls.cpp, test_hybrid_nn.cpp, test_fused.cpp) and run
// against the device through noma:: -> include/noma_cuda.h.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "noma/detector.hpp"

using namespace noma;

static int g_failed = 0, g_checks = 0;
#define CHECK(cond)                                                                   \
    do {                                                                              \
        ++g_checks;                                                                   \
        if (!(cond)) {                                                                \
            ++g_failed;                                                               \
            std::printf("  FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);              \
        }                                                                             \
    } while (0)

template <class E, class F>
static bool throws(F &&f) {
    try {
        f();
    } catch (const E &) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

struct Case {
    const char *name;
    std::function<void()> fn;
};
static std::vector<Case> &cases() {
    static std::vector<Case> c;
    return c;
}
#define TEST_CASE(NAME)                                                              \
    static void NAME();                                                              \
    static const bool reg_##NAME = (cases().push_back({#NAME, NAME}), true);         \
    static void NAME()

// Box-Muller draws of the reference Rng (rng.hpp:58-62), host-side helper
// for building seeded test inputs exactly like the reference tests do.
static double gaussian(Rng &r) {
    const double u1 = 1.0 - static_cast<double>(r.next_u64() >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(r.next_u64() >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
}

static Mat random_mat(int rows, int cols, std::uint64_t seed) {  // test_lls.cpp:13-19
    Rng rng(seed);
    Mat m(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) m(r, c) = gaussian(rng);
    return m;
}

static Vec matvec(const Mat &x, const Vec &w) {
    Vec y(x.rows());
    for (int r = 0; r < x.rows(); ++r) {
        double s = 0;
        for (int c = 0; c < x.cols(); ++c) s += x(r, c) * w[c];
        y[r] = s;
    }
    return y;
}

static CMat random_cmat(int rows, int cols, std::uint64_t seed) {
    Mat a = random_mat(rows, cols, seed), b = random_mat(rows, cols, seed + 7);
    CMat x(rows, cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) x(r, c) = cplx(a(r, c), b(r, c));
    return x;
}

TEST_CASE(lls_identity_design_returns_targets) {  // test_lls.cpp:23-30
    Mat x(2, 2);
    x(0, 0) = 1;
    x(1, 1) = 1;
    Vec y{0.3, 0.7};
    LlsWeights w = lls::fit(x, y);
    CHECK(std::abs(w.w[0] - 0.3) < 1e-14);
    CHECK(std::abs(w.w[1] - 0.7) < 1e-14);
}

TEST_CASE(lls_residual_orthogonality) {  // test_lls.cpp:89-100
    for (std::uint64_t seed = 0; seed < 5; ++seed) {
        Mat x = random_mat(200, 8, 10 + seed);
        Rng rng(20 + seed);
        Vec y(200);
        for (int i = 0; i < 200; ++i) y[i] = gaussian(rng);
        Vec w = lls::fit(x, y).w;
        Vec res = matvec(x, w);
        double lhs = 0, xm = 0, ym = 0;
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int r = 0; r < 200; ++r) s += x(r, c) * (res[r] - y[r]);
            lhs = std::max(lhs, std::abs(s));
        }
        for (int i = 0; i < x.size(); ++i) xm = std::max(xm, std::abs(x.data()[i]));
        for (int i = 0; i < 200; ++i) ym = std::max(ym, std::abs(y[i]));
        CHECK(lhs <= 1e-8 * xm * ym);
    }
}

TEST_CASE(lls_widened_design_recovers_noiseless_symbols) {  // test_lls.cpp:75-87
    CMat h = random_cmat(2, 1, 3);  // M=2 antennas, K=1 user
    CVec b(80);
    Rng rng(12);
    const double a = 1.0 / std::sqrt(2.0);
    for (int t = 0; t < 80; ++t) {
        const auto bits = rng.next_u64() >> 62;
        b[t] = cplx(bits & 1 ? -a : a, bits & 2 ? -a : a);
    }
    CMat rx(80, 2);
    for (int t = 0; t < 80; ++t)
        for (int m = 0; m < 2; ++m) rx(t, m) = b[t] * h(m, 0);
    CMat train(16, 2), data(64, 2);
    CVec yt(16);
    for (int t = 0; t < 16; ++t) {
        yt[t] = b[t];
        for (int m = 0; m < 2; ++m) train(t, m) = rx(t, m);
    }
    for (int t = 0; t < 64; ++t)
        for (int m = 0; m < 2; ++m) data(t, m) = rx(16 + t, m);
    LlsWeights w = lls::fit(widen_dataset(train, yt, 1));
    CVec pred = lls::predict(w, widen_design(data));
    double err = 0;
    for (int t = 0; t < 64; ++t) err = std::max(err, std::abs(pred[t] - b[16 + t]));
    CHECK(err < 1e-10);
}

TEST_CASE(lls_rank_deficient_min_norm_and_inconsistent_error) {  // test_lls.cpp:136-166
    Mat x(6, 4);
    for (int r = 0; r < 6; ++r) {
        x(r, 0) = 1;
        x(r, 1) = 1;
        x(r, 2) = r;
        x(r, 3) = 2.0 * r;
    }
    Vec y(6);
    for (int r = 0; r < 6; ++r) y[r] = 1.0 + 3.0 * r;
    LlsWeights w = lls::fit(x, y);
    Vec res = matvec(x, w.w);
    double e = 0;
    for (int r = 0; r < 6; ++r) e += (res[r] - y[r]) * (res[r] - y[r]);
    CHECK(std::sqrt(e) < 1e-10);
    CHECK(std::abs(w.w[0] - w.w[1]) < 1e-9);
    CHECK(std::abs(w.w[3] - 2.0 * w.w[2]) < 1e-9);
    Vec bad(6);
    bad[0] = 1.0;
    bool thrown = false;
    try {
        lls::fit(x, bad);
    } catch (const ill_conditioned_error &err) {
        thrown = err.gram_condition > 1e12;
    }
    CHECK(thrown);
}

TEST_CASE(lls_dimension_errors) {  // test_lls.cpp:168-176
    CHECK(throws<dimension_error>([] { lls::fit(Mat(4, 8), Vec(4)); }));
    LlsWeights w;
    w.w = Vec(6);
    CHECK(throws<dimension_error>([&] { lls::predict(w, Mat(2, 8)); }));
}

TEST_CASE(init_output_equals_lls_branch_and_count) {  // test_hybrid_nn.cpp:44-64
    LlsWeights w0;
    w0.w = Vec(8);
    Rng wr(17);
    for (int i = 0; i < 8; ++i) w0.w[i] = gaussian(wr);
    Rng a(9), b(9);
    HybridNetParams pa = hybrid_nn::init_params({8, 64, 64, 64}, w0, a);
    HybridNetParams pb = hybrid_nn::init_params({8, 64, 64, 64}, w0, b);
    for (std::size_t n = 0; n < pa.weights.size(); ++n) CHECK(pa.weights[n] == pb.weights[n]);
    CHECK(pa.trainable_count() == std::size_t(8 * 64 + 64 + 64 * 64 + 64 + 64 * 64 + 64 + 64));
    // the caller's Rng is advanced by exactly 2 draws per weight
    Rng c(9);
    for (int i = 0; i < 2 * (8 * 64 + 64 * 64 + 64 * 64); ++i) c.next_u64();
    CHECK(a.state[0] == c.state[0] && a.state[3] == c.state[3]);
    // first weight equals the host Box-Muller draw
    Rng d(9);
    CHECK(std::abs(pa.weights[0](0, 0) - gaussian(d) * std::sqrt(2.0 / 8)) < 1e-15);
    Mat x = random_mat(32, 8, 5);
    Vec y = hybrid_nn::forward(pa, x), lin = matvec(x, w0.w);
    double e = 0, s = 1;
    for (int r = 0; r < 32; ++r) {
        e = std::max(e, std::abs(y[r] - lin[r]));
        s = std::max(s, std::abs(lin[r]));
    }
    CHECK(e / s < 1e-5);  // FP32 device inference tolerance (test_fused.cpp:128-130)
}

TEST_CASE(train_determinism_frozen_w0_and_trace) {  // test_hybrid_nn.cpp:229-311
    CMat rx = random_cmat(128, 4, 101);
    CVec y(128);
    for (int t = 0; t < 128; ++t) y[t] = cplx(rx(t, 0).real() > 0 ? 0.7 : -0.7, rx(t, 1).imag() > 0 ? 0.7 : -0.7);
    WidenedDataset ds = widen_dataset(rx, y, 1);
    LlsWeights w0 = lls::fit(ds);
    Rng ra(112), rb(112);
    HybridNetParams pa = hybrid_nn::init_params({8, 16, 16}, w0, ra);
    HybridNetParams pb = hybrid_nn::init_params({8, 16, 16}, w0, rb);
    TrainConfig tc;
    tc.epochs = 0;
    CHECK(hybrid_nn::train(pa, ds, tc).empty());
    tc.epochs = 6;
    tc.shuffle_seed = 7;
    auto ta = hybrid_nn::train(pa, ds, tc);
    auto tb = hybrid_nn::train(pb, ds, tc);
    CHECK(ta.size() == 6);
    CHECK(ta == tb);
    for (std::size_t n = 0; n < pa.weights.size(); ++n) CHECK(pa.weights[n] == pb.weights[n]);
    CHECK(pa.final_weights == pb.final_weights);
    CHECK(pa.w0 == w0.w);  // frozen branch, bitwise
    CHECK(ta.back() <= ta.front());
}

TEST_CASE(train_error_paths) {  // test_hybrid_nn.cpp:342-352
    LlsWeights w0;
    w0.w = Vec(4);
    Rng rng(2);
    CHECK(throws<dimension_error>([&] { hybrid_nn::init_params({8, 16}, w0, rng); }));
    HybridNetParams p = hybrid_nn::init_params({4, 8}, w0, rng);
    CHECK(throws<dimension_error>([&] { hybrid_nn::forward(p, Mat(2, 5)); }));
    WidenedDataset empty;
    empty.design = Mat(0, 4);
    empty.targets = Vec();
    CHECK(throws<dimension_error>([&] { hybrid_nn::train(p, empty, TrainConfig{}); }));
    WidenedDataset one;
    one.design = Mat(4, 4);
    one.targets = Vec(4);
    TrainConfig bad;
    bad.batch_size = 0;
    CHECK(throws<config_error>([&] { hybrid_nn::train(p, one, bad); }));
}

TEST_CASE(fused_plan_round_trip_and_f32_path) {  // test_fused.cpp:64-74, :121-131
    LlsWeights w0;
    w0.w = Vec(8);
    Rng rng(11);
    for (int i = 0; i < 8; ++i) w0.w[i] = gaussian(rng);
    HybridNetParams p = hybrid_nn::init_params({8, 64, 48, 64}, w0, rng);
    for (auto &b : p.biases)
        for (int i = 0; i < b.size(); ++i) b[i] = gaussian(rng) * 0.1;
    for (int i = 0; i < p.final_weights.size(); ++i) p.final_weights[i] = gaussian(rng) * 0.3;
    FusedPlan plan = fused::build_plan(p);
    CHECK(plan.fused);
    HybridNetParams u = plan.unpack();
    CHECK(u.w0 == p.w0 && u.final_weights == p.final_weights);
    for (std::size_t n = 0; n < p.weights.size(); ++n) CHECK(u.weights[n] == p.weights[n]);
    Mat x = random_mat(512, 8, 12);
    MatF xf(512, 8);
    for (int r = 0; r < 512; ++r)
        for (int c = 0; c < 8; ++c) xf(r, c) = static_cast<float>(x(r, c));
    VecF got = fused::fused_forward_f32(plan, xf);
    // FP64 straight-line reference (oracles.hpp:75-96) for the tolerance check
    double e = 0, s = 1;
    for (int r = 0; r < 512; ++r) {
        std::vector<double> act(8);
        double lin = 0;
        for (int c = 0; c < 8; ++c) {
            act[c] = x(r, c);
            lin += p.w0[c] * act[c];
        }
        for (std::size_t n = 0; n < p.weights.size(); ++n) {
            std::vector<double> nxt(p.dims[n + 1]);
            for (int j = 0; j < p.dims[n + 1]; ++j) {
                double acc = p.biases[n][j];
                for (int c = 0; c < p.dims[n]; ++c) acc += p.weights[n](j, c) * act[c];
                nxt[j] = acc > 0 ? acc : 0;
            }
            act = nxt;
        }
        double br = 0;
        for (int c = 0; c < p.dims.back(); ++c) br += p.final_weights[c] * act[c];
        e = std::max(e, std::abs(got[r] - (lin + br)));
        s = std::max(s, std::abs(lin + br));
    }
    CHECK(e / s < 1e-5);
}

TEST_CASE(eval_hard_decision_and_ber) {  // test_eval.cpp:10-37
    CVec s{cplx(0.9, 0.8), cplx(-0.1, -2.0), cplx(0.0, 0.0)};
    BitMat bits = hard_decision_qpsk(s);
    CHECK(bits(0, 0) == 0 && bits(0, 1) == 0 && bits(1, 0) == 1 && bits(1, 1) == 1);
    CHECK(bits(2, 0) == 0 && bits(2, 1) == 0);
    BitMat a(50, 2), c(50, 2);
    c(7, 1) = 1;
    CHECK(bit_error_rate(a, a) == 0.0);
    CHECK(std::abs(bit_error_rate(c, a) - 0.01) < 1e-15);
    CHECK(throws<dimension_error>([&] { bit_error_rate(a, BitMat(10, 2)); }));
}

int main() {
    for (const Case &c : cases()) {
        const int before = g_failed;
        try {
            c.fn();
        } catch (const std::exception &e) {
            ++g_failed;
            std::printf("  EXCEPTION in %s: %s\n", c.name, e.what());
        }
        std::printf("%s %s\n", g_failed == before ? "PASS" : "FAIL", c.name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
