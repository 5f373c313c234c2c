// B200-specific checks of the C++ API, beyond the reference's own unit tests
// (oracle/reftests.mk builds and tests/test_gpu_reference_suite.py runs
// those unmodified).  Written against the reference's API only.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "noma/channel_sim.hpp"
#include "noma/errors.hpp"
#include "noma/fused_inference.hpp"
#include "noma/hybrid_nn.hpp"
#include "noma/iq_transform.hpp"
#include "noma/lls.hpp"

using namespace noma;

namespace {

Mat gauss_mat(Eigen::Index rows, Eigen::Index cols, std::uint64_t seed) {
    Rng rng(seed);
    Mat m(rows, cols);
    for (Eigen::Index r = 0; r < rows; ++r)
        for (Eigen::Index c = 0; c < cols; ++c) m(r, c) = rng.gaussian();
    return m;
}

HybridNetParams net_of(const std::vector<int> &dims, std::uint64_t seed) {
    Rng rng(seed);
    LlsWeights w0;
    w0.w = Vec(dims[0]);
    for (int i = 0; i < dims[0]; ++i) w0.w[i] = rng.gaussian();
    HybridNetParams p = hybrid_nn::init_params(dims, w0, rng);
    for (auto &b : p.biases)
        for (Eigen::Index i = 0; i < b.size(); ++i) b[i] = 0.1 * rng.gaussian();
    for (Eigen::Index i = 0; i < p.final_weights.size(); ++i) p.final_weights[i] = 0.3 * rng.gaussian();
    return p;
}

double max_abs(const Vec &a) { return a.size() ? a.cwiseAbs().maxCoeff() : 0.0; }

// a synthetic widened training set of one user (the reference call chain,
// noma_cli.cpp:86-104)
WidenedDataset user_set(int M, int K, int NT, double snr, int user, std::uint64_t seed) {
    ScenarioConfig cfg;
    cfg.num_users = K;
    cfg.num_antennas = M;
    cfg.train_symbols = NT;
    cfg.data_symbols = 8;
    cfg.snr_db = snr;
    cfg.rx_nonlinearity_gain = 0.05;
    cfg.seed = seed;
    const TransmissionRecord rec = synthesize(cfg);
    return widen_dataset(rec.train_rx, CVec(rec.train_symbols.col(user)), user + 1);
}

// hybrid_nn::train restated from the API's own pieces: per epoch a
// Fisher-Yates shuffle of Rng(substream_seed(seed, epoch)), minibatches in
// that order, loss_and_grad + adam_step (hybrid_nn.cpp:148-195)
std::vector<double> train_by_composition(HybridNetParams &p, const WidenedDataset &ds, const TrainConfig &tc) {
    const Mat &x = ds.design;
    const Vec &y = *ds.targets;
    const Eigen::Index n = x.rows();
    AdamState s = AdamState::init(p, tc.lr);
    std::vector<double> trace;
    for (int e = 0; e < tc.epochs; ++e) {
        Rng rng(substream_seed(tc.shuffle_seed, static_cast<std::uint64_t>(e)));
        std::vector<Eigen::Index> idx(n);
        std::iota(idx.begin(), idx.end(), Eigen::Index{0});
        for (Eigen::Index i = n - 1; i > 0; --i) std::swap(idx[i], idx[rng.below(static_cast<std::uint64_t>(i) + 1)]);
        double sum = 0.0;
        for (Eigen::Index start = 0; start < n; start += tc.batch_size) {
            const Eigen::Index b = std::min<Eigen::Index>(tc.batch_size, n - start);
            Mat xb(b, x.cols());
            Vec yb(b);
            for (Eigen::Index i = 0; i < b; ++i) {
                xb.row(i) = x.row(idx[start + i]);
                yb[i] = y[idx[start + i]];
            }
            auto [loss, g] = hybrid_nn::loss_and_grad(p, xb, yb);
            hybrid_nn::adam_step(p, g, s);
            sum += loss * static_cast<double>(b);
        }
        trace.push_back(sum / static_cast<double>(n));
    }
    return trace;
}

double param_dev(const HybridNetParams &a, const HybridNetParams &b) {
    double d = max_abs(a.final_weights - b.final_weights), s = max_abs(b.final_weights);
    for (std::size_t n = 0; n < a.weights.size(); ++n) {
        d = std::max(d, (a.weights[n] - b.weights[n]).cwiseAbs().maxCoeff());
        d = std::max(d, max_abs(a.biases[n] - b.biases[n]));
        s = std::max(s, b.weights[n].cwiseAbs().maxCoeff());
    }
    return d / std::max(s, 1e-30);
}

}  // namespace

TEST_CASE("fused and per-layer device paths agree on a wide network (fused_inference.cpp:132-151)") {
    HybridNetParams p = net_of({8, 300, 200}, 1);
    FusedPlan plan = fused::build_plan(p);
    REQUIRE_FALSE(plan.fused);
    Mat x = gauss_mat(777, 8, 2);
    const Vec a = fused::fused_forward(plan, x);
    const Vec b = hybrid_nn::forward(p, x);
    CHECK(max_abs(a - b) / std::max(1.0, max_abs(b)) < 1e-12);
    // the FP32 evaluator at the reference's FP32 tolerance
    const MatF xf = x.cast<float>();
    const VecF f = fused::fused_forward_f32(plan, xf);
    CHECK(max_abs(f.cast<double>() - b) / std::max(1.0, max_abs(b)) < 1e-5);
    BenchReport rep = fused::bench_compare(plan, 256, 3);
    CHECK(rep.fused_ns_per_sample > 0);
    CHECK(rep.fallback_ns_per_sample > 0);
}

TEST_CASE("FP64 device training equals loss_and_grad + adam_step composed (hybrid_nn.cpp:158-195)") {
    const WidenedDataset ds = user_set(4, 3, 96, 15.0, 1, 7);
    const LlsWeights w0 = lls::fit(ds);
    Rng rng(8);
    HybridNetParams p = hybrid_nn::init_params({8, 24, 16}, w0, rng);
    HybridNetParams q = p;
    TrainConfig tc;
    tc.epochs = 3;
    tc.batch_size = 40;
    tc.shuffle_seed = 9;
    setenv("NOMA_TRAIN_PRECISION", "f64", 1);
    const std::vector<double> t1 = hybrid_nn::train(p, ds, tc);
    unsetenv("NOMA_TRAIN_PRECISION");
    const std::vector<double> t2 = train_by_composition(q, ds, tc);
    REQUIRE(t1.size() == t2.size());
    for (std::size_t e = 0; e < t1.size(); ++e) CHECK(std::abs(t1[e] - t2[e]) <= 1e-10 * std::abs(t2[e]));
    CHECK(param_dev(p, q) < 1e-9);
}

TEST_CASE("layers wider than 128 and minibatches above 128 rows train on the device") {
    const WidenedDataset ds = user_set(4, 2, 300, 20.0, 0, 11);
    const LlsWeights w0 = lls::fit(ds);
    for (const auto &cfg : {std::pair<std::vector<int>, int>{{8, 256}, 128}, {{8, 32}, 256}}) {
        Rng rng(12);
        HybridNetParams p = hybrid_nn::init_params(cfg.first, w0, rng);
        HybridNetParams q = p, r = p;
        TrainConfig tc;
        tc.epochs = 4;
        tc.batch_size = cfg.second;
        tc.shuffle_seed = 13;
        const std::vector<double> t = hybrid_nn::train(p, ds, tc);
        REQUIRE(t.size() == 4);
        CHECK(std::isfinite(t.back()));
        CHECK(t.back() <= t.front());
        // determinism (test_hybrid_nn.cpp:290-311)
        hybrid_nn::train(q, ds, tc);
        CHECK(q.weights[0] == p.weights[0]);
        CHECK(q.final_weights == p.final_weights);
        // FP32 against the FP64 composition of the API's own pieces
        train_by_composition(r, ds, tc);
        CHECK(param_dev(p, r) < 1e-3);
    }
}

TEST_CASE("a network without hidden layers (dims = [2M]) trains and detects") {
    const WidenedDataset ds = user_set(4, 2, 128, 20.0, 0, 21);
    const LlsWeights w0 = lls::fit(ds);
    Rng rng(22);
    HybridNetParams p = hybrid_nn::init_params({8}, w0, rng);
    REQUIRE(p.weights.empty());
    REQUIRE(p.final_weights.size() == 8);
    TrainConfig tc;
    tc.epochs = 3;
    const std::vector<double> t = hybrid_nn::train(p, ds, tc);
    CHECK(t.size() == 3);
    const Vec y = hybrid_nn::forward(p, ds.design);
    const Vec want = ds.design * (p.w0 + p.final_weights);
    CHECK(max_abs(y - want) < 1e-12);
}
