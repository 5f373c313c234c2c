// The reference detector's C++ API (proj/include/noma/*.hpp) implemented on
// the B200 through the C-ABI (include/noma_cuda.h).
//
// This file compiles against the reference's own headers, unmodified, when
// they are present (host/Makefile), else against host/include/noma/
// detector.hpp, which declares the same API.  Each function restates the
// reference's argument checks and exceptions (errors.hpp) and hands the
// arithmetic to the GPU: LLS, init, forward, loss/gradients, Adam, training,
// detection and channel synthesis all run in sm_100a kernels.  What stays on
// the host is layout work (packing Eigen column-major containers into the
// device layouts and back), argument validation, the sweep's bookkeeping, and
// draws from a caller-held Rng& whose stream the caller observes
// (gen_symbols / gen_channel take it by reference, channel_sim.hpp:64-67).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <locale>
#include <mutex>
#include <sstream>
#include <type_traits>

#include "noma/channel_sim.hpp"
#include "noma/errors.hpp"
#include "noma/eval.hpp"
#include "noma/format.hpp"
#include "noma/fused_inference.hpp"
#include "noma/hybrid_nn.hpp"
#include "noma/iq_transform.hpp"
#include "noma/lls.hpp"
#include "noma/rng.hpp"
#include "noma/types.hpp"
#include "noma_cuda.h"

namespace noma {
namespace {

// One context (device 0, or NOMA_DEVICE) per process; every call is
// synchronous on its stream, like the reference's free functions.
noma_ctx_t ctx() {
    static noma_ctx_t c = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *e = std::getenv("NOMA_DEVICE");
        if (noma_ctx_create(e ? std::atoi(e) : 0, &c) != NOMA_OK) c = nullptr;
    });
    if (!c) throw std::runtime_error("noma: no CUDA device (the B200 path has no CPU fallback)");
    return c;
}

[[noreturn]] void raise(int st, const std::string &what, double cond = 0.0) {
    const std::string msg = what + ": " + noma_ctx_last_error(ctx());
    switch (st) {
        case NOMA_ERR_DIMENSION: throw dimension_error(msg);
        case NOMA_ERR_CONFIG: throw config_error(msg);
        case NOMA_ERR_ILL_CONDITIONED: throw ill_conditioned_error(msg, cond);
        default: throw std::runtime_error(msg);
    }
}

void check(int st, const char *what) {
    if (st != NOMA_OK) raise(st, what);
}

noma_net_desc desc_of(const std::vector<int> &dims) {
    noma_net_desc d{};
    if (dims.empty() || dims.size() > NOMA_MAX_DIMS)
        throw dimension_error("noma: networks take 1 to " + std::to_string(NOMA_MAX_DIMS) + " widths");
    d.ndims = static_cast<int>(dims.size());
    for (std::size_t i = 0; i < dims.size(); ++i) d.dims[i] = dims[i];
    return d;
}

int pad8(int w) { return ((w + 7) / 8) * 8; }

// FusedPlan buffer offsets (fused_inference.cpp:19-42): w0[pad0] | per layer
// W rows x pad_{l-1}, b[pad_l] | final[pad_N]
struct PlanOffsets {
    std::vector<std::size_t> w, b;
    std::size_t f = 0, total = 0;
    explicit PlanOffsets(const std::vector<int> &dims) {
        std::size_t o = static_cast<std::size_t>(pad8(dims[0]));
        for (std::size_t l = 1; l < dims.size(); ++l) {
            w.push_back(o);
            o += static_cast<std::size_t>(dims[l]) * pad8(dims[l - 1]);
            b.push_back(o);
            o += static_cast<std::size_t>(pad8(dims[l]));
        }
        f = o;
        total = o + static_cast<std::size_t>(pad8(dims.back()));
    }
};

template <class T>
std::vector<T> pack_plan(const HybridNetParams &p) {
    const PlanOffsets lo(p.dims);
    std::vector<T> buf(lo.total, T(0));
    for (Eigen::Index c = 0; c < p.w0.size(); ++c) buf[c] = static_cast<T>(p.w0[c]);
    for (std::size_t n = 0; n < p.weights.size(); ++n) {
        const Mat &w = p.weights[n];
        const std::size_t pin = static_cast<std::size_t>(pad8(p.dims[n]));
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) buf[lo.w[n] + r * pin + c] = static_cast<T>(w(r, c));
        for (Eigen::Index j = 0; j < p.biases[n].size(); ++j) buf[lo.b[n] + j] = static_cast<T>(p.biases[n][j]);
    }
    for (Eigen::Index j = 0; j < p.final_weights.size(); ++j) buf[lo.f + j] = static_cast<T>(p.final_weights[j]);
    return buf;
}

// trainable block of a plan buffer back into params (w0 untouched)
template <class T>
void unpack_trainable(const T *buf, HybridNetParams &p) {
    const PlanOffsets lo(p.dims);
    for (std::size_t n = 0; n < p.weights.size(); ++n) {
        Mat &w = p.weights[n];
        const std::size_t pin = static_cast<std::size_t>(pad8(p.dims[n]));
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = static_cast<double>(buf[lo.w[n] + r * pin + c]);
        for (Eigen::Index j = 0; j < p.biases[n].size(); ++j) p.biases[n][j] = static_cast<double>(buf[lo.b[n] + j]);
    }
    for (Eigen::Index j = 0; j < p.final_weights.size(); ++j)
        p.final_weights[j] = static_cast<double>(buf[lo.f + j]);
}

void check_params(const HybridNetParams &p) {
    if (p.dims.empty() || p.weights.size() + 1 != p.dims.size() || p.biases.size() != p.weights.size() ||
        p.w0.size() != p.dims[0] || p.final_weights.size() != p.dims.back())
        throw dimension_error("noma: HybridNetParams shapes do not match dims");
    for (std::size_t n = 0; n < p.weights.size(); ++n)
        if (p.weights[n].rows() != p.dims[n + 1] || p.weights[n].cols() != p.dims[n] ||
            p.biases[n].size() != p.dims[n + 1])
            throw dimension_error("noma: HybridNetParams layer shapes do not match dims");
}

// flat reference order (W_1 row-major, b_1, ..., final) <-> Gradients
Gradients grads_from_flat(const HybridNetParams &p, const std::vector<double> &g) {
    Gradients out;
    std::size_t o = 0;
    for (std::size_t n = 0; n < p.weights.size(); ++n) {
        Mat w(p.dims[n + 1], p.dims[n]);
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = g[o++];
        out.weights.push_back(std::move(w));
        Vec b(p.dims[n + 1]);
        for (Eigen::Index j = 0; j < b.size(); ++j) b[j] = g[o++];
        out.biases.push_back(std::move(b));
    }
    out.final_weights = Vec(p.dims.back());
    for (Eigen::Index j = 0; j < out.final_weights.size(); ++j) out.final_weights[j] = g[o++];
    return out;
}

// element order of the Adam state: any fixed order works (the update is
// elementwise); Eigen storage order keeps the copies trivial
template <class F>
void for_each_block(HybridNetParams &p, const Gradients &g, AdamState &s, F &&f) {
    for (std::size_t n = 0; n < p.weights.size(); ++n) {
        f(p.weights[n].data(), g.weights[n].data(), s.m.weights[n].data(), s.v.weights[n].data(), p.weights[n].size());
        f(p.biases[n].data(), g.biases[n].data(), s.m.biases[n].data(), s.v.biases[n].data(), p.biases[n].size());
    }
    f(p.final_weights.data(), g.final_weights.data(), s.m.final_weights.data(), s.v.final_weights.data(),
      p.final_weights.size());
}

// A real design is the widened one when every row pair is [a, b] / [b, -a]
// (iq_transform.cpp:17-20); the device then works on the complex rows.
bool is_widened(const Mat &x) {
    if (x.rows() % 2 || x.cols() % 2 || x.rows() == 0) return false;
    const Eigen::Index m = x.cols() / 2;
    for (Eigen::Index t = 0; 2 * t < x.rows(); ++t)
        for (Eigen::Index j = 0; j < m; ++j)
            if (x(2 * t + 1, j) != x(2 * t, m + j) || x(2 * t + 1, m + j) != -x(2 * t, j)) return false;
    return true;
}

std::vector<double> complex_rows(const Mat &x) {  // [rows/2][cols/2] interleaved
    const Eigen::Index n = x.rows() / 2, m = x.cols() / 2;
    std::vector<double> out(static_cast<std::size_t>(n * m * 2));
    for (Eigen::Index t = 0; t < n; ++t)
        for (Eigen::Index j = 0; j < m; ++j) {
            out[(t * m + j) * 2] = x(2 * t, j);
            out[(t * m + j) * 2 + 1] = x(2 * t, m + j);
        }
    return out;
}

std::vector<double> row_major(const Mat &x) {
    std::vector<double> out(static_cast<std::size_t>(x.size()));
    for (Eigen::Index r = 0; r < x.rows(); ++r)
        for (Eigen::Index c = 0; c < x.cols(); ++c) out[r * x.cols() + c] = x(r, c);
    return out;
}

// X w on the device: the FP64 forward of the network [cols] with final layer
// zero, i.e. the linear branch alone, accumulated exactly as forward() does
Vec linear_forward(const Vec &w, const Mat &x) {
    const std::vector<int> dims{static_cast<int>(w.size())};
    const noma_net_desc d = desc_of(dims);
    std::vector<double> plan(static_cast<std::size_t>(2 * pad8(dims[0])), 0.0);
    for (Eigen::Index c = 0; c < w.size(); ++c) plan[c] = w[c];
    Vec out(x.rows());
    check(noma_forward_f64(ctx(), &d, plan.data(), static_cast<int>(x.rows()), x.data(), out.data(), NOMA_PATH_FUSED,
                           NOMA_MEM_HOST),
          "lls::predict");
    return out;
}

std::uint64_t mix_tag(std::uint64_t a, std::uint64_t b, std::uint64_t c = 0, std::uint64_t d = 0) {
    // eval.cpp:77-84; C++17 sequences splitmix64's update of s before the xor
    std::uint64_t s = a * 0x9E3779B97F4A7C15ULL + 1;
    for (const std::uint64_t v : {b, c, d}) {
        const std::uint64_t r = splitmix64(s) + v;
        s ^= r;
    }
    return splitmix64(s);
}

CMat rows_to_cmat(const double *p, Eigen::Index rows, Eigen::Index cols) {  // [rows][cols] c64
    CMat m(rows, cols);
    for (Eigen::Index r = 0; r < rows; ++r)
        for (Eigen::Index c = 0; c < cols; ++c) m(r, c) = cplx(p[(r * cols + c) * 2], p[(r * cols + c) * 2 + 1]);
    return m;
}

}  // namespace

// =============================================================== channel_sim
void ScenarioConfig::validate() const {  // channel_sim.cpp:9-21
    if (num_users < 1) throw config_error("num_users must be >= 1");
    if (num_antennas < 1) throw config_error("num_antennas must be >= 1");
    if (train_symbols < 1 || data_symbols < 1) throw config_error("symbol counts must be >= 1");
    if (train_symbols < 2 * num_antennas)
        throw config_error("train_symbols must be >= 2*num_antennas for an over-determined widened system");
    if (power_step_db < 0.0) throw config_error("power_step_db must be >= 0");
    if (rx_nonlinearity_gain < 0.0) throw config_error("rx_nonlinearity_gain must be >= 0");
    if (std::isnan(snr_db)) throw config_error("snr_db must not be NaN");
}

Vec power_profile(int num_users, double step_db) {  // channel_sim.cpp:23-28
    Vec p(num_users);
    for (int k = 0; k < num_users; ++k) p[k] = std::pow(10.0, -k * step_db / 10.0);
    return p;
}

// The two draw helpers consume the caller's Rng& (row-major symbols via
// below(4), channel k then m); the device synthesiser restates the same
// streams for whole records.
CMat gen_symbols(int num_users, int num_symbols, Modulation, Rng &rng) {  // channel_sim.cpp:30-46
    if (num_users < 1 || num_symbols < 1) throw dimension_error("gen_symbols: dimensions must be >= 1");
    const double a = 1.0 / std::sqrt(2.0);
    CMat out(num_symbols, num_users);
    for (int t = 0; t < num_symbols; ++t)
        for (int k = 0; k < num_users; ++k) {
            const std::uint64_t bits = rng.below(4);
            out(t, k) = cplx((bits & 1) ? -a : a, (bits & 2) ? -a : a);
        }
    return out;
}

CMat gen_channel(int num_users, int num_antennas, Rng &rng) {  // channel_sim.cpp:48-57
    if (num_users < 1 || num_antennas < 1) throw dimension_error("gen_channel: dimensions must be >= 1");
    const double s = 1.0 / std::sqrt(2.0);
    CMat h(num_antennas, num_users);
    for (int k = 0; k < num_users; ++k)
        for (int m = 0; m < num_antennas; ++m) {
            // cplx(g() * s, g() * s): the reference's g++ build evaluates the
            // imaginary argument first (tests/golden/probe_eval_order.cpp)
            const double im = rng.gaussian() * s;
            const double re = rng.gaussian() * s;
            h(m, k) = cplx(re, im);
        }
    return h;
}

TransmissionRecord synthesize(const ScenarioConfig &cfg) { return synthesize(cfg, SeedBundle::from_master(cfg.seed)); }

TransmissionRecord synthesize(const ScenarioConfig &cfg, const SeedBundle &seeds) {  // channel_sim.cpp:76-117
    cfg.validate();
    const int K = cfg.num_users, M = cfg.num_antennas, NT = cfg.train_symbols, ND = cfg.data_symbols;
    const noma_scenario sc{K, M, NT, ND, cfg.power_step_db, cfg.snr_db, cfg.rx_nonlinearity_gain};
    const std::uint64_t bundle[3] = {seeds.symbols, seeds.channel, seeds.noise};
    std::vector<double> prx(static_cast<std::size_t>(NT) * M * 2), psym(static_cast<std::size_t>(NT) * K * 2),
        drx(static_cast<std::size_t>(ND) * M * 2), chan(static_cast<std::size_t>(M) * K * 2);
    std::vector<std::uint8_t> codes(static_cast<std::size_t>(ND) * K);
    double np = 0.0;
    check(noma_synthesize_f64(ctx(), &sc, 1, bundle, prx.data(), psym.data(), drx.data(), codes.data(), chan.data(),
                              &np, NOMA_MEM_HOST),
          "synthesize");
    TransmissionRecord rec;
    rec.powers = power_profile(K, cfg.power_step_db);
    rec.channel = rows_to_cmat(chan.data(), M, K);
    rec.train_rx = rows_to_cmat(prx.data(), NT, M);
    rec.train_symbols = rows_to_cmat(psym.data(), NT, K);
    rec.data_rx = rows_to_cmat(drx.data(), ND, M);
    const double a = 1.0 / std::sqrt(2.0);
    rec.data_symbols = CMat(ND, K);
    for (int t = 0; t < ND; ++t)
        for (int k = 0; k < K; ++k) {
            const std::uint8_t b = codes[static_cast<std::size_t>(t) * K + k];
            rec.data_symbols(t, k) = cplx((b & 1) ? -a : a, (b & 2) ? -a : a);
        }
    rec.noise_power = np;
    return rec;
}

// ============================================================== iq_transform
Mat widen_design(const CMat &x) {  // iq_transform.cpp:7-24
    if (x.rows() == 0 || x.cols() == 0) throw dimension_error("widen_design: empty input");
    const Eigen::Index n = x.rows(), m = x.cols();
    Mat out(2 * n, 2 * m);
    for (Eigen::Index t = 0; t < n; ++t)
        for (Eigen::Index j = 0; j < m; ++j) {
            const double re = x(t, j).real(), im = x(t, j).imag();
            out(2 * t, j) = re;
            out(2 * t, m + j) = im;
            out(2 * t + 1, j) = im;
            out(2 * t + 1, m + j) = -re;
        }
    return out;
}

Vec widen_targets(const CVec &y) {  // iq_transform.cpp:26-33
    Vec out(2 * y.size());
    for (Eigen::Index t = 0; t < y.size(); ++t) {
        out[2 * t] = y[t].real();
        out[2 * t + 1] = y[t].imag();
    }
    return out;
}

WidenedDataset widen_dataset(const CMat &x, const std::optional<CVec> &y, int user_index) {  // :35-45
    WidenedDataset ds;
    ds.design = widen_design(x);
    if (y) {
        if (y->size() != x.rows()) throw dimension_error("widen_dataset: target length does not match rows");
        ds.targets = widen_targets(*y);
        ds.user_index = user_index;
    }
    return ds;
}

CVec narrow_predictions(const Vec &yhat) {  // iq_transform.cpp:47-54
    if (yhat.size() % 2 != 0) throw dimension_error("narrow_predictions: length must be even");
    CVec out(yhat.size() / 2);
    for (Eigen::Index t = 0; t < out.size(); ++t) out[t] = cplx(yhat[2 * t], yhat[2 * t + 1]);
    return out;
}

// ======================================================================= lls
namespace lls {

LlsWeights fit(const Mat &design, const Vec &targets, int user_index) {  // lls.cpp:10-54
    if (design.rows() < design.cols()) throw dimension_error("lls::fit: system must be over-determined");
    if (design.rows() != targets.size()) throw dimension_error("lls::fit: design rows and target length differ");
    // widened designs go to the device as their complex rows (complex Gram,
    // DESIGN.md 4); any other design as real rows
    const bool wid = is_widened(design);
    const std::vector<double> x = wid ? complex_rows(design) : row_major(design);
    const noma_dataset ds{wid ? NOMA_LAYOUT_WIDEN_COMPLEX : NOMA_LAYOUT_REAL, 1, 1, static_cast<int>(design.rows()),
                          static_cast<int>(design.cols()), x.data(), targets.data()};
    LlsWeights out;
    out.user_index = user_index;
    out.w = Vec(design.cols());
    int status = 0;
    const int st = noma_lls_fit(ctx(), &ds, out.w.data(), &out.gram_condition, &status, NOMA_MEM_HOST);
    if (st == NOMA_ERR_ILL_CONDITIONED)
        throw ill_conditioned_error("lls::fit: design matrix rank deficient and system inconsistent",
                                    out.gram_condition);
    check(st, "lls::fit");
    return out;
}

LlsWeights fit(const WidenedDataset &train) {  // lls.cpp:56-60
    if (!train.targets) throw dimension_error("lls::fit: training set has no targets");
    return fit(train.design, *train.targets, train.user_index);
}

CVec predict(const LlsWeights &weights, const Mat &widened_detect) {  // lls.cpp:62-66
    if (widened_detect.cols() != weights.w.size())
        throw dimension_error("lls::predict: column count does not match weights");
    return narrow_predictions(linear_forward(weights.w, widened_detect));
}

}  // namespace lls

// ================================================================= hybrid_nn
std::size_t HybridNetParams::trainable_count() const {  // hybrid_nn.cpp:11-16
    std::size_t n = static_cast<std::size_t>(final_weights.size());
    for (std::size_t i = 0; i < weights.size(); ++i)
        n += static_cast<std::size_t>(weights[i].size() + biases[i].size());
    return n;
}

AdamState AdamState::init(const HybridNetParams &params, double lr) {  // hybrid_nn.cpp:18-30
    AdamState s;
    s.lr = lr;
    for (Gradients *g : {&s.m, &s.v}) {
        for (std::size_t i = 0; i < params.weights.size(); ++i) {
            g->weights.push_back(Mat::Zero(params.weights[i].rows(), params.weights[i].cols()));
            g->biases.push_back(Vec::Zero(params.biases[i].size()));
        }
        g->final_weights = Vec::Zero(params.final_weights.size());
    }
    return s;
}

namespace hybrid_nn {

HybridNetParams init_params(const std::vector<int> &dims, const LlsWeights &w0, Rng &rng) {  // :34-55
    if (dims.empty() || dims[0] != w0.w.size()) throw dimension_error("init_params: dims[0] must equal the w0 length");
    for (int d : dims)
        if (d < 1) throw dimension_error("init_params: layer widths must be >= 1");
    const noma_net_desc d = desc_of(dims);
    // the device draws from the caller's xoshiro256++ state and hands back
    // the advanced state (Rng is a standard-layout wrapper of that state)
    static_assert(sizeof(Rng) == 4 * sizeof(std::uint64_t) && std::is_trivially_copyable_v<Rng>);
    std::uint64_t state[4];
    std::memcpy(state, &rng, sizeof state);
    std::vector<double> theta(static_cast<std::size_t>(noma_param_count(&d)));
    check(noma_init_params_state(ctx(), &d, 1, state, w0.w.data(), nullptr, theta.data(), NOMA_MEM_HOST),
          "init_params");
    std::memcpy(static_cast<void *>(&rng), state, sizeof state);
    HybridNetParams p;
    p.dims = dims;
    p.w0 = w0.w;
    std::size_t o = 0;
    for (std::size_t l = 1; l < dims.size(); ++l) {
        Mat w(dims[l], dims[l - 1]);
        for (int r = 0; r < dims[l]; ++r)
            for (int c = 0; c < dims[l - 1]; ++c) w(r, c) = theta[o++];
        p.weights.push_back(std::move(w));
        p.biases.push_back(Vec::Zero(dims[l]));
        o += static_cast<std::size_t>(dims[l]);
    }
    p.final_weights = Vec::Zero(dims.back());
    return p;
}

Vec forward(const HybridNetParams &p, const Mat &x) {  // hybrid_nn.cpp:77-82
    if (x.cols() != p.w0.size()) throw dimension_error("forward: input width does not match network");
    check_params(p);
    const noma_net_desc d = desc_of(p.dims);
    const std::vector<double> plan = pack_plan<double>(p);
    Vec out(x.rows());
    check(noma_forward_f64(ctx(), &d, plan.data(), static_cast<int>(x.rows()), x.data(), out.data(), NOMA_PATH_AUTO,
                           NOMA_MEM_HOST),
          "forward");
    return out;
}

std::pair<double, Gradients> loss_and_grad(const HybridNetParams &p, const Mat &x, const Vec &y) {  // :84-114
    if (x.rows() == 0) throw dimension_error("loss_and_grad: empty batch");
    if (x.cols() != p.w0.size() || y.size() != x.rows()) throw dimension_error("loss_and_grad: dimension mismatch");
    check_params(p);
    const noma_net_desc d = desc_of(p.dims);
    const std::vector<double> plan = pack_plan<double>(p);
    std::vector<double> g(p.trainable_count());
    double loss = 0.0;
    check(noma_loss_and_grad(ctx(), &d, plan.data(), static_cast<int>(x.rows()), x.data(), y.data(), &loss, g.data(),
                             NOMA_MEM_HOST),
          "loss_and_grad");
    return {loss, grads_from_flat(p, g)};
}

void adam_step(HybridNetParams &p, const Gradients &g, AdamState &s) {  // hybrid_nn.cpp:126-144
    if (g.weights.size() != p.weights.size() || g.final_weights.size() != p.final_weights.size())
        throw dimension_error("adam_step: gradient shapes do not match");
    if (g.biases.size() != p.biases.size() || s.m.weights.size() != p.weights.size() ||
        s.v.weights.size() != p.weights.size())
        throw dimension_error("adam_step: gradient shapes do not match");
    for (std::size_t n = 0; n < p.weights.size(); ++n)
        if (g.weights[n].size() != p.weights[n].size() || g.biases[n].size() != p.biases[n].size() ||
            s.m.weights[n].size() != p.weights[n].size() || s.v.weights[n].size() != p.weights[n].size())
            throw dimension_error("adam_step: gradient shapes do not match");
    ++s.step;
    const double corr1 = 1.0 - std::pow(s.beta1, static_cast<double>(s.step));
    const double corr2 = 1.0 - std::pow(s.beta2, static_cast<double>(s.step));
    // one elementwise launch over every block, staged contiguously
    const std::size_t n = p.trainable_count();
    std::vector<double> th(n), gr(n), m(n), v(n);
    std::size_t o = 0;
    for_each_block(p, g, s, [&](double *a, const double *b, double *c, double *e, Eigen::Index k) {
        std::copy(a, a + k, th.begin() + o);
        std::copy(b, b + k, gr.begin() + o);
        std::copy(c, c + k, m.begin() + o);
        std::copy(e, e + k, v.begin() + o);
        o += static_cast<std::size_t>(k);
    });
    check(noma_adam_step(ctx(), static_cast<int>(n), th.data(), gr.data(), m.data(), v.data(), corr1, corr2, s.lr,
                         s.beta1, s.beta2, s.eps, NOMA_MEM_HOST),
          "adam_step");
    o = 0;
    for_each_block(p, g, s, [&](double *a, const double *, double *c, double *e, Eigen::Index k) {
        std::copy(th.begin() + o, th.begin() + o + k, a);
        std::copy(m.begin() + o, m.begin() + o + k, c);
        std::copy(v.begin() + o, v.begin() + o + k, e);
        o += static_cast<std::size_t>(k);
    });
}

std::vector<double> train(HybridNetParams &p, const WidenedDataset &set, const TrainConfig &cfg) {  // :158-195
    if (!set.targets) throw dimension_error("train: training set has no targets");
    if (set.design.rows() == 0) throw dimension_error("train: empty training set");
    if (cfg.epochs < 0 || cfg.batch_size < 1 || cfg.lr <= 0.0)
        throw config_error("train: invalid training configuration");
    std::vector<double> trace(static_cast<std::size_t>(cfg.epochs));
    if (cfg.epochs == 0) return trace;
    if (set.design.cols() != p.w0.size() || set.targets->size() != set.design.rows())
        throw dimension_error("loss_and_grad: dimension mismatch");
    check_params(p);
    const bool wid = is_widened(set.design);
    const std::vector<double> x = wid ? complex_rows(set.design) : row_major(set.design);
    const noma_dataset ds{wid ? NOMA_LAYOUT_WIDEN_COMPLEX : NOMA_LAYOUT_REAL, 1, 1,
                          static_cast<int>(set.design.rows()), static_cast<int>(set.design.cols()), x.data(),
                          set.targets->data()};
    const noma_net_desc d = desc_of(p.dims);
    const noma_train_cfg tc{cfg.epochs, cfg.batch_size, cfg.lr, 0.9, 0.999, 1e-8};  // AdamState defaults
    std::uint64_t seed = cfg.shuffle_seed;
    // FP32 FFMA training (north star); NOMA_TRAIN_PRECISION=f64 selects the
    // reference's FP64 arithmetic on the device instead
    const char *prec = std::getenv("NOMA_TRAIN_PRECISION");
    if (prec && std::string(prec) == "f64") {
        std::vector<double> theta;
        theta.reserve(p.trainable_count());
        for (std::size_t n = 0; n < p.weights.size(); ++n) {
            for (Eigen::Index r = 0; r < p.weights[n].rows(); ++r)
                for (Eigen::Index c = 0; c < p.weights[n].cols(); ++c) theta.push_back(p.weights[n](r, c));
            theta.insert(theta.end(), p.biases[n].data(), p.biases[n].data() + p.biases[n].size());
        }
        theta.insert(theta.end(), p.final_weights.data(), p.final_weights.data() + p.final_weights.size());
        check(noma_train_f64(ctx(), &ds, &d, &tc, p.w0.data(), theta.data(), &seed, trace.data(), nullptr,
                             NOMA_MEM_HOST),
              "train");
        const Gradients t = grads_from_flat(p, theta);
        p.weights = t.weights;
        p.biases = t.biases;
        p.final_weights = t.final_weights;
        return trace;
    }
    std::vector<float> plan = pack_plan<float>(p);
    check(noma_train(ctx(), &ds, &d, &tc, p.w0.data(), plan.data(), &seed, trace.data(), nullptr, NOMA_MEM_HOST),
          "train");
    unpack_trainable(plan.data(), p);
    return trace;
}

CVec detect(const HybridNetParams &p, const Mat &widened_detect) {  // hybrid_nn.cpp:197-199
    return narrow_predictions(forward(p, widened_detect));
}

}  // namespace hybrid_nn

// =========================================================== fused_inference
HybridNetParams FusedPlan::unpack() const {  // fused_inference.cpp:155-170
    const PlanOffsets lo(dims);
    HybridNetParams p;
    p.dims = dims;
    p.w0 = Vec(dims[0]);
    for (int c = 0; c < dims[0]; ++c) p.w0[c] = buffer[c];
    for (std::size_t l = 1; l < dims.size(); ++l) {
        p.weights.push_back(Mat(dims[l], dims[l - 1]));
        p.biases.push_back(Vec(dims[l]));
    }
    p.final_weights = Vec(dims.back());
    unpack_trainable(buffer.data(), p);
    return p;
}

std::string BenchReport::to_csv(bool with_header) const {  // fused_inference.cpp:325-338
    std::ostringstream os;
    os.imbue(std::locale::classic());
    if (with_header) os << "path,dims,batch,ns_per_sample,speedup_vs_naive\n";
    std::string ds;
    for (std::size_t i = 0; i < dims.size(); ++i) ds += (i ? "x" : "") + std::to_string(dims[i]);
    os << "fused," << ds << ',' << batch << ',' << fused_ns_per_sample << ',' << speedup_vs_naive << '\n';
    os << "naive," << ds << ',' << batch << ',' << naive_ns_per_sample << ",1\n";
    os << "fallback," << ds << ',' << batch << ',' << fallback_ns_per_sample << ','
       << naive_ns_per_sample / fallback_ns_per_sample << '\n';
    return os.str();
}

namespace fused {

FusedPlan build_plan(const HybridNetParams &params) {  // fused_inference.cpp:174-203
    check_params(params);
    FusedPlan plan;
    plan.dims = params.dims;
    plan.max_width = *std::max_element(params.dims.begin(), params.dims.end());
    plan.fused = plan.max_width <= kFusedMaxWidth;
    for (int d : params.dims) plan.padded.push_back(pad8(d));
    plan.buffer = pack_plan<double>(params);
    plan.buffer_f32.assign(plan.buffer.begin(), plan.buffer.end());
    for (std::size_t i = 0; i < plan.buffer.size(); ++i) plan.buffer_f32[i] = static_cast<float>(plan.buffer[i]);
    return plan;
}

// Single-pass on-chip tiles when the plan is fused, one launch per layer
// otherwise (the reference's dispatch, fused_inference.cpp:205-214).  The
// descriptor lives on the stack and the staging buffers in the context's
// device workspace: no heap allocation here (test_fused.cpp:133-144).
void fused_forward_into(const FusedPlan &plan, const Mat &x, Vec &out) {
    if (x.cols() != plan.dims[0]) throw dimension_error("fused_forward: input width does not match plan");
    if (out.size() != x.rows()) throw dimension_error("fused_forward: output not presized to batch");
    if (plan.dims.size() > NOMA_MAX_DIMS) throw dimension_error("fused_forward: too many layers");
    noma_net_desc d{};
    d.ndims = static_cast<int>(plan.dims.size());
    for (std::size_t i = 0; i < plan.dims.size(); ++i) d.dims[i] = plan.dims[i];
    const int st = noma_forward_f64(ctx(), &d, plan.buffer.data(), static_cast<int>(x.rows()), x.data(), out.data(),
                                    plan.fused ? NOMA_PATH_FUSED : NOMA_PATH_FALLBACK, NOMA_MEM_HOST);
    if (st != NOMA_OK) raise(st, "fused_forward");
}

Vec fused_forward(const FusedPlan &plan, const Mat &x) {
    Vec out(x.rows());
    fused_forward_into(plan, x, out);
    return out;
}

VecF fused_forward_f32(const FusedPlan &plan, const MatF &x) {  // fused_inference.cpp:222-231
    if (x.cols() != plan.dims[0]) throw dimension_error("fused_forward_f32: input width does not match plan");
    const noma_net_desc d = desc_of(plan.dims);
    VecF out(x.rows());
    check(noma_forward_f32(ctx(), &d, plan.buffer_f32.data(), static_cast<int>(x.rows()), x.data(), out.data(),
                           plan.fused ? NOMA_PATH_FUSED : NOMA_PATH_FALLBACK, NOMA_MEM_HOST),
          "fused_forward_f32");
    return out;
}

// The three device evaluators on the same random batch: an equivalence gate
// first (1e-12 against the naive per-layer path, as the reference gates
// against its naive forward), then the median device time of each over
// `repeats` launches with the batch resident in HBM (fused_inference.cpp:
// 262-314 times the CPU paths the same way, steady_clock medians).
BenchReport bench_compare(const FusedPlan &plan, int batch, int repeats) {
    if (batch < 1 || repeats < 1) throw dimension_error("bench_compare: batch and repeats must be >= 1");
    Rng rng(0x9E24Au);
    Mat x(batch, plan.dims[0]);
    for (Eigen::Index r = 0; r < x.rows(); ++r)
        for (Eigen::Index c = 0; c < x.cols(); ++c) x(r, c) = rng.gaussian();
    const noma_net_desc d = desc_of(plan.dims);
    Vec outs[3] = {Vec(batch), Vec(batch), Vec(batch)};
    const int paths[3] = {NOMA_PATH_FUSED, NOMA_PATH_NAIVE, NOMA_PATH_FALLBACK};
    double ns[3];
    for (int i = 0; i < 3; ++i) {
        check(noma_forward_f64(ctx(), &d, plan.buffer.data(), batch, x.data(), outs[i].data(), paths[i],
                               NOMA_MEM_HOST),
              "bench_compare");
        check(noma_bench_forward_f64(ctx(), &d, plan.buffer.data(), batch, x.data(), paths[i], repeats, &ns[i]),
              "bench_compare");
    }
    const Vec &ref = outs[1];
    const double scale = std::max(1.0, ref.cwiseAbs().maxCoeff());
    for (int i : {0, 2})
        if ((outs[i] - ref).cwiseAbs().maxCoeff() / scale > 1e-12)
            throw std::runtime_error("bench_compare: evaluation paths disagree");
    BenchReport rep;
    rep.dims = plan.dims;
    rep.batch = batch;
    rep.repeats = repeats;
    rep.fused_ns_per_sample = ns[0] / batch;
    rep.naive_ns_per_sample = ns[1] / batch;
    rep.fallback_ns_per_sample = ns[2] / batch;
    rep.speedup_vs_naive = rep.naive_ns_per_sample / rep.fused_ns_per_sample;
    rep.machine = "NVIDIA B200 (sm_100a), device-resident batch, FP64";
    return rep;
}

}  // namespace fused

// ====================================================================== eval
std::string to_string(DetectorId id) { return id == DetectorId::Lls ? "LLS" : "HybridNN"; }  // eval.cpp:12-14

std::string to_string(Ablation a) {  // eval.cpp:16-23
    switch (a) {
        case Ablation::SymmetryOn: return "symmetry_on";
        case Ablation::SymmetryOff: return "symmetry_off";
        case Ablation::SymmetryOnHalfData: return "symmetry_on_half_data";
    }
    return "?";
}

DetectorId detector_from_string(const std::string &s) {  // eval.cpp:25-29
    if (s == "LLS") return DetectorId::Lls;
    if (s == "HybridNN") return DetectorId::HybridNn;
    throw config_error("unknown detector id: " + s);
}

Ablation ablation_from_string(const std::string &s) {  // eval.cpp:31-36
    for (Ablation a : {Ablation::SymmetryOn, Ablation::SymmetryOff, Ablation::SymmetryOnHalfData})
        if (s == to_string(a)) return a;
    throw config_error("unknown ablation: " + s);
}

// The batched device path fuses these into the detection epilogue
// (noma_detect / noma_pipeline); here they act on host-resident results.
BitMat hard_decision_qpsk(const CVec &symbols) {  // eval.cpp:38-45
    BitMat bits(symbols.size(), 2);
    for (Eigen::Index t = 0; t < symbols.size(); ++t) {
        bits(t, 0) = symbols[t].real() < 0.0 ? 1 : 0;
        bits(t, 1) = symbols[t].imag() < 0.0 ? 1 : 0;
    }
    return bits;
}

CVec map_qpsk_bits(const BitMat &bits) {  // eval.cpp:47-54
    if (bits.cols() != 2) throw dimension_error("map_qpsk_bits: expected N x 2");
    const double a = 1.0 / std::sqrt(2.0);
    CVec out(bits.rows());
    for (Eigen::Index t = 0; t < bits.rows(); ++t)
        out[t] = cplx((1 - 2 * bits(t, 0)) * a, (1 - 2 * bits(t, 1)) * a);
    return out;
}

double bit_error_rate(const BitMat &predicted, const BitMat &truth) {  // eval.cpp:56-65
    if (predicted.rows() != truth.rows() || predicted.cols() != truth.cols())
        throw dimension_error("bit_error_rate: shape mismatch");
    if (predicted.size() == 0) throw dimension_error("bit_error_rate: empty input");
    long long errors = 0;
    for (Eigen::Index c = 0; c < predicted.cols(); ++c)
        for (Eigen::Index r = 0; r < predicted.rows(); ++r) errors += predicted(r, c) != truth(r, c);
    return static_cast<double>(errors) / static_cast<double>(predicted.size());
}

std::string BerReport::to_csv() const {  // eval.cpp:257-266
    std::ostringstream os;
    os << "snr_db,user,detector,ablation,trials,mean_ber,sd_ber,total_bits\n";
    for (const BerCell &c : cells)
        os << format_double(c.snr_db) << ',' << c.user << ',' << to_string(c.detector) << ','
           << to_string(c.ablation) << ',' << c.trials << ',' << format_double(c.mean_ber) << ','
           << format_double(c.sd_ber) << ',' << c.total_bits << '\n';
    return os.str();
}

namespace {

std::vector<int> full_dims(int width, const std::vector<int> &hidden) {
    std::vector<int> dims{width};
    dims.insert(dims.end(), hidden.begin(), hidden.end());
    return dims;
}

struct Trial {  // one synthesized record and its four design views
    TransmissionRecord rec;
    Mat wide_train, wide_detect, real_train, real_detect;
};

Mat real_rows(const CMat &x) {  // [Re r | Im r] per symbol (eval.cpp:70-75)
    Mat out(x.rows(), 2 * x.cols());
    for (Eigen::Index t = 0; t < x.rows(); ++t)
        for (Eigen::Index m = 0; m < x.cols(); ++m) {
            out(t, m) = x(t, m).real();
            out(t, x.cols() + m) = x(t, m).imag();
        }
    return out;
}

// detect_user (eval.cpp:100-166): per (user, detector, ablation) the fit /
// init / train / detect chain, every step on the device
CVec sweep_detect(const SweepOptions &o, const Trial &tr, int user, DetectorId det, Ablation abl,
                  std::uint64_t tag) {
    const CVec y = tr.rec.train_symbols.col(user - 1);
    if (abl != Ablation::SymmetryOff) {
        Mat design;
        Vec targets;
        if (abl == Ablation::SymmetryOn) {
            design = tr.wide_train;
            targets = widen_targets(y);
        } else {
            const Eigen::Index half = tr.rec.train_rx.rows() / 2;
            design = widen_design(tr.rec.train_rx.topRows(half));
            targets = widen_targets(y.head(half));
        }
        const LlsWeights w = lls::fit(design, targets, user);
        if (det == DetectorId::Lls) return lls::predict(w, tr.wide_detect);
        Rng init_rng(substream_seed(o.master_seed, mix_tag(tag, 11)));
        HybridNetParams net =
            hybrid_nn::init_params(full_dims(static_cast<int>(design.cols()), o.hidden_dims), w, init_rng);
        TrainConfig tc = o.train;
        tc.shuffle_seed = substream_seed(o.master_seed, mix_tag(tag, 12));
        const WidenedDataset ds{std::move(design), std::move(targets), user};
        hybrid_nn::train(net, ds, tc);
        return hybrid_nn::detect(net, tr.wide_detect);
    }
    // symmetry off: Re and Im get independently fitted / trained slots on the
    // non-widened rows
    const Vec y_re = y.real(), y_im = y.imag();
    const LlsWeights w_re = lls::fit(tr.real_train, y_re, user), w_im = lls::fit(tr.real_train, y_im, user);
    Vec pr, pi;
    if (det == DetectorId::Lls) {
        pr = linear_forward(w_re.w, tr.real_detect);
        pi = linear_forward(w_im.w, tr.real_detect);
    } else {
        const auto dims = full_dims(static_cast<int>(tr.real_train.cols()), o.hidden_dims);
        auto slot = [&](const LlsWeights &w, const Vec &t, std::uint64_t k) {
            Rng init_rng(substream_seed(o.master_seed, mix_tag(tag, 11, k)));
            HybridNetParams net = hybrid_nn::init_params(dims, w, init_rng);
            TrainConfig tc = o.train;
            tc.shuffle_seed = substream_seed(o.master_seed, mix_tag(tag, 12, k));
            const WidenedDataset ds{tr.real_train, t, user};
            hybrid_nn::train(net, ds, tc);
            return hybrid_nn::forward(net, tr.real_detect);
        };
        pr = slot(w_re, y_re, 1);
        pi = slot(w_im, y_im, 2);
    }
    CVec out(pr.size());
    for (Eigen::Index t = 0; t < pr.size(); ++t) out[t] = cplx(pr[t], pi[t]);
    return out;
}

}  // namespace

BerReport run_noise_sweep(const SweepOptions &o) {  // eval.cpp:170-254
    if (o.snr_list.empty()) throw config_error("run_noise_sweep: empty SNR list");
    if (o.trials < 1) throw config_error("run_noise_sweep: trials must be >= 1");
    if (o.detectors.empty()) throw config_error("run_noise_sweep: no detectors");
    o.scenario.validate();
    std::vector<int> users = o.users;
    if (users.empty())
        for (int u = 1; u <= o.scenario.num_users; ++u) users.push_back(u);
    for (int u : users)
        if (u < 1 || u > o.scenario.num_users) throw config_error("run_noise_sweep: user index out of range");

    BerReport rep;
    rep.master_seed = o.master_seed;
    rep.trials = o.trials;
    // cell order: snr -> detector -> ablation -> user
    struct Key {
        std::size_t si, di, ai, ui;
    };
    std::vector<Key> keys;
    for (std::size_t si = 0; si < o.snr_list.size(); ++si)
        for (std::size_t di = 0; di < o.detectors.size(); ++di)
            for (std::size_t ai = 0; ai < o.ablations.size(); ++ai)
                for (std::size_t ui = 0; ui < users.size(); ++ui) keys.push_back({si, di, ai, ui});
    for (const Key &k : keys) {
        BerCell c;
        c.snr_db = o.snr_list[k.si];
        c.user = users[k.ui];
        c.detector = o.detectors[k.di];
        c.ablation = o.ablations[k.ai];
        c.trials = o.trials;
        c.total_bits = 2LL * o.scenario.data_symbols * o.trials;
        rep.cells.push_back(std::move(c));
    }
    for (std::size_t si = 0; si < o.snr_list.size(); ++si) {
        ScenarioConfig cfg = o.scenario;
        cfg.snr_db = o.snr_list[si];
        for (int trial = 0; trial < o.trials; ++trial) {
            const auto tu = static_cast<std::uint64_t>(trial);
            SeedBundle seeds;  // eval.cpp:212-219
            seeds.symbols = substream_seed(o.master_seed, 1);
            seeds.channel = o.fresh_channel_per_trial ? substream_seed(o.master_seed, mix_tag(2, tu))
                                                      : substream_seed(o.master_seed, 2);
            seeds.noise = substream_seed(o.master_seed, mix_tag(3, si, tu));
            Trial tr{synthesize(cfg, seeds), {}, {}, {}, {}};
            tr.wide_train = widen_design(tr.rec.train_rx);
            tr.wide_detect = widen_design(tr.rec.data_rx);
            tr.real_train = real_rows(tr.rec.train_rx);
            tr.real_detect = real_rows(tr.rec.data_rx);
            for (std::size_t i = 0; i < keys.size(); ++i) {
                const Key &k = keys[i];
                if (k.si != si) continue;
                BerCell &cell = rep.cells[i];
                const std::uint64_t tag =
                    mix_tag(si, tu, static_cast<std::uint64_t>(cell.user), (k.di << 8) | k.ai);
                const CVec pred = sweep_detect(o, tr, cell.user, cell.detector, cell.ablation, tag);
                cell.per_trial_ber.push_back(bit_error_rate(
                    hard_decision_qpsk(pred), hard_decision_qpsk(tr.rec.data_symbols.col(cell.user - 1))));
            }
        }
    }
    for (BerCell &c : rep.cells) {  // mean and population SD (eval.cpp:244-252)
        double sum = 0.0;
        for (double b : c.per_trial_ber) sum += b;
        c.mean_ber = sum / static_cast<double>(c.per_trial_ber.size());
        double var = 0.0;
        for (double b : c.per_trial_ber) var += (b - c.mean_ber) * (b - c.mean_ber);
        c.sd_ber = std::sqrt(var / static_cast<double>(c.per_trial_ber.size()));
    }
    return rep;
}

}  // namespace noma
