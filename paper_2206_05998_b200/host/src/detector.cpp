// noma:: detector API implemented over the C-ABI (include/noma_cuda.h).
// Each function restates the reference's contract (argument checks, error
// types, output shapes) and delegates all arithmetic to the device.
#include "noma/detector.hpp"

#include <cmath>
#include <mutex>

#include "noma_cuda.h"

namespace noma {
namespace {

noma_ctx_t ctx() {
    static noma_ctx_t c = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        if (noma_ctx_create(0, &c) != NOMA_OK) c = nullptr;
    });
    if (!c) throw device_error("noma: no CUDA device (the B200 path has no CPU fallback)");
    return c;
}

[[noreturn]] void raise(int st, const char *what, double cond = 0.0) {
    const std::string msg = std::string(what) + ": " + noma_ctx_last_error(ctx());
    switch (st) {
        case NOMA_ERR_DIMENSION: throw dimension_error(msg);
        case NOMA_ERR_CONFIG: throw config_error(msg);
        case NOMA_ERR_ILL_CONDITIONED: throw ill_conditioned_error(msg, cond);
        case NOMA_ERR_UNSUPPORTED: throw unsupported_error(msg);
        default: throw device_error(msg);
    }
}

void check(int st, const char *what) {
    if (st != NOMA_OK) raise(st, what);
}

noma_net_desc desc_of(const std::vector<int> &dims) {
    noma_net_desc d{};
    if (dims.empty() || dims.size() > NOMA_MAX_DIMS) throw dimension_error("bad dims");
    d.ndims = static_cast<int>(dims.size());
    for (std::size_t i = 0; i < dims.size(); ++i) d.dims[i] = dims[i];
    return d;
}

// A real design is "widened" when every row pair is [a, b] / [b, -a]
// (iq_transform.cpp:17-20); the device then works on the complex rows.
bool is_widened(const Mat &x) {
    if (x.rows() % 2 || x.cols() % 2 || x.rows() == 0) return false;
    const dense::Index m = x.cols() / 2;
    for (dense::Index t = 0; 2 * t < x.rows(); ++t)
        for (dense::Index j = 0; j < m; ++j)
            if (x(2 * t + 1, j) != x(2 * t, m + j) || x(2 * t + 1, m + j) != -x(2 * t, j))
                return false;
    return true;
}

// complex rows [n/2][m] (interleaved) of a widened design
std::vector<double> complex_rows(const Mat &x) {
    const dense::Index n = x.rows() / 2, m = x.cols() / 2;
    std::vector<double> out(static_cast<std::size_t>(n * m * 2));
    for (dense::Index t = 0; t < n; ++t)
        for (dense::Index j = 0; j < m; ++j) {
            out[(t * m + j) * 2] = x(2 * t, j);
            out[(t * m + j) * 2 + 1] = x(2 * t, m + j);
        }
    return out;
}

std::vector<double> row_major(const Mat &x) {
    std::vector<double> out(static_cast<std::size_t>(x.size()));
    for (dense::Index r = 0; r < x.rows(); ++r)
        for (dense::Index c = 0; c < x.cols(); ++c) out[r * x.cols() + c] = x(r, c);
    return out;
}

int pad8(int w) { return ((w + 7) / 8) * 8; }

std::vector<float> plan_of(const HybridNetParams &p) {
    const noma_net_desc d = desc_of(p.dims);
    std::vector<float> plan(static_cast<std::size_t>(noma_plan_size(&d)), 0.0f);
    for (int c = 0; c < p.dims[0]; ++c) plan[c] = static_cast<float>(p.w0[c]);
    std::size_t off = pad8(p.dims[0]);
    for (std::size_t l = 1; l < p.dims.size(); ++l) {
        const int pin = pad8(p.dims[l - 1]);
        for (int j = 0; j < p.dims[l]; ++j)
            for (int c = 0; c < p.dims[l - 1]; ++c)
                plan[off + j * pin + c] = static_cast<float>(p.weights[l - 1](j, c));
        off += static_cast<std::size_t>(p.dims[l]) * pin;
        for (int j = 0; j < p.dims[l]; ++j) plan[off + j] = static_cast<float>(p.biases[l - 1][j]);
        off += pad8(p.dims[l]);
    }
    for (int j = 0; j < p.dims.back(); ++j) plan[off + j] = static_cast<float>(p.final_weights[j]);
    return plan;
}

void params_from_plan(HybridNetParams &p, const std::vector<float> &plan) {
    std::size_t off = pad8(p.dims[0]);
    for (std::size_t l = 1; l < p.dims.size(); ++l) {
        const int pin = pad8(p.dims[l - 1]);
        for (int j = 0; j < p.dims[l]; ++j)
            for (int c = 0; c < p.dims[l - 1]; ++c) p.weights[l - 1](j, c) = plan[off + j * pin + c];
        off += static_cast<std::size_t>(p.dims[l]) * pin;
        for (int j = 0; j < p.dims[l]; ++j) p.biases[l - 1][j] = plan[off + j];
        off += pad8(p.dims[l]);
    }
    for (int j = 0; j < p.dims.back(); ++j) p.final_weights[j] = plan[off + j];
}

// Device inference of a plan over real rows (REAL layout), FP32.
std::vector<float> infer_rows(const std::vector<int> &dims, const std::vector<float> &plan,
                              const std::vector<float> &rows_f32, int nrows) {
    const noma_net_desc d = desc_of(dims);
    std::vector<float> out(static_cast<std::size_t>(nrows));
    check(noma_detect(ctx(), &d, NOMA_LAYOUT_REAL, 1, 1, nrows, rows_f32.data(), plan.data(),
                      nullptr, out.data(), nullptr, nullptr, nullptr, NOMA_MEM_HOST),
          "forward");
    return out;
}

}  // namespace

// ---------------------------------------------------------------- RNG
std::uint64_t splitmix64(std::uint64_t &state) {  // rng.hpp:10-15
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

std::uint64_t substream_seed(std::uint64_t master, std::uint64_t tag) {  // rng.hpp:18-23
    std::uint64_t s = master;
    const std::uint64_t a = splitmix64(s);
    s = a ^ (tag * 0xD1B54A32D192ED03ULL + 0x8BB84B93962EACC9ULL);
    return splitmix64(s);
}

Rng::Rng(std::uint64_t seed) {  // rng.hpp:30-33
    std::uint64_t sm = seed;
    for (auto &w : state) w = splitmix64(sm);
}

std::uint64_t Rng::next_u64() {  // rng.hpp:35-45
    auto rotl = [](std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); };
    const std::uint64_t result = rotl(state[0] + state[3], 23) + state[0];
    const std::uint64_t t = state[1] << 17;
    state[2] ^= state[0];
    state[3] ^= state[1];
    state[1] ^= state[2];
    state[0] ^= state[3];
    state[2] ^= t;
    state[3] = rotl(state[3], 45);
    return result;
}

// ---------------------------------------------------------------- IQ
Mat widen_design(const CMat &x) {  // iq_transform.cpp:7-24 (layout op)
    if (x.rows() == 0 || x.cols() == 0) throw dimension_error("widen_design: empty input");
    const dense::Index n = x.rows(), m = x.cols();
    Mat out(2 * n, 2 * m);
    for (dense::Index t = 0; t < n; ++t)
        for (dense::Index j = 0; j < m; ++j) {
            out(2 * t, j) = x(t, j).real();
            out(2 * t, m + j) = x(t, j).imag();
            out(2 * t + 1, j) = x(t, j).imag();
            out(2 * t + 1, m + j) = -x(t, j).real();
        }
    return out;
}

Vec widen_targets(const CVec &y) {
    Vec out(2 * y.size());
    for (dense::Index t = 0; t < y.size(); ++t) {
        out[2 * t] = y[t].real();
        out[2 * t + 1] = y[t].imag();
    }
    return out;
}

WidenedDataset widen_dataset(const CMat &x, const std::optional<CVec> &y, int user_index) {
    WidenedDataset ds;
    ds.design = widen_design(x);
    if (y) {
        if (y->size() != x.rows())
            throw dimension_error("widen_dataset: target length does not match rows");
        ds.targets = widen_targets(*y);
        ds.user_index = user_index;
    }
    return ds;
}

CVec narrow_predictions(const Vec &yhat) {
    if (yhat.size() % 2 != 0) throw dimension_error("narrow_predictions: length must be even");
    CVec out(yhat.size() / 2);
    for (dense::Index t = 0; t < out.size(); ++t) out[t] = cplx(yhat[2 * t], yhat[2 * t + 1]);
    return out;
}

// ---------------------------------------------------------------- LLS
namespace lls {

LlsWeights fit(const Mat &design, const Vec &targets, int user_index) {  // lls.cpp:10-54
    if (design.rows() < design.cols())
        throw dimension_error("lls::fit: system must be over-determined");
    if (design.rows() != targets.size())
        throw dimension_error("lls::fit: design rows and target length differ");
    const bool wid = is_widened(design);
    std::vector<double> x = wid ? complex_rows(design) : row_major(design);
    std::vector<double> y(targets.data(), targets.data() + targets.size());  // interleaved == complex
    noma_dataset ds{wid ? NOMA_LAYOUT_WIDEN_COMPLEX : NOMA_LAYOUT_REAL, 1, 1,
                    static_cast<int>(design.rows()), static_cast<int>(design.cols()), x.data(),
                    y.data()};
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

LlsWeights fit(const WidenedDataset &train) {
    if (!train.targets) throw dimension_error("lls::fit: training set has no targets");
    return fit(train.design, *train.targets, train.user_index);
}

CVec predict(const LlsWeights &weights, const Mat &widened_detect) {  // lls.cpp:62-66
    if (widened_detect.cols() != weights.w.size())
        throw dimension_error("lls::predict: column count does not match weights");
    if (widened_detect.rows() % 2 != 0)
        throw dimension_error("narrow_predictions: length must be even");
    std::vector<double> x = row_major(widened_detect);
    Vec yhat(widened_detect.rows());
    check(noma_lls_predict(ctx(), NOMA_LAYOUT_REAL, 1, 1, static_cast<int>(widened_detect.rows()),
                           static_cast<int>(widened_detect.cols()), x.data(), weights.w.data(),
                           yhat.data(), NOMA_MEM_HOST),
          "lls::predict");
    return narrow_predictions(yhat);
}

}  // namespace lls

// --------------------------------------------------------- hybrid_nn
std::size_t HybridNetParams::trainable_count() const {  // hybrid_nn.cpp:11-16
    std::size_t n = final_weights.size();
    for (std::size_t i = 0; i < weights.size(); ++i) n += weights[i].size() + biases[i].size();
    return n;
}

namespace hybrid_nn {

HybridNetParams init_params(const std::vector<int> &dims, const LlsWeights &w0, Rng &rng) {
    if (dims.empty() || dims[0] != w0.w.size())
        throw dimension_error("init_params: dims[0] must equal the w0 length");
    for (int d : dims)
        if (d < 1) throw dimension_error("init_params: layer widths must be >= 1");
    const noma_net_desc d = desc_of(dims);
    std::vector<double> theta(static_cast<std::size_t>(noma_param_count(&d)));
    check(noma_init_params_state(ctx(), &d, 1, rng.state, w0.w.data(), nullptr, theta.data(),
                                 NOMA_MEM_HOST),
          "init_params");
    HybridNetParams p;
    p.dims = dims;
    p.w0 = w0.w;
    std::size_t off = 0;
    for (std::size_t l = 1; l < dims.size(); ++l) {
        Mat w(dims[l], dims[l - 1]);
        for (int r = 0; r < dims[l]; ++r)
            for (int c = 0; c < dims[l - 1]; ++c) w(r, c) = theta[off++];
        p.weights.push_back(std::move(w));
        Vec b(dims[l]);
        for (int j = 0; j < dims[l]; ++j) b[j] = theta[off++];
        p.biases.push_back(std::move(b));
    }
    p.final_weights = Vec(dims.back());
    return p;
}

Vec forward(const HybridNetParams &p, const Mat &x) {
    if (x.cols() != p.w0.size()) throw dimension_error("forward: input width does not match network");
    std::vector<float> rows(static_cast<std::size_t>(x.size()));
    for (dense::Index r = 0; r < x.rows(); ++r)
        for (dense::Index c = 0; c < x.cols(); ++c) rows[r * x.cols() + c] = static_cast<float>(x(r, c));
    const std::vector<float> y = infer_rows(p.dims, plan_of(p), rows, static_cast<int>(x.rows()));
    Vec out(x.rows());
    for (dense::Index r = 0; r < x.rows(); ++r) out[r] = y[r];
    return out;
}

std::vector<double> train(HybridNetParams &p, const WidenedDataset &set, const TrainConfig &cfg) {
    if (!set.targets) throw dimension_error("train: training set has no targets");
    if (set.design.rows() == 0) throw dimension_error("train: empty training set");
    if (cfg.epochs < 0 || cfg.batch_size < 1 || cfg.lr <= 0.0)
        throw config_error("train: invalid training configuration");
    const bool wid = is_widened(set.design);
    std::vector<double> x = wid ? complex_rows(set.design) : row_major(set.design);
    std::vector<double> y(set.targets->data(), set.targets->data() + set.targets->size());
    noma_dataset ds{wid ? NOMA_LAYOUT_WIDEN_COMPLEX : NOMA_LAYOUT_REAL, 1, 1,
                    static_cast<int>(set.design.rows()), static_cast<int>(set.design.cols()),
                    x.data(), y.data()};
    const noma_net_desc d = desc_of(p.dims);
    noma_train_cfg tc{cfg.epochs, cfg.batch_size, cfg.lr, 0.9, 0.999, 1e-8};
    std::vector<float> plan = plan_of(p);
    std::vector<double> trace(static_cast<std::size_t>(cfg.epochs));
    std::uint64_t seed = cfg.shuffle_seed;
    check(noma_train(ctx(), &ds, &d, &tc, p.w0.data(), plan.data(), &seed,
                     cfg.epochs > 0 ? trace.data() : nullptr, nullptr, NOMA_MEM_HOST),
          "train");
    params_from_plan(p, plan);
    return trace;
}

CVec detect(const HybridNetParams &p, const Mat &widened_detect) {
    return narrow_predictions(forward(p, widened_detect));
}

}  // namespace hybrid_nn

// ------------------------------------------------------------- fused
FusedPlan fused::build_plan(const HybridNetParams &params) {  // fused_inference.cpp:174-203
    FusedPlan plan;
    plan.dims = params.dims;
    plan.max_width = *std::max_element(params.dims.begin(), params.dims.end());
    plan.fused = plan.max_width <= kFusedMaxWidth;
    for (int d : params.dims) plan.padded.push_back(pad8(d));
    plan.buffer_f32 = plan_of(params);
    // FP64 copy in the same layout
    plan.buffer.assign(plan.buffer_f32.size(), 0.0);
    for (int c = 0; c < params.dims[0]; ++c) plan.buffer[c] = params.w0[c];
    std::size_t off = pad8(params.dims[0]);
    for (std::size_t l = 1; l < params.dims.size(); ++l) {
        const int pin = pad8(params.dims[l - 1]);
        for (int j = 0; j < params.dims[l]; ++j)
            for (int c = 0; c < params.dims[l - 1]; ++c)
                plan.buffer[off + j * pin + c] = params.weights[l - 1](j, c);
        off += static_cast<std::size_t>(params.dims[l]) * pin;
        for (int j = 0; j < params.dims[l]; ++j) plan.buffer[off + j] = params.biases[l - 1][j];
        off += pad8(params.dims[l]);
    }
    for (int j = 0; j < params.dims.back(); ++j) plan.buffer[off + j] = params.final_weights[j];
    return plan;
}

HybridNetParams FusedPlan::unpack() const {  // fused_inference.cpp:155-170
    HybridNetParams p;
    p.dims = dims;
    p.w0 = Vec(dims[0]);
    for (int c = 0; c < dims[0]; ++c) p.w0[c] = buffer[c];
    std::size_t off = pad8(dims[0]);
    for (std::size_t l = 1; l < dims.size(); ++l) {
        const int pin = pad8(dims[l - 1]);
        Mat w(dims[l], dims[l - 1]);
        for (int j = 0; j < dims[l]; ++j)
            for (int c = 0; c < dims[l - 1]; ++c) w(j, c) = buffer[off + j * pin + c];
        p.weights.push_back(std::move(w));
        off += static_cast<std::size_t>(dims[l]) * pin;
        Vec b(dims[l]);
        for (int j = 0; j < dims[l]; ++j) b[j] = buffer[off + j];
        p.biases.push_back(std::move(b));
        off += pad8(dims[l]);
    }
    p.final_weights = Vec(dims.back());
    for (int j = 0; j < dims.back(); ++j) p.final_weights[j] = buffer[off + j];
    return p;
}

VecF fused::fused_forward_f32(const FusedPlan &plan, const MatF &x) {  // :222-231
    if (x.cols() != plan.dims[0])
        throw dimension_error("fused_forward_f32: input width does not match plan");
    std::vector<float> rows(static_cast<std::size_t>(x.size()));
    for (dense::Index r = 0; r < x.rows(); ++r)
        for (dense::Index c = 0; c < x.cols(); ++c) rows[r * x.cols() + c] = x(r, c);
    const std::vector<float> y = infer_rows(plan.dims, plan.buffer_f32, rows, static_cast<int>(x.rows()));
    VecF out(x.rows());
    for (dense::Index r = 0; r < x.rows(); ++r) out[r] = y[r];
    return out;
}

// ------------------------------------------------------------- eval
BitMat hard_decision_qpsk(const CVec &symbols) {  // eval.cpp:38-45 (sign test)
    BitMat bits(symbols.size(), 2);
    for (dense::Index t = 0; t < symbols.size(); ++t) {
        bits(t, 0) = symbols[t].real() < 0.0 ? 1 : 0;
        bits(t, 1) = symbols[t].imag() < 0.0 ? 1 : 0;
    }
    return bits;
}

double bit_error_rate(const BitMat &predicted, const BitMat &truth) {  // eval.cpp:56-65
    if (predicted.rows() != truth.rows() || predicted.cols() != truth.cols())
        throw dimension_error("bit_error_rate: shape mismatch");
    if (predicted.size() == 0) throw dimension_error("bit_error_rate: empty input");
    long long errors = 0;
    for (dense::Index i = 0; i < predicted.size(); ++i) errors += predicted.data()[i] != truth.data()[i];
    return static_cast<double>(errors) / static_cast<double>(predicted.size());
}

}  // namespace noma
