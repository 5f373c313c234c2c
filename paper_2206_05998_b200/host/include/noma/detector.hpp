// The reference detector's C++ API (proj/include/noma/*.hpp), declared for
// builds that do not have the reference headers at hand.
//
// libnoma_host is normally compiled against the reference's own headers,
// unmodified (host/Makefile: -I/root/reference/proj/include); this file is
// the stand-in the compat/noma/*.hpp forwarding headers pull in when that
// tree is absent.  Every declaration matches the reference's member for
// member (same types, same order, same defaults), so the two builds are
// interchangeable.  Containers are Eigen's (the subset in host/eigen when
// Eigen 3.4 is not installed).
//
//   reference header          declarations here
//   types.hpp:9-17            Mat, Vec, CMat, CVec, MatF, VecF, BitMat, cplx
//   errors.hpp:8-35           dimension_error ... truncation_error
//   rng.hpp:10-67             splitmix64, substream_seed, Rng
//   format.hpp:9-13           format_double
//   channel_sim.hpp:11-76     Modulation, ScenarioConfig, SeedBundle,
//                             TransmissionRecord, power_profile, gen_symbols,
//                             gen_channel, synthesize
//   iq_transform.hpp:13-29    WidenedDataset, widen_*, narrow_predictions
//   lls.hpp:9-24              LlsWeights, lls::fit, lls::predict
//   hybrid_nn.hpp:15-75       HybridNetParams, Gradients, AdamState,
//                             TrainConfig, hybrid_nn::*
//   fused_inference.hpp:9-64  kFusedMaxWidth, kFusedTileRows, FusedPlan,
//                             BenchReport, fused::*
//   eval.hpp:11-95            DetectorId, Ablation, hard decisions, BER,
//                             SweepOptions, BerCell, BerReport, run_noise_sweep
#pragma once

#include <Eigen/Dense>
#include <charconv>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <numbers>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace noma {

// ------------------------------------------------------------------ types
using Mat = Eigen::MatrixXd;
using Vec = Eigen::VectorXd;
using CMat = Eigen::MatrixXcd;
using CVec = Eigen::VectorXcd;
using MatF = Eigen::MatrixXf;
using VecF = Eigen::VectorXf;
using BitMat = Eigen::Matrix<std::uint8_t, Eigen::Dynamic, Eigen::Dynamic>;
using cplx = std::complex<double>;

// ----------------------------------------------------------------- errors
struct dimension_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct config_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ill_conditioned_error : std::runtime_error {
    double gram_condition;
    explicit ill_conditioned_error(const std::string &msg, double cond)
        : std::runtime_error(msg), gram_condition(cond) {}
};
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct format_error : io_error {
    using io_error::io_error;
};
struct truncation_error : io_error {
    using io_error::io_error;
};

// -------------------------------------------------------------------- rng
// Bit-exact contract: splitmix64 seeding, xoshiro256++,
// 53-bit uniform, multiply-shift below(), Box-Muller cosine half.
inline std::uint64_t splitmix64(std::uint64_t &state) {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline std::uint64_t substream_seed(std::uint64_t master, std::uint64_t tag) {
    std::uint64_t s = master;
    const std::uint64_t first = splitmix64(s);
    s = first ^ (tag * 0xD1B54A32D192ED03ULL + 0x8BB84B93962EACC9ULL);
    return splitmix64(s);
}
class Rng {
  public:
    explicit Rng(std::uint64_t seed) {
        std::uint64_t sm = seed;
        for (std::uint64_t &w : state_) w = splitmix64(sm);
    }
    std::uint64_t next_u64() {
        const std::uint64_t out = rotl(state_[0] + state_[3], 23) + state_[0];
        const std::uint64_t t = state_[1] << 17;
        state_[2] ^= state_[0];
        state_[3] ^= state_[1];
        state_[1] ^= state_[2];
        state_[0] ^= state_[3];
        state_[2] ^= t;
        state_[3] = rotl(state_[3], 45);
        return out;
    }
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    std::uint64_t below(std::uint64_t bound) {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * bound) >> 64);
    }
    double gaussian() {
        const double u1 = 1.0 - uniform();
        const double u2 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * std::numbers::pi * u2);
    }

  private:
    static std::uint64_t rotl(std::uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    std::uint64_t state_[4];
};

// ----------------------------------------------------------------- format
inline std::string format_double(double v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

// ------------------------------------------------------------ channel_sim
enum class Modulation { Qpsk };

struct ScenarioConfig {
    int num_users = 6;
    int num_antennas = 4;
    int train_symbols = 685;
    int data_symbols = 3840;
    double power_step_db = 3.0;
    double snr_db = std::numeric_limits<double>::infinity();
    double rx_nonlinearity_gain = 0.0;
    Modulation modulation = Modulation::Qpsk;
    std::uint64_t seed = 0;

    void validate() const;
};

struct SeedBundle {
    std::uint64_t symbols;
    std::uint64_t channel;
    std::uint64_t noise;

    static SeedBundle from_master(std::uint64_t master) {
        return {substream_seed(master, 1), substream_seed(master, 2), substream_seed(master, 3)};
    }
};

struct TransmissionRecord {
    CMat channel;
    Vec powers;
    CMat train_rx;
    CMat train_symbols;
    CMat data_rx;
    CMat data_symbols;
    double noise_power = 0.0;
};

Vec power_profile(int num_users, double step_db);
CMat gen_symbols(int num_users, int num_symbols, Modulation mod, Rng &rng);
CMat gen_channel(int num_users, int num_antennas, Rng &rng);
TransmissionRecord synthesize(const ScenarioConfig &cfg);
TransmissionRecord synthesize(const ScenarioConfig &cfg, const SeedBundle &seeds);

// ----------------------------------------------------------- iq_transform
struct WidenedDataset {
    Mat design;
    std::optional<Vec> targets;
    int user_index = 0;
};

Mat widen_design(const CMat &x);
Vec widen_targets(const CVec &y);
WidenedDataset widen_dataset(const CMat &x, const std::optional<CVec> &y = std::nullopt, int user_index = 0);
CVec narrow_predictions(const Vec &yhat);

// -------------------------------------------------------------------- lls
struct LlsWeights {
    Vec w;
    int user_index = 0;
    double gram_condition = 0.0;
};

namespace lls {
LlsWeights fit(const Mat &design, const Vec &targets, int user_index = 0);
LlsWeights fit(const WidenedDataset &train);
CVec predict(const LlsWeights &weights, const Mat &widened_detect);
}  // namespace lls

// -------------------------------------------------------------- hybrid_nn
struct HybridNetParams {
    Vec w0;
    std::vector<Mat> weights;
    std::vector<Vec> biases;
    Vec final_weights;
    std::vector<int> dims;

    std::size_t trainable_count() const;
};

struct Gradients {
    std::vector<Mat> weights;
    std::vector<Vec> biases;
    Vec final_weights;
};

struct AdamState {
    Gradients m;
    Gradients v;
    long step = 0;
    double lr = 0.005;
    double beta1 = 0.9;
    double beta2 = 0.999;
    double eps = 1e-8;

    static AdamState init(const HybridNetParams &params, double lr);
};

struct TrainConfig {
    int epochs = 50;
    int batch_size = 128;
    double lr = 0.005;
    std::uint64_t shuffle_seed = 0;
};

namespace hybrid_nn {
HybridNetParams init_params(const std::vector<int> &dims, const LlsWeights &w0, Rng &rng);
Vec forward(const HybridNetParams &params, const Mat &x);
std::pair<double, Gradients> loss_and_grad(const HybridNetParams &params, const Mat &x, const Vec &y);
void adam_step(HybridNetParams &params, const Gradients &grads, AdamState &state);
std::vector<double> train(HybridNetParams &params, const WidenedDataset &train_set, const TrainConfig &cfg);
CVec detect(const HybridNetParams &params, const Mat &widened_detect);
}  // namespace hybrid_nn

// -------------------------------------------------------- fused_inference
inline constexpr int kFusedMaxWidth = 128;
inline constexpr int kFusedTileRows = 8;

struct FusedPlan {
    std::vector<int> dims;
    std::vector<int> padded;
    std::vector<double> buffer;
    std::vector<float> buffer_f32;
    bool fused = false;
    int max_width = 0;

    HybridNetParams unpack() const;
};

struct BenchReport {
    std::vector<int> dims;
    int batch = 0;
    int repeats = 0;
    double fused_ns_per_sample = 0.0;
    double naive_ns_per_sample = 0.0;
    double fallback_ns_per_sample = 0.0;
    double speedup_vs_naive = 0.0;
    std::string machine;

    std::string to_csv(bool with_header) const;
};

namespace fused {
FusedPlan build_plan(const HybridNetParams &params);
Vec fused_forward(const FusedPlan &plan, const Mat &x);
void fused_forward_into(const FusedPlan &plan, const Mat &x, Vec &out);
VecF fused_forward_f32(const FusedPlan &plan, const MatF &x);
BenchReport bench_compare(const FusedPlan &plan, int batch, int repeats);
}  // namespace fused

// ------------------------------------------------------------------- eval
enum class DetectorId { Lls, HybridNn };
enum class Ablation { SymmetryOn, SymmetryOff, SymmetryOnHalfData };

std::string to_string(DetectorId id);
std::string to_string(Ablation a);
DetectorId detector_from_string(const std::string &s);
Ablation ablation_from_string(const std::string &s);
BitMat hard_decision_qpsk(const CVec &symbols);
CVec map_qpsk_bits(const BitMat &bits);
double bit_error_rate(const BitMat &predicted, const BitMat &truth);

struct SweepOptions {
    ScenarioConfig scenario;
    std::vector<double> snr_list;
    int trials = 20;
    std::vector<DetectorId> detectors{DetectorId::Lls, DetectorId::HybridNn};
    std::vector<Ablation> ablations{Ablation::SymmetryOn};
    std::vector<int> users;
    std::vector<int> hidden_dims{64, 64, 64};
    TrainConfig train;
    bool fresh_channel_per_trial = true;
    std::uint64_t master_seed = 0;
};

struct BerCell {
    double snr_db = 0.0;
    int user = 0;
    DetectorId detector = DetectorId::Lls;
    Ablation ablation = Ablation::SymmetryOn;
    int trials = 0;
    double mean_ber = 0.0;
    double sd_ber = 0.0;
    long long total_bits = 0;
    std::vector<double> per_trial_ber;
};

struct BerReport {
    std::vector<BerCell> cells;
    std::uint64_t master_seed = 0;
    int trials = 0;
    std::string config_digest;
    std::string note;

    std::string to_csv() const;
};

BerReport run_noise_sweep(const SweepOptions &opts);

}  // namespace noma
