// noma:: detector API on the B200 -- the host side above the C-ABI.
//
// Mirrors the reference's public surface for the hot path (proj/include/noma:
// types.hpp, errors.hpp, rng.hpp, iq_transform.hpp, lls.hpp, hybrid_nn.hpp,
// fused_inference.hpp, eval.hpp:27-33): same names, argument meaning and
// exceptions, so code written against the reference links against this
// library instead.  Every compute call goes to the GPU through
// include/noma_cuda.h; there is no CPU compute path.  The dense containers
// are column-major with contiguous data() exactly like Eigen's owning
// Matrix, so the pointer/size contract holds if real Eigen is dropped in.
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "noma/dense.hpp"

namespace noma {

using Mat = dense::Matrix<double>;
using Vec = dense::Vector<double>;
using CMat = dense::Matrix<std::complex<double>>;
using CVec = dense::Vector<std::complex<double>>;
using MatF = dense::Matrix<float>;
using VecF = dense::Vector<float>;
using BitMat = dense::Matrix<std::uint8_t>;
using cplx = std::complex<double>;

// ---- errors (reference errors.hpp:8-35) ------------------------------------
struct dimension_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct config_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct ill_conditioned_error : std::runtime_error {
    double gram_condition;
    ill_conditioned_error(const std::string &msg, double cond)
        : std::runtime_error(msg), gram_condition(cond) {}
};
// Shapes outside the device kernels (layer wider than 128, batch > 128, ...).
struct unsupported_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- RNG handle (reference rng.hpp:28-67: xoshiro256++ state) -------------
// Only the state is kept host-side; draws for init_params happen on device
// and advance this state exactly as the reference's Rng& would be advanced.
std::uint64_t splitmix64(std::uint64_t &state);
std::uint64_t substream_seed(std::uint64_t master, std::uint64_t tag);
class Rng {
  public:
    explicit Rng(std::uint64_t seed);
    std::uint64_t next_u64();
    std::uint64_t state[4];
};

// ---- IQ transform (reference iq_transform.hpp:13-29) -----------------------
struct WidenedDataset {
    Mat design;
    std::optional<Vec> targets;
    int user_index = 0;
};
Mat widen_design(const CMat &x);
Vec widen_targets(const CVec &y);
WidenedDataset widen_dataset(const CMat &x, const std::optional<CVec> &y = std::nullopt,
                             int user_index = 0);
CVec narrow_predictions(const Vec &yhat);

// ---- LLS (reference lls.hpp:9-24) ------------------------------------------
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

// ---- hybrid network (reference hybrid_nn.hpp:15-75) ------------------------
struct HybridNetParams {
    Vec w0;
    std::vector<Mat> weights;  // W_n: L_n x L_{n-1}
    std::vector<Vec> biases;
    Vec final_weights;
    std::vector<int> dims;
    std::size_t trainable_count() const;
};
struct TrainConfig {
    int epochs = 50;
    int batch_size = 128;
    double lr = 0.005;
    std::uint64_t shuffle_seed = 0;
};
namespace hybrid_nn {
HybridNetParams init_params(const std::vector<int> &dims, const LlsWeights &w0, Rng &rng);
// FP32 device inference (the reference's FP64 forward within the FP32
// tolerance of fused_forward_f32, test_fused.cpp:121-131).
Vec forward(const HybridNetParams &params, const Mat &x);
std::vector<double> train(HybridNetParams &params, const WidenedDataset &train_set,
                          const TrainConfig &cfg);
CVec detect(const HybridNetParams &params, const Mat &widened_detect);
}  // namespace hybrid_nn

// ---- fused plan (reference fused_inference.hpp:13-60) ----------------------
inline constexpr int kFusedMaxWidth = 128;
struct FusedPlan {
    std::vector<int> dims;
    std::vector<int> padded;
    std::vector<double> buffer;
    std::vector<float> buffer_f32;
    bool fused = false;
    int max_width = 0;
    HybridNetParams unpack() const;
};
namespace fused {
FusedPlan build_plan(const HybridNetParams &params);
VecF fused_forward_f32(const FusedPlan &plan, const MatF &x);
}  // namespace fused

// ---- evaluation (reference eval.hpp:27-33) ---------------------------------
// Per-element sign test / mismatch count on host-resident results; the batched
// device path fuses both into the detection epilogue (noma_detect).
BitMat hard_decision_qpsk(const CVec &symbols);
double bit_error_rate(const BitMat &predicted, const BitMat &truth);

}  // namespace noma
