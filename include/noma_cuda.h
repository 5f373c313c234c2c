/*
 * noma_cuda.h -- C-ABI of the B200-native (sm_100a) NOMA detector.
 *
 * This is the drop-in boundary for the hot path of the reference
 * "noma-detect" (arxiv 2206.05998, /root/reference/proj).  Plain pointers,
 * sizes and status codes only; no C++ or torch types cross it.  Each entry
 * point names the reference interface it replaces.  The C++ host layer
 * (paper_2206_05998_b200/host, namespace noma::) implements the reference's
 * own headers on top of these calls; INTEGRATION.md shows the bindings.
 *
 * Memory: every data call takes `mem`.  NOMA_MEM_HOST pointers are host
 * memory: the call stages them to the device, runs, copies results back and
 * synchronises.  NOMA_MEM_DEVICE pointers are device memory: the call is
 * asynchronous on the context's stream.
 *
 * Layouts (row-major, complex = interleaved re,im):
 *   WIDEN_COMPLEX design : [n_designs][rows/2][width/2] complex f64 -- the
 *                          complex receive matrix X; the widened real rows
 *                          2t = [Re x_t; Im x_t], 2t+1 = [Im x_t; -Re x_t]
 *                          (iq_transform.cpp:7-24) are formed on device.
 *   WIDEN_COMPLEX targets: [n_designs][rows/2][nets_per_design] complex f64
 *                          (TransmissionRecord::train_symbols per slot).
 *   REAL design          : [n_designs][rows][width] f64.
 *   REAL targets         : [n_designs][nets_per_design][rows] f64.
 *   params ("plan")      : [net][noma_plan_size] f32, the reference FusedPlan
 *                          buffer layout (fused_inference.cpp:19-42):
 *                          w0[pad8(d0)] | per layer l: d_l rows x pad8(d_{l-1}),
 *                          bias[pad8(d_l)] | final[pad8(d_N)].
 *   net index            : net = design * nets_per_design + user (0-based).
 */
#ifndef NOMA_CUDA_H
#define NOMA_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define NOMA_API __attribute__((visibility("default")))
#else
#define NOMA_API
#endif

/* Status codes; the C++ layer maps them onto the reference exceptions
 * (errors.hpp:8-35). */
enum noma_status {
    NOMA_OK = 0,
    NOMA_ERR_DIMENSION = 1,      /* noma::dimension_error                   */
    NOMA_ERR_CONFIG = 2,         /* noma::config_error                      */
    NOMA_ERR_ILL_CONDITIONED = 3,/* noma::ill_conditioned_error (per net)   */
    NOMA_ERR_UNSUPPORTED = 4,    /* shape outside the device kernels' range */
    NOMA_ERR_CUDA = 5,           /* CUDA runtime failure (see last_error)   */
    NOMA_ERR_ARGUMENT = 6        /* null / inconsistent argument            */
};

enum noma_mem { NOMA_MEM_HOST = 0, NOMA_MEM_DEVICE = 1 };
enum noma_layout { NOMA_LAYOUT_WIDEN_COMPLEX = 0, NOMA_LAYOUT_REAL = 1 };

#define NOMA_MAX_DIMS 9      /* input width + up to 8 hidden layers       */
#define NOMA_MAX_WIDTH 128   /* kFusedMaxWidth (fused_inference.hpp:15)   */
#define NOMA_MAX_BATCH 128   /* device minibatch tile                      */

typedef struct noma_ctx_s *noma_ctx_t;

/* [dims[0] = 2M, L_1, ..., L_N] -- HybridNetParams::dims (hybrid_nn.hpp:21) */
typedef struct {
    int ndims;
    int dims[NOMA_MAX_DIMS];
} noma_net_desc;

/* TrainConfig + AdamState hyper-parameters (hybrid_nn.hpp:31-49) */
typedef struct {
    int epochs;       /* 50    */
    int batch_size;   /* 128   */
    double lr;        /* 0.005 */
    double beta1;     /* 0.9   */
    double beta2;     /* 0.999 */
    double eps;       /* 1e-8  */
} noma_train_cfg;

/* Training / LLS data set: one design shared by nets_per_design targets
 * (WidenedDataset, iq_transform.hpp:13-17, batched over slots and users). */
typedef struct {
    int layout;            /* enum noma_layout                         */
    int n_designs;         /* slots S                                  */
    int nets_per_design;   /* users K                                  */
    int rows;              /* widened rows 2*N_T (WIDEN) or rows (REAL) */
    int width;             /* 2M (WIDEN) or columns (REAL)              */
    const double *design;
    const double *targets;
} noma_dataset;

/* ScenarioConfig (channel_sim.hpp:14-31) */
typedef struct {
    int num_users;
    int num_antennas;
    int train_symbols;
    int data_symbols;
    double power_step_db;
    double snr_db;               /* +inf: noiseless */
    double rx_nonlinearity_gain;
} noma_scenario;

/* ---------------------------------------------------------------- context */
NOMA_API int noma_version(void);
NOMA_API int noma_ctx_create(int device, noma_ctx_t *out);
NOMA_API int noma_ctx_destroy(noma_ctx_t ctx);
NOMA_API const char *noma_ctx_last_error(noma_ctx_t ctx);
/* Run subsequent calls on this cudaStream_t (NULL = the context's own). */
NOMA_API int noma_ctx_set_stream(noma_ctx_t ctx, void *cuda_stream);
NOMA_API int noma_ctx_synchronize(noma_ctx_t ctx);
/* Number of kernels this context has launched (instrumentation). */
NOMA_API long long noma_ctx_kernel_launches(noma_ctx_t ctx);
/* Which training kernel the last noma_train / noma_pipeline call launched:
 * 1 = one CTA per net (16 warps), 2 = two 8-warp CTAs per SM,
 * 10 + c = row-split cluster of c CTAs per net (DSMEM gradient reduce),
 * 100 + c = neuron-split latency cluster of c CTAs per net (k_train_lat.cu),
 * 3 = 4-warp one-hidden-layer kernel (k_train_w4.cu: inputs 32 / 64),
 * 4 = 8-warp one-hidden-layer kernel (k_train_w8.cu: 128-wide inputs, C4),
 * 5 = 8-warp two-hidden-layer kernel (k_train_l2.cu: [32 | 64, 64, 64], C2),
 * 200 = shape-general FP32 kernel (k_train_generic.cu: layers wider than 128,
 *       minibatches above 128 rows), 201 = its FP64 instance (noma_train_f64),
 * 300 = on-chip FP64 kernel (k_train_f64.cu), 301 = register-tiled FP64
 *       kernel (k_train_w8d.cu: one hidden layer of 64, inputs 32 / 64), 0 = none yet.
 * NOMA_TRAIN_GENERIC=1 in the environment forces the shape-general kernel. */
NOMA_API int noma_ctx_train_mode(noma_ctx_t ctx);
/* Which detection kernel the last noma_detect / noma_pipeline call used:
 * 1 = FP32 FFMA register tiles (k_detect.cu), 2 = tcgen05 3xTF32 tensor-core
 * kernel (k_detect_tc.cu; widened input 32/64, hidden layers of 64),
 * 3 = shape-general single-pass tiles (k_dense.cu: layers wider than 128),
 * 0 = none yet.  NOMA_DETECT_TC=0 in the environment forces the FFMA kernel. */
NOMA_API int noma_ctx_detect_mode(noma_ctx_t ctx);
/* Slot chunks the last noma_pipeline call ran in (instrumentation). */
NOMA_API int noma_ctx_pipeline_chunks(noma_ctx_t ctx);
/* Instrumentation: when on, noma_pipeline records CUDA events around its
 * phases (init and shuffles run on a side stream, overlapping the LLS);
 * noma_ctx_phase_ms waits for the last call and returns ms for
 * [lls, init, shuffle, train, detect, whole pipeline]. */
NOMA_API int noma_ctx_set_profiling(noma_ctx_t ctx, int on);
NOMA_API int noma_ctx_phase_ms(noma_ctx_t ctx, double *ms6);
/* FP32 FFMA throughput of this device (TFLOP/s) over every SM, the roofline
 * denominators of the FP32-bound training and detection kernels.
 * form 0: FFMA with constant operands (the issue-rate peak);
 * form 1: an 8x4 register outer product in scalar FFMA, all operands in
 *         registers (3-register FFMA is register-file-read limited,
 *         profiles/r01_microbench_ffma_forms.txt);
 * form 2: the same outer product in packed FFMA2 with one broadcast operand
 *         -- the instruction form the training tiles use, so the ceiling of
 *         their inner loops (profiles/r01_microbench_ffma2.txt). */
NOMA_API int noma_measure_fp32_tflops(noma_ctx_t ctx, int form, double *tflops);

/* Floats in the FusedPlan buffer for `desc` (fused_inference.cpp:19-42). */
/* Page-locked host buffers for NOMA_MEM_HOST calls: with them the per-chunk
 * uploads / downloads of noma_pipeline and noma_detect run asynchronously on
 * the copy streams (pageable memory serialises every transfer). */
NOMA_API int noma_host_alloc(size_t bytes, void **out);
NOMA_API int noma_host_free(void *p);

NOMA_API int noma_plan_size(const noma_net_desc *desc);
/* Trainable parameters (HybridNetParams::trainable_count, hybrid_nn.cpp:11-16). */
NOMA_API int noma_param_count(const noma_net_desc *desc);

/* ------------------------------------------------------------- hot path */

/* Replaces lls::fit (lls.hpp:19-21, lls.cpp:10-60), batched over every
 * (design, target) pair.  FP64 Gram accumulation + Jacobi eigensolve in
 * shared memory.  Outputs [net][width] w0, [net] gram_condition, [net] status
 * (NOMA_OK or NOMA_ERR_ILL_CONDITIONED with gram_condition set). */
NOMA_API int noma_lls_fit(noma_ctx_t ctx, const noma_dataset *ds, double *w0,
                          double *gram_condition, int *status, int mem);

/* Replaces hybrid_nn::init_params (hybrid_nn.hpp:55-56, hybrid_nn.cpp:34-55)
 * for n_nets networks: net i draws from Rng(seeds[i]) exactly as the
 * reference (He-normal rows then columns, layer by layer; biases and final
 * layer zero); w0 ([net][dims[0]], nullable) is copied into the plan. */
NOMA_API int noma_init_params(noma_ctx_t ctx, const noma_net_desc *desc, int n_nets,
                              const uint64_t *seeds, const double *w0, float *plans, int mem);

/* init_params with the caller's Rng (hybrid_nn.hpp:55: `Rng& rng` is advanced):
 * states [net][4] hold xoshiro256++ states (rng.hpp:28-45) on entry and the
 * advanced states on return.  Outputs (nullable): plans [net][plan] f32, and
 * theta [net][trainable] f64 in the reference parameter order W_1, b_1, ...,
 * W_N, b_N, final (HybridNetParams, hybrid_nn.hpp:15-23). */
NOMA_API int noma_init_params_state(noma_ctx_t ctx, const noma_net_desc *desc, int n_nets,
                                    uint64_t *states, const double *w0, float *plans,
                                    double *theta, int mem);

/* Replaces lls::predict (lls.hpp:24, lls.cpp:62-66) for every net: FP64
 * yhat = X w0.  WIDEN_COMPLEX: data [n_designs][rows][width/2] c64, out
 * [net][rows] c64 (narrow(X_widened w0)); REAL: data [n_designs][rows][width]
 * f64, out [net][rows] f64. */
NOMA_API int noma_lls_predict(noma_ctx_t ctx, int layout, int n_designs, int nets_per_design,
                              int rows, int width, const double *data, const double *w0,
                              double *out, int mem);

/* Replaces hybrid_nn::train (hybrid_nn.hpp:70-72, hybrid_nn.cpp:158-195)
 * for every net of `ds`: one fused kernel per net runs all epochs x
 * minibatches (forward, backward, Adam) with the weights resident on chip;
 * shapes outside the on-chip kernels (a layer wider than 128, batch_size
 * above 128) run the shape-general kernel (train mode 200).
 * plans_inout [net][plan] holds the initial parameters (incl. w0) and
 * receives the trained ones; shuffle_seeds [net] are TrainConfig::shuffle_seed;
 * loss_trace [net][epochs] nullable; status [net] nullable. */
NOMA_API int noma_train(noma_ctx_t ctx, const noma_dataset *ds, const noma_net_desc *desc,
                        const noma_train_cfg *cfg, const double *w0, float *plans_inout,
                        const uint64_t *shuffle_seeds, double *loss_trace, int *status, int mem);

/* FP64 parity mode of noma_train: the reference's precision end to end
 * (residual x w0 + a w - y formed in FP64, FP64 Adam).  theta_inout
 * [net][trainable] holds HybridNetParams in the reference flat order (W_1,
 * b_1, ..., W_N, b_N, final) on entry and the trained values on return. */
NOMA_API int noma_train_f64(noma_ctx_t ctx, const noma_dataset *ds, const noma_net_desc *desc,
                            const noma_train_cfg *cfg, const double *w0, double *theta_inout,
                            const uint64_t *shuffle_seeds, double *loss_trace, int *status,
                            int mem);

/* Replaces hybrid_nn::detect / fused::fused_forward_f32 + hard_decision_qpsk
 * + bit_error_rate (hybrid_nn.cpp:197-199, fused_inference.cpp:222-231,
 * eval.cpp:38-65): streaming inference of every net over its design's data.
 *   WIDEN_COMPLEX: data [n_designs][rows][width/2] complex f32 (rows = N_D
 *     symbols); soft [net][rows] complex f32; codes [net][rows] u8 with
 *     bit0 = Re<0, bit1 = Im<0; truth [n_designs][rows][nets_per_design] u8
 *     codes; bit_errors [net] u32 (mismatched bits, the numerator of
 *     bit_error_rate); symbol_errors [net] u32 (symbols whose decision
 *     differs from the truth in either bit: SER numerator).
 *   REAL: data [n_designs][rows][width] f32; soft [net][rows] f32 (no codes).
 * All outputs nullable.  An ill-conditioned net's counters read 0xFFFFFFFF. */
NOMA_API int noma_detect(noma_ctx_t ctx, const noma_net_desc *desc, int layout, int n_designs,
                         int nets_per_design, int rows, const float *data, const float *plans,
                         const uint8_t *truth, float *soft, uint8_t *codes, uint32_t *bit_errors,
                         uint32_t *symbol_errors, int mem);

/* One slot batch end to end (noma_cli.cpp:86-160 per user, eval.cpp:228-241):
 * LLS -> init (Rng(init_seeds[net])) -> train (shuffle_seeds[net]) -> detect.
 * pilots/targets as the WIDEN_COMPLEX dataset; data_rx [S][ND][M] complex f32;
 * truth [S][ND][K] codes (nullable).  Outputs nullable except status;
 * bit_errors / symbol_errors [S][K] as noma_detect.  Slots run in chunks of
 * bounded scratch (NOMA_CHUNK_MB, default 4096); with NOMA_MEM_HOST each
 * chunk's inputs are uploaded ahead on a copy stream and its results
 * downloaded while the next chunk computes.  Networks wider than 128 or
 * minibatches above 128 rows train and detect in the shape-general kernels
 * (train mode 200, detect mode 3). */
NOMA_API int noma_pipeline(noma_ctx_t ctx, const noma_net_desc *desc, const noma_train_cfg *cfg,
                           int S, int K, int M, int NT, int ND, const double *pilot_rx,
                           const double *pilot_sym, const float *data_rx, const uint8_t *truth,
                           const uint64_t *init_seeds, const uint64_t *shuffle_seeds,
                           double *w0, double *gram_condition, float *plans, double *loss_trace,
                           float *soft, uint8_t *codes, uint32_t *bit_errors,
                           uint32_t *symbol_errors, int *status, int mem);

/* ------------------------------------------------ one network, FP64 API */

/* Evaluation paths of noma_forward_* (fused_inference.cpp:172-231 dispatch). */
enum noma_path {
    NOMA_PATH_AUTO = 0,     /* single-pass when every width <= 128, else per-layer */
    NOMA_PATH_FUSED = 1,    /* single-pass row tiles, activations on chip (fused_kernel) */
    NOMA_PATH_FALLBACK = 2, /* one launch per layer, activations in HBM (fallback_kernel) */
    NOMA_PATH_NAIVE = 3     /* per layer: GEMM, bias, ReLU as separate launches */
};

/* Replaces fused::fused_forward / fused_forward_into (FP64) and
 * fused_forward_f32 (FP32), and hybrid_nn::forward (fused_inference.hpp:53-60,
 * hybrid_nn.hpp:59): out[rows] = X w0 + a_N w_{N+1} for ONE network.
 *   plan : the FusedPlan buffer (fused_inference.cpp:19-42), f64 or f32;
 *   x    : COLUMN-major [dims[0]][rows] (Eigen storage of the B x 2M input);
 *   path : enum noma_path.  Any widths (the on-chip tile height adapts).
 * The linear branch is accumulated in column order without FMA, so a zero
 * final layer returns X w0 exactly as the reference's GEMV does.  With
 * NOMA_MEM_HOST the call stages through a persistent device workspace and
 * performs no host heap allocation once warm (test_fused.cpp:133-144). */
NOMA_API int noma_forward_f64(noma_ctx_t ctx, const noma_net_desc *desc, const double *plan, int rows,
                              const double *x, double *out, int path, int mem);
NOMA_API int noma_forward_f32(noma_ctx_t ctx, const noma_net_desc *desc, const float *plan, int rows,
                              const float *x, float *out, int path, int mem);

/* Device timing behind fused::bench_compare (fused_inference.cpp:262-314):
 * median over `repeats` (<= 64) launches of one evaluation path with the
 * batch resident in HBM, CUDA events on the context stream, in ns. */
NOMA_API int noma_bench_forward_f64(noma_ctx_t ctx, const noma_net_desc *desc, const double *plan, int rows,
                                    const double *x, int path, int repeats, double *ns_median);

/* Replaces hybrid_nn::loss_and_grad (hybrid_nn.hpp:63-64, hybrid_nn.cpp:84-114)
 * in FP64 for one network: loss = ||X w0 + a_N w - y||^2 / B, grad [trainable]
 * in the reference flat order W_1 (row-major L_1 x L_0), b_1, ..., W_N, b_N,
 * final.  plan: FP64 FusedPlan buffer; x column-major [dims[0]][rows]. */
NOMA_API int noma_loss_and_grad(noma_ctx_t ctx, const noma_net_desc *desc, const double *plan, int rows,
                                const double *x, const double *y, double *loss, double *grad, int mem);

/* Replaces hybrid_nn::adam_step (hybrid_nn.hpp:67, hybrid_nn.cpp:118-144) on a
 * flat FP64 parameter vector: m, v updated in place; corr_i = 1 - beta_i^step
 * computed by the caller with std::pow as the reference does (:133-135). */
NOMA_API int noma_adam_step(noma_ctx_t ctx, int n, double *theta, const double *grad, double *m, double *v,
                            double corr1, double corr2, double lr, double beta1, double beta2, double eps,
                            int mem);

/* noma_pipeline in the reference's FP64 arithmetic (bit-consistent mode):
 * FP64 He-normal init from Rng(init_seeds[net]), FP64 training on the FP64
 * pilots (train mode 300, or 201 for shapes beyond k_train_f64's on-chip
 * layout), the trained parameters rounded to FP32 for detection.  Same
 * arguments and outputs as noma_pipeline. */
NOMA_API int noma_pipeline_f64(noma_ctx_t ctx, const noma_net_desc *desc, const noma_train_cfg *cfg,
                               int S, int K, int M, int NT, int ND, const double *pilot_rx,
                               const double *pilot_sym, const float *data_rx, const uint8_t *truth,
                               const uint64_t *init_seeds, const uint64_t *shuffle_seeds,
                               double *w0, double *gram_condition, float *plans, double *loss_trace,
                               float *soft, uint8_t *codes, uint32_t *bit_errors,
                               uint32_t *symbol_errors, int *status, int mem);

/* Replaces synthesize(cfg, SeedBundle::from_master(seed)) (channel_sim.cpp:76-117)
 * on device for S slots with master seeds [S].  Outputs (nullable):
 * pilot_rx [S][NT][M] c64, pilot_sym [S][NT][K] c64, data_rx [S][ND][M] c32,
 * data_codes [S][ND][K] u8, channel [S][M][K] c64, noise_power [S]. */
NOMA_API int noma_synthesize(noma_ctx_t ctx, const noma_scenario *sc, int S,
                             const uint64_t *master_seeds, double *pilot_rx, double *pilot_sym,
                             float *data_rx, uint8_t *data_codes, double *channel,
                             double *noise_power, int mem);
/* As noma_synthesize with explicit SeedBundles [S][3] = {symbols, channel,
 * noise} (synthesize(cfg, seeds), channel_sim.cpp:76-117) -- the per-trial
 * seeds of run_noise_sweep (eval.cpp:212-219). */
NOMA_API int noma_synthesize_bundles(noma_ctx_t ctx, const noma_scenario *sc, int S,
                                     const uint64_t *bundles, double *pilot_rx, double *pilot_sym,
                                     float *data_rx, uint8_t *data_codes, double *channel,
                                     double *noise_power, int mem);

/* As noma_synthesize_bundles with the data-phase receive matrix in FP64
 * (data_rx [S][ND][M] c64): the C++ API's TransmissionRecord is all FP64. */
NOMA_API int noma_synthesize_f64(noma_ctx_t ctx, const noma_scenario *sc, int S, const uint64_t *bundles,
                                 double *pilot_rx, double *pilot_sym, double *data_rx, uint8_t *data_codes,
                                 double *channel, double *noise_power, int mem);

#ifdef __cplusplus
}
#endif
#endif
