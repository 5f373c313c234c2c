/*
 * noma_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * FP64 CPU restatement of the reference detector path (arxiv 2206.05998,
 * "noma-detect", /root/reference/proj).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library,
 * and only as the checker or the timed CPU baseline -- never as the product.
 *
 * The reference itself cannot be built here: it needs Eigen 3.4 and
 * vendor/ single headers that are absent from the image (CMakeLists.txt:10-13).
 * Every function below cites the reference file:line whose behaviour it
 * restates.  Parity of this restatement is pinned by the reference's own
 * known-answer tests and independent oracles, ported in tests/test_oracle_*.py.
 *
 * Conventions: real matrices are row-major double[rows][cols]; complex
 * matrices are row-major interleaved double[rows][cols][2] (re, im).
 */
#ifndef NOMA_ORACLE_H
#define NOMA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, shared with the product C-ABI (include/noma_cuda.h) */
enum {
    ORC_OK = 0,
    ORC_ERR_DIMENSION = 1,   /* noma::dimension_error  (errors.hpp:8)  */
    ORC_ERR_CONFIG = 2,      /* noma::config_error     (errors.hpp:12) */
    ORC_ERR_ILL = 3          /* noma::ill_conditioned_error (errors.hpp:17) */
};

#define ORC_MAX_DIMS 9 /* input width + up to 8 hidden layers */

/* ---------------- rng.hpp:10-67 ---------------- */
typedef struct { uint64_t s[4]; } orc_rng;

uint64_t orc_splitmix64(uint64_t *state);
uint64_t orc_substream_seed(uint64_t master, uint64_t tag);
uint64_t orc_mix_tag(uint64_t a, uint64_t b, uint64_t c, uint64_t d); /* eval.cpp:77-84 */
void     orc_rng_seed(orc_rng *r, uint64_t seed);
uint64_t orc_rng_next(orc_rng *r);
double   orc_rng_uniform(orc_rng *r);
uint64_t orc_rng_below(orc_rng *r, uint64_t bound);
double   orc_rng_gaussian(orc_rng *r);
/* bulk helpers for tests: n draws of each kind */
void orc_rng_fill_u64(uint64_t seed, int n, uint64_t *out);
void orc_rng_fill_gaussian(uint64_t seed, int n, double *out);

/* ---------------- channel_sim.hpp / channel_sim.cpp ---------------- */
typedef struct {
    int num_users;
    int num_antennas;
    int train_symbols;
    int data_symbols;
    double power_step_db;
    double snr_db;               /* +inf disables noise */
    double rx_nonlinearity_gain; /* cubic distortion gain, 0 disables */
} orc_scenario;

int  orc_scenario_validate(const orc_scenario *sc);             /* channel_sim.cpp:9-21 */
void orc_power_profile(int num_users, double step_db, double *p); /* :23-28 */
int  orc_gen_symbols(int num_users, int num_symbols, orc_rng *r, double *out); /* :30-47, N x K */
int  orc_gen_channel(int num_users, int num_antennas, orc_rng *r, double *h);  /* :49-58, M x K */
/* channel_sim.cpp:80-117.  Outputs are caller-allocated:
 *   channel M*K*2, powers K, train_rx NT*M*2, train_sym NT*K*2,
 *   data_rx ND*M*2, data_sym ND*K*2; *noise_power scalar. */
int orc_synthesize(const orc_scenario *sc, uint64_t sym_seed, uint64_t chan_seed,
                   uint64_t noise_seed, double *channel, double *powers, double *train_rx,
                   double *train_sym, double *data_rx, double *data_sym, double *noise_power);
/* SeedBundle::from_master (channel_sim.hpp:38-41) */
void orc_seed_bundle(uint64_t master, uint64_t out3[3]);

/* ---------------- iq_transform.cpp:7-54 ---------------- */
int orc_widen_design(int n, int m, const double *x, double *out);            /* out 2n x 2m */
/* y: complex vector with element stride `stride` (in complex elements) */
void orc_widen_targets(int n, const double *y, int stride, double *out);     /* out 2n */
int orc_narrow_predictions(int n2, const double *yhat, double *out);          /* out n2/2 complex */

/* ---------------- lls.cpp:10-66 ---------------- */
/* Minimises ||X w - y||: JacobiSVD rank/condition test, column-pivoted
 * Householder QR solve when full rank, SVD minimum-norm solution for a
 * consistent rank-deficient system, ILL error otherwise. */
int orc_lls_fit(int rows, int cols, const double *x, const double *y, double *w,
                double *gram_condition);
/* singular values (descending) of x, rows >= cols; for tests */
int orc_singular_values(int rows, int cols, const double *x, double *sv);

/* ---------------- hybrid_nn.cpp ---------------- */
/* Flat trainable-parameter order (also the Adam/gradient order):
 *   W_1 (L1 x L0 row-major), b_1, W_2, b_2, ..., W_N, b_N, final (L_N). */
int  orc_param_count(int ndims, const int *dims);
int  orc_init_params(int ndims, const int *dims, orc_rng *r, double *theta); /* :34-55 */
int  orc_forward(int ndims, const int *dims, const double *w0, const double *theta, int b,
                 const double *x, double *out);                            /* :60-82 */
int  orc_loss_and_grad(int ndims, const int *dims, const double *w0, const double *theta,
                       int b, const double *x, const double *y, double *loss,
                       double *grad);                                      /* :84-114 */
/* :118-144; *step is incremented before the bias corrections */
void orc_adam_step(int p, double *theta, const double *grad, double *m, double *v,
                   long *step, double lr, double beta1, double beta2, double eps);
/* :148-195; trace has `epochs` entries */
int  orc_train(int ndims, const int *dims, const double *w0, double *theta, int n,
               const double *x, const double *y, int epochs, int batch, double lr,
               uint64_t shuffle_seed, double *trace);
/* :148-154, Fisher-Yates with rng seeded substream_seed(seed, epoch) */
void orc_shuffled_indices(int n, uint64_t shuffle_seed, int epoch, int *idx);

/* ---------------- fused_inference.cpp ---------------- */
int  orc_plan_size(int ndims, const int *dims);                       /* :19-42 */
void orc_build_plan(int ndims, const int *dims, const double *w0, const double *theta,
                    double *buf);                                    /* :174-203 */
void orc_unpack_plan(int ndims, const int *dims, const double *buf, double *w0,
                     double *theta);                                 /* :155-170 */
void orc_fused_forward_f64(int ndims, const int *dims, const double *buf, int b,
                           const double *x, double *out);            /* :62-127 */
void orc_fused_forward_f32(int ndims, const int *dims, const float *buf, int b,
                           const float *x, float *out);              /* :222-231 */
/* naive_forward + time_median_ns semantics (fused_inference.cpp:236-278):
 * returns median ns per sample over `repeats` runs of fused_forward_f64. */
double orc_bench_fused_ns(int ndims, const int *dims, const double *buf, int b,
                          const double *x, int repeats, double *out);

/* ---------------- eval.cpp:38-65 ---------------- */
void   orc_hard_decision_qpsk(int n, const double *sym, int stride, uint8_t *bits); /* N x 2 */
long   orc_bit_errors(int n2, const uint8_t *a, const uint8_t *b);

/* ---------------- slot pipeline ----------------
 * One slot end to end as the reference's callers compose it
 * (noma_cli.cpp:86-160, eval.cpp:100-166): synthesize with
 * SeedBundle::from_master(seed), then for every user u = 1..K:
 *   widen_dataset(train_rx, train_symbols.col(u-1)) -> lls::fit
 *   init_params(dims, w0, Rng(substream_seed(seed, 0x1000+u)))   (noma_cli.cpp:97)
 *   train(..., shuffle_seed = substream_seed(seed, u))             (noma_cli.cpp:103)
 *   detect(widen_design(data_rx)) -> hard_decision_qpsk -> bit errors vs truth.
 * Outputs (each nullable): w0 K*2M, gram_cond K, status K, plan K*plan_size,
 * trace K*epochs, soft K*ND*2 (complex), bit_errors K. */
typedef struct {
    orc_scenario sc;
    int ndims;
    int dims[ORC_MAX_DIMS]; /* dims[0] == 2M */
    int epochs;
    int batch;
    double lr;
} orc_slot_cfg;

int orc_slot_run(const orc_slot_cfg *cfg, uint64_t seed, double *w0, double *gram_cond,
                 int *status, double *plan, double *trace, double *soft, long *bit_errors);
/* S slots with seeds[s], spread over `threads` pthreads; outputs are the
 * per-slot outputs above concatenated over slots (each nullable). */
int orc_slots_run_threaded(const orc_slot_cfg *cfg, int S, const uint64_t *seeds,
                           int threads, double *w0, double *gram_cond, int *status,
                           double *plan, double *trace, double *soft, long *bit_errors);

#ifdef __cplusplus
}
#endif
#endif
