// Kernel parameter blocks and host-side launchers (one definition, shared by
// the kernel translation units and the C-ABI in capi.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace noma_dev {

struct LlsParams {
    int layout;           // NOMA_LAYOUT_*
    int n_designs, K, rows, width;
    int m;                // complex columns (width/2 for WIDEN, width for REAL)
    int nrow_c;           // complex rows (rows/2 for WIDEN, rows for REAL)
    const double *design, *targets;
    double *w0, *cond;
    int *status;
    float *design32;      // nullable: FP32 copy for training, [S][nrow_c][width]
    float *r0;            // nullable: [net][rows]
    long long *clocks;    // nullable: phase cycles of block 0 (NOMA_PHASE_CLOCKS)
    float *plans;         // nullable: FusedPlan buffers whose w0 slot gets (float) w0
    int plan_total;
    unsigned char *fast;  // nullable (WIDEN, mode 1): per design, 1 = Cholesky path taken and r0
                          // left to lls_r0_launch (many CTAs) instead of the one-CTA pass
    int mode;             // 0: Jacobi path; 1: Cholesky fast path (Jacobi fallback), no
                          // cond for fast-path nets; 2: condition numbers only
};

struct TrainParams {
    NetGeom g;
    int layout, n_nets, K, rows, width, epochs, batch;
    const float *design32;  // WIDEN: [S][rows/2][width] ([Re x_t | Im x_t]); REAL: [S][rows][width]
    const float *r0;        // [net][rows]
    const uint16_t *perm;   // [net][epochs][rows]
    float *plans;           // [net][plan_total] in/out
    double *trace;          // [net][epochs] nullable
    const int *status;      // [net] nullable
    float lr, b1, b2, eps, omb1, omb2;
    double lr_d, b1d, b2d;
    // shared-memory carve-up (floats)
    int off_x, off_a[NOMA_MAX_DIMS], off_ps, off_gs, off_r0b, off_dy, off_red, off_yp, off_misc,
        off_end, gs_stride, gsplit, off_mom;
    long long *clocks;      // nullable: phase cycles of block 0 (NOMA_PHASE_CLOCKS)
    int mode;               // out: kernel shape launched (noma_ctx_train_mode codes)
    float *xprep, *r0prep;  // latency kernel: per-step minibatch tiles (scratch, nullable)
    float *agbuf;           // latency kernel, 2+ layers: [net][2][H][kSR] all-gather staging (nullable)
    const float *atab;      // [total steps][2] Adam constants lr / c1, 1 / c2 (nullable)
    size_t prep_floats;     // capacity of xprep (floats)
};

struct TrainF64Params {
    NetGeom g;
    int layout, n_nets, K, rows, width, epochs, batch;
    const double *design;   // as noma_dataset (FP64)
    const double *targets;
    const double *w0;       // [net][width]
    const uint16_t *perm;   // [net][epochs][rows]
    double *theta;          // [net][ptrain] in/out, reference flat order
    double *moments;        // [net][2][ptrain] scratch
    double *trace;          // [net][epochs] nullable
    const int *status;
    double lr, b1, b2, eps;
    int ptrain, maxw, chunk, act_total;
    int mode = 0;           // out: 300 = k_train_f64, 301 = register-tiled k_train_w8d
};

struct DetectParams {
    NetGeom g;
    int layout, n_nets, K, rows, width;
    const float *data;      // WIDEN: [S][rows][width/2] c32; REAL: [S][rows][width]
    const float *plans;     // [net][plan_total]
    const uint8_t *truth;   // WIDEN: [S][rows][K] codes, nullable
    float *soft;            // WIDEN: [net][rows] c32; REAL: [net][rows]
    uint8_t *codes;         // WIDEN: [net][rows]
    uint32_t *errors;       // [net] bit errors (nullable)
    uint32_t *sym_errors;   // [net] symbol errors: decision != truth (nullable)
    const int *status;      // [net] nullable
    int tiles;              // per net
    int stride = 0;         // row stride of data / truth / soft / codes (0: rows); a
                            // launch over rows [r0, r0 + rows) passes offset pointers
    int off_x, off_a0, off_a1, off_ps, off_w0, off_y, off_yp, off_end;
    int mode;               // out: 1 = FFMA kernel, 2 = tcgen05 3xTF32 kernel
};

struct SynthParams {
    int S, K, M, NT, ND;
    double gain;           // cubic distortion
    int noisy;             // snr finite
    double snr_lin;        // 10^(snr/10), computed on the host (glibc pow)
    const uint64_t *seeds; // master seeds [S], or [S][3] {symbols, channel, noise} if bundles
    int bundles;           // 1: seeds are explicit SeedBundles (eval.cpp:212-219 sweep seeds)
    const double *powers;  // [K], host-computed power_profile
    double *pilot_rx;      // [S][NT][M] c64
    double *pilot_sym;     // [S][NT][K] c64
    float *data_rx;        // [S][ND][M] c32
    double *data_rx64;     // [S][ND][M] c64 (nullable; the C++ API's FP64 record)
    uint8_t *data_codes;   // [S][ND][K]
    double *channel;       // [S][M][K] c64 (scratch or output)
    double *noise_power;   // [S]
    uint8_t *codes_all;    // scratch [S][NT+ND][K]
    double *noise;         // scratch [S][NT+ND][M] c64 (unit gaussians, g++ draw order)
};

// Shape-general forward (k_dense.cu): input source of fwd_tile_kernel
constexpr int kSrcColMajor = 0;  // x[c * ldx + R] (Eigen column-major, one design)
constexpr int kSrcRowMajor = 1;  // REAL rows [S][stride][width]
constexpr int kSrcComplex = 2;   // complex rows [S][stride][width/2], widened at load

template <class T>
struct FwdParams {
    NetGeom g;
    int src, n_nets, K;
    int rows;                 // input rows of this launch (widened rows for kSrcComplex)
    int stride;               // row stride per design (symbols for kSrcComplex)
    const T *x;
    long long ldx;            // kSrcColMajor leading dimension
    const T *plan;            // [net][plan_total]
    T *out;                   // out[net * out_stride + R] (nullable)
    long long out_stride;
    uint8_t *codes;           // kSrcComplex: [net][code_stride] QPSK codes (nullable)
    long long code_stride;
    const uint8_t *truth;     // kSrcComplex: [S][stride][K] (nullable)
    uint32_t *errors, *sym_errors;  // [net] (nullable)
    const int *status;        // [net] (nullable)
    int TR, maxh;             // set by the launcher
};

// Shape-general training (k_train_generic.cu): parameters trained in place in
// the FusedPlan layout; scratch [net][scratch_per_net] (train_generic_scratch)
template <class T>
struct TrainGenParams {
    NetGeom g;
    int layout, n_nets, K, rows, epochs, batch;
    const float *design32;    // T = float: as TrainParams::design32
    const float *r0;          // T = float: [net][rows]
    const double *design;     // T = double: as noma_dataset
    const double *targets;
    const double *w0;         // T = double: [net][dims[0]]
    const uint16_t *perm;     // [net][epochs][rows]
    T *plan;                  // [net][plan_total] in/out
    double *trace;            // [net][epochs] nullable
    const int *status;
    T *scratch;
    size_t scratch_per_net;
    double lr, b1, b2, eps;
};

int lls_launch(const LlsParams &p, cudaStream_t st);
int perm_launch(int n_nets, int epochs, int n, const uint64_t *seeds, uint16_t *perm,
                cudaStream_t st, int max_tpb = 64);
int init_launch(const NetGeom &g, int n_nets, const uint64_t *seeds, const double *w0, bool keep_w0,
                float *plans, cudaStream_t st);
int set_w0_launch(int n_nets, int d0, int plan_total, const double *w0, float *plans,
                  cudaStream_t st);
int init_state_launch(const NetGeom &g, int n_nets, uint64_t *states, const double *w0,
                      float *plans, double *theta, int ptrain, cudaStream_t st);
int lls_predict_launch(int layout, int S, int K, int rows, int width, const double *data,
                       const double *w0, double *out, cudaStream_t st);
int train_launch(TrainParams &p, cudaStream_t st);
int train_lat_launch(TrainParams &p, cudaStream_t st);
bool train_w4_fits(const TrainParams &p);
int train_w4_launch(TrainParams &p, cudaStream_t st);
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link); no swizzle / interleave, zero fill out of bounds.  false on failure.
bool tensor_map_encode_tiled(CUtensorMap *tm, CUtensorMapDataType dt, int rank, void *base, const cuuint64_t *gdim,
                             const cuuint64_t *gstride, const cuuint32_t *box, const cuuint32_t *estride);
bool train_w8_fits(const TrainParams &p);
int train_w8_launch(TrainParams &p, cudaStream_t st);
int adam_table_launch(double lr, double b1, double b2, int total, float *t, cudaStream_t st);
int lls_r0_launch(const LlsParams &p, cudaStream_t st);
bool train_l2_fits(const TrainParams &p);
int train_l2_launch(TrainParams &p, cudaStream_t st);
// widened FP32 design rows (2t = [Re|Im], 2t+1 = [Im|-Re]) for the cp.async gathers
int widen_rows_launch(const float *d32, float *wide, size_t nrow_c, int width, cudaStream_t st);
int train_f64_launch(TrainF64Params &p, cudaStream_t st);
bool train_w8d_fits(const TrainF64Params &p);
int train_w8d_launch(TrainF64Params &p, cudaStream_t st);
int detect_launch(DetectParams &p, cudaStream_t st);
int detect_tc_launch(const DetectParams &p, cudaStream_t st);
int synth_launch(SynthParams p, double *noise_power_scratch, cudaStream_t st);

template <class T>
int fwd_tile_launch(FwdParams<T> &p, cudaStream_t st);
template <class T>
int layer_forward_launch(const NetGeom &g, const T *plan, const T *X, long long ld, int rows, T *acts, bool naive,
                         const T *y, T *out, T *dy, cudaStream_t st);
size_t loss_grad_scratch(const NetGeom &g, int rows);
int loss_grad_launch(const NetGeom &g, const double *plan, const double *X, int rows, const double *y, double *ws,
                     double *loss, double *grad, cudaStream_t st);
int adam_launch(int n, double *theta, const double *grad, double *m, double *v, double c1, double c2, double lr,
                double b1, double b2, double eps, cudaStream_t st);
size_t train_generic_scratch(const NetGeom &g, int batch);
int theta_plan_launch(const NetGeom &g, int n_nets, double *theta, double *plan, const double *w0, int to_plan,
                      cudaStream_t st);
int theta_plan32_launch(const NetGeom &g, int n_nets, const double *theta, float *plan, const double *w0,
                        cudaStream_t st);
int init_theta_launch(const NetGeom &g, int n_nets, const uint64_t *seeds, double *theta, int ptrain,
                      cudaStream_t st);
template <class T>
int train_generic_launch(TrainGenParams<T> &p, cudaStream_t st);

}  // namespace noma_dev
