/*
 * TEST INFRASTRUCTURE ONLY -- FP64 CPU restatement (see noma_oracle.h).
 *
 * hybrid_nn (hybrid_nn.cpp:11-199) and the fused inference plan
 * (fused_inference.cpp:15-231).  Dense products are plain loops summing over
 * the contraction index in increasing order (the reference delegates them to
 * Eigen; only FP64 rounding differs).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "noma_oracle.h"

int orc_param_count(int nd, const int *d) { /* hybrid_nn.cpp:11-16 */
    int n = d[nd - 1];
    for (int l = 1; l < nd; ++l) n += d[l] * d[l - 1] + d[l];
    return n;
}

static int check_dims(int nd, const int *d) {
    if (nd < 1 || nd > ORC_MAX_DIMS) return ORC_ERR_DIMENSION;
    for (int l = 0; l < nd; ++l)
        if (d[l] < 1) return ORC_ERR_DIMENSION;
    return ORC_OK;
}

int orc_init_params(int nd, const int *d, orc_rng *r, double *theta) { /* :34-55 */
    int st = check_dims(nd, d);
    if (st) return st;
    size_t off = 0;
    for (int l = 1; l < nd; ++l) {
        const int fan_in = d[l - 1];
        const double scale = sqrt(2.0 / fan_in);
        for (int row = 0; row < d[l]; ++row)
            for (int c = 0; c < fan_in; ++c) theta[off++] = orc_rng_gaussian(r) * scale;
        for (int j = 0; j < d[l]; ++j) theta[off++] = 0.0;
    }
    for (int j = 0; j < d[nd - 1]; ++j) theta[off++] = 0.0;
    return ORC_OK;
}

/* per-layer offsets into the flat theta */
static void offsets(int nd, const int *d, size_t *w_off, size_t *b_off, size_t *f_off) {
    size_t off = 0;
    for (int l = 1; l < nd; ++l) {
        w_off[l] = off;
        off += (size_t)d[l] * d[l - 1];
        b_off[l] = off;
        off += d[l];
    }
    *f_off = off;
}

/* acts[l] (b x d[l]) for l = 1..nd-1; acts[0] = x.  hybrid_nn.cpp:60-72 */
static void forward_hidden(int nd, const int *d, const double *theta, int b, const double *x,
                           double **acts) {
    size_t wo[ORC_MAX_DIMS], bo[ORC_MAX_DIMS], fo;
    offsets(nd, d, wo, bo, &fo);
    const double *prev = x;
    for (int l = 1; l < nd; ++l) {
        const int in = d[l - 1], out = d[l];
        const double *W = theta + wo[l], *bias = theta + bo[l];
        double *wt = (double *)malloc(sizeof(double) * (size_t)in * out); /* W^T, in x out */
        for (int j = 0; j < out; ++j)
            for (int c = 0; c < in; ++c) wt[(size_t)c * out + j] = W[(size_t)j * in + c];
        double *a = acts[l];
        for (int r = 0; r < b; ++r) {
            double *ar = a + (size_t)r * out;
            const double *pr = prev + (size_t)r * in;
            for (int j = 0; j < out; ++j) ar[j] = 0.0;
            for (int c = 0; c < in; ++c) {
                const double xv = pr[c];
                const double *wc = wt + (size_t)c * out;
                for (int j = 0; j < out; ++j) ar[j] += xv * wc[j];
            }
            for (int j = 0; j < out; ++j) {
                const double z = ar[j] + bias[j];
                ar[j] = z > 0.0 ? z : 0.0; /* cwiseMax(0) */
            }
        }
        free(wt);
        prev = a;
    }
}

static double **alloc_acts(int nd, const int *d, int b, const double *x) {
    double **acts = (double **)calloc(nd, sizeof(double *));
    acts[0] = (double *)x;
    for (int l = 1; l < nd; ++l) acts[l] = (double *)malloc(sizeof(double) * (size_t)b * d[l]);
    return acts;
}

static void free_acts(int nd, double **acts) {
    for (int l = 1; l < nd; ++l) free(acts[l]);
    free(acts);
}

int orc_forward(int nd, const int *d, const double *w0, const double *theta, int b,
                const double *x, double *out) { /* :76-82 */
    int st = check_dims(nd, d);
    if (st) return st;
    size_t wo[ORC_MAX_DIMS], bo[ORC_MAX_DIMS], fo;
    offsets(nd, d, wo, bo, &fo);
    double **acts = alloc_acts(nd, d, b, x);
    forward_hidden(nd, d, theta, b, x, acts);
    const double *last = acts[nd - 1];
    const int L = d[nd - 1], in = d[0];
    const double *wf = theta + fo;
    for (int r = 0; r < b; ++r) {
        double lin = 0.0, br = 0.0;
        for (int c = 0; c < in; ++c) lin += x[(size_t)r * in + c] * w0[c];
        for (int c = 0; c < L; ++c) br += last[(size_t)r * L + c] * wf[c];
        out[r] = lin + br;
    }
    free_acts(nd, acts);
    return ORC_OK;
}

int orc_loss_and_grad(int nd, const int *d, const double *w0, const double *theta, int b,
                      const double *x, const double *y, double *loss, double *grad) { /* :84-114 */
    if (b == 0) return ORC_ERR_DIMENSION;
    int st = check_dims(nd, d);
    if (st) return st;
    size_t wo[ORC_MAX_DIMS], bo[ORC_MAX_DIMS], fo;
    offsets(nd, d, wo, bo, &fo);
    double **acts = alloc_acts(nd, d, b, x);
    forward_hidden(nd, d, theta, b, x, acts);
    const double *last = acts[nd - 1];
    const int L = d[nd - 1], in = d[0];
    const double *wf = theta + fo;
    const double batch = (double)b;

    double *dy = (double *)malloc(sizeof(double) * b);
    double sq = 0.0;
    for (int r = 0; r < b; ++r) {
        double lin = 0.0, br = 0.0;
        for (int c = 0; c < in; ++c) lin += x[(size_t)r * in + c] * w0[c];
        for (int c = 0; c < L; ++c) br += last[(size_t)r * L + c] * wf[c];
        const double res = lin + br - y[r];  /* :94 */
        sq += res * res;
        dy[r] = (2.0 / batch) * res;         /* :98 */
    }
    *loss = sq / batch;                      /* :95 */

    double *gf = grad + fo;                  /* :99 g_final = last^T dy */
    for (int j = 0; j < L; ++j) gf[j] = 0.0;
    for (int r = 0; r < b; ++r)
        for (int j = 0; j < L; ++j) gf[j] += last[(size_t)r * L + j] * dy[r];

    /* da = dy * wf^T (b x L), :102 */
    int maxw = 0;
    for (int l = 0; l < nd; ++l) maxw = d[l] > maxw ? d[l] : maxw;
    double *da = (double *)malloc(sizeof(double) * (size_t)b * maxw);
    double *dz = (double *)malloc(sizeof(double) * (size_t)b * maxw);
    for (int r = 0; r < b; ++r)
        for (int j = 0; j < L; ++j) da[(size_t)r * L + j] = dy[r] * wf[j];

    for (int l = nd - 1; l >= 1; --l) { /* :105-112 */
        const int out = d[l], inw = d[l - 1];
        const double *a = acts[l], *below = acts[l - 1];
        for (size_t i = 0; i < (size_t)b * out; ++i) dz[i] = a[i] > 0.0 ? da[i] : 0.0;
        double *gW = grad + wo[l], *gb = grad + bo[l];
        memset(gW, 0, sizeof(double) * (size_t)out * inw);
        memset(gb, 0, sizeof(double) * out);
        for (int r = 0; r < b; ++r) {
            const double *dzr = dz + (size_t)r * out, *br = below + (size_t)r * inw;
            for (int j = 0; j < out; ++j) {
                const double g = dzr[j];
                double *gwj = gW + (size_t)j * inw;
                for (int c = 0; c < inw; ++c) gwj[c] += g * br[c];
                gb[j] += g;
            }
        }
        if (l > 1) { /* da = dz * W_l */
            const double *W = theta + wo[l];
            for (int r = 0; r < b; ++r) {
                double *dar = da + (size_t)r * inw;
                const double *dzr = dz + (size_t)r * out;
                for (int c = 0; c < inw; ++c) dar[c] = 0.0;
                for (int j = 0; j < out; ++j) {
                    const double g = dzr[j];
                    const double *wj = W + (size_t)j * inw;
                    for (int c = 0; c < inw; ++c) dar[c] += g * wj[c];
                }
            }
        }
    }
    free(da); free(dz); free(dy);
    free_acts(nd, acts);
    return ORC_OK;
}

void orc_adam_step(int p, double *theta, const double *g, double *m, double *v, long *step,
                   double lr, double beta1, double beta2, double eps) { /* :118-144 */
    ++*step;
    const double corr1 = 1.0 - pow(beta1, (double)*step);
    const double corr2 = 1.0 - pow(beta2, (double)*step);
    for (int i = 0; i < p; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * (g[i] * g[i]);
        theta[i] -= lr * (m[i] / corr1) / (sqrt(v[i] / corr2) + eps);
    }
}

void orc_shuffled_indices(int n, uint64_t shuffle_seed, int epoch, int *idx) { /* :148-154 */
    orc_rng r;
    orc_rng_seed(&r, orc_substream_seed(shuffle_seed, (uint64_t)epoch));
    for (int i = 0; i < n; ++i) idx[i] = i;
    for (int i = n - 1; i > 0; --i) {
        const int j = (int)orc_rng_below(&r, (uint64_t)i + 1);
        const int t = idx[i]; idx[i] = idx[j]; idx[j] = t;
    }
}

int orc_train(int nd, const int *d, const double *w0, double *theta, int n, const double *x,
              const double *y, int epochs, int batch, double lr, uint64_t shuffle_seed,
              double *trace) { /* :158-195 */
    if (n == 0) return ORC_ERR_DIMENSION;
    if (epochs < 0 || batch < 1 || !(lr > 0.0)) return ORC_ERR_CONFIG;
    int st = check_dims(nd, d);
    if (st) return st;
    const int P = orc_param_count(nd, d), in = d[0];
    double *m = (double *)calloc(P, sizeof(double));
    double *v = (double *)calloc(P, sizeof(double));
    double *g = (double *)malloc(sizeof(double) * P);
    int *idx = (int *)malloc(sizeof(int) * n);
    const int bmax = batch < n ? batch : n;
    double *xb = (double *)malloc(sizeof(double) * (size_t)bmax * in);
    double *yb = (double *)malloc(sizeof(double) * bmax);
    long step = 0;
    for (int e = 0; e < epochs; ++e) {
        orc_shuffled_indices(n, shuffle_seed, e, idx);
        double loss_sum = 0.0;
        for (int start = 0; start < n; start += batch) {
            const int b = batch < n - start ? batch : n - start;
            for (int i = 0; i < b; ++i) {
                memcpy(xb + (size_t)i * in, x + (size_t)idx[start + i] * in, sizeof(double) * in);
                yb[i] = y[idx[start + i]];
            }
            double loss;
            orc_loss_and_grad(nd, d, w0, theta, b, xb, yb, &loss, g);
            orc_adam_step(P, theta, g, m, v, &step, lr, 0.9, 0.999, 1e-8);
            loss_sum += loss * (double)b;
        }
        if (trace) trace[e] = loss_sum / (double)n;
    }
    free(m); free(v); free(g); free(idx); free(xb); free(yb);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* FusedPlan buffer (fused_inference.cpp:19-42): w0[pad0] | per layer l:
 * d[l] rows x pad[l-1] weights, bias[pad[l]] | final[pad_N]; pad = ceil8. */

static int pad8(int w) { return ((w + 7) / 8) * 8; }

int orc_plan_size(int nd, const int *d) {
    int off = pad8(d[0]);
    for (int l = 1; l < nd; ++l) off += d[l] * pad8(d[l - 1]) + pad8(d[l]);
    return off + pad8(d[nd - 1]);
}

void orc_build_plan(int nd, const int *d, const double *w0, const double *theta, double *buf) {
    memset(buf, 0, sizeof(double) * (size_t)orc_plan_size(nd, d));
    size_t wo[ORC_MAX_DIMS], bo[ORC_MAX_DIMS], fo;
    offsets(nd, d, wo, bo, &fo);
    memcpy(buf, w0, sizeof(double) * d[0]);
    size_t off = pad8(d[0]);
    for (int l = 1; l < nd; ++l) {
        const int pin = pad8(d[l - 1]);
        for (int j = 0; j < d[l]; ++j)
            memcpy(buf + off + (size_t)j * pin, theta + wo[l] + (size_t)j * d[l - 1],
                   sizeof(double) * d[l - 1]);
        off += (size_t)d[l] * pin;
        memcpy(buf + off, theta + bo[l], sizeof(double) * d[l]);
        off += pad8(d[l]);
    }
    memcpy(buf + off, theta + fo, sizeof(double) * d[nd - 1]);
}

void orc_unpack_plan(int nd, const int *d, const double *buf, double *w0, double *theta) {
    size_t wo[ORC_MAX_DIMS], bo[ORC_MAX_DIMS], fo;
    offsets(nd, d, wo, bo, &fo);
    memcpy(w0, buf, sizeof(double) * d[0]);
    size_t off = pad8(d[0]);
    for (int l = 1; l < nd; ++l) {
        const int pin = pad8(d[l - 1]);
        for (int j = 0; j < d[l]; ++j)
            memcpy(theta + wo[l] + (size_t)j * d[l - 1], buf + off + (size_t)j * pin,
                   sizeof(double) * d[l - 1]);
        off += (size_t)d[l] * pin;
        memcpy(theta + bo[l], buf + off, sizeof(double) * d[l]);
        off += pad8(d[l]);
    }
    memcpy(theta + fo, buf + off, sizeof(double) * d[nd - 1]);
}

/* fused_kernel<T> (fused_inference.cpp:62-127): 8-row tiles, zero-padded
 * lanes, linear branch first, hidden layers through two scratch tiles. */
#define FUSED_KERNEL(NAME, T)                                                              \
    static void NAME(int nd, const int *d, const T *buf, int rows, const T *x, T *out) {   \
        enum { TILE = 8, MAXW = 128 };                                                     \
        T sa[TILE * MAXW], sb[TILE * MAXW], lin[TILE];                                     \
        const int in_w = d[0], in_pad = pad8(d[0]);                                        \
        for (int tile = 0; tile < rows; tile += TILE) {                                    \
            const int tr = rows - tile < TILE ? rows - tile : TILE;                        \
            for (int r = 0; r < tr; ++r) {                                                 \
                T *dst = sa + r * MAXW;                                                    \
                for (int c = 0; c < in_w; ++c) dst[c] = x[(size_t)(tile + r) * in_w + c]; \
                for (int c = in_w; c < in_pad; ++c) dst[c] = (T)0;                         \
            }                                                                              \
            for (int r = 0; r < tr; ++r) {                                                 \
                const T *row = sa + r * MAXW;                                              \
                T acc = (T)0;                                                              \
                for (int c = 0; c < in_pad; ++c) acc += buf[c] * row[c];                   \
                lin[r] = acc;                                                              \
            }                                                                              \
            T *cur = sa, *nxt = sb;                                                        \
            size_t off = in_pad;                                                           \
            for (int l = 1; l < nd; ++l) {                                                 \
                const int width = d[l], ppad = pad8(d[l - 1]), wpad = pad8(d[l]);          \
                const T *w = buf + off;                                                    \
                off += (size_t)width * ppad;                                               \
                const T *bb = buf + off;                                                   \
                off += wpad;                                                               \
                for (int r = 0; r < tr; ++r) {                                             \
                    const T *iv = cur + r * MAXW;                                          \
                    T *dst = nxt + r * MAXW;                                               \
                    for (int j = 0; j < width; ++j) {                                      \
                        const T *wr = w + (size_t)j * ppad;                                \
                        T acc = bb[j];                                                     \
                        for (int c = 0; c < ppad; ++c) acc += wr[c] * iv[c];               \
                        dst[j] = acc > (T)0 ? acc : (T)0;                                  \
                    }                                                                      \
                    for (int j = width; j < wpad; ++j) dst[j] = (T)0;                      \
                }                                                                          \
                T *tmp = cur; cur = nxt; nxt = tmp;                                        \
            }                                                                              \
            const T *fw = buf + off;                                                       \
            const int lpad = pad8(d[nd - 1]);                                              \
            for (int r = 0; r < tr; ++r) {                                                 \
                const T *iv = cur + r * MAXW;                                              \
                T acc = (T)0;                                                              \
                for (int c = 0; c < lpad; ++c) acc += fw[c] * iv[c];                       \
                out[tile + r] = lin[r] + acc;                                              \
            }                                                                              \
        }                                                                                  \
    }

FUSED_KERNEL(tile_kernel_f64, double)
FUSED_KERNEL(tile_kernel_f32, float)

/* fallback_kernel (fused_inference.cpp:131-151): per-layer evaluation over
 * the packed buffer for plans with a layer wider than kFusedMaxWidth. */
#define FALLBACK_KERNEL(NAME, T)                                                          \
    static void NAME(int nd, const int *d, const T *buf, int rows, const T *x, T *out) {  \
        int maxw = 0;                                                                     \
        for (int l = 0; l < nd; ++l) maxw = d[l] > maxw ? d[l] : maxw;                    \
        T *cur = (T *)malloc(sizeof(T) * maxw), *nxt = (T *)malloc(sizeof(T) * maxw);     \
        for (int r = 0; r < rows; ++r) {                                                  \
            const T *xr = x + (size_t)r * d[0];                                           \
            T lin = (T)0;                                                                 \
            for (int c = 0; c < d[0]; ++c) lin += xr[c] * buf[c];                         \
            for (int c = 0; c < d[0]; ++c) cur[c] = xr[c];                                \
            size_t off = pad8(d[0]);                                                      \
            for (int l = 1; l < nd; ++l) {                                                \
                const int pin = pad8(d[l - 1]);                                           \
                const T *w = buf + off;                                                   \
                const T *bb = buf + off + (size_t)d[l] * pin;                             \
                for (int j = 0; j < d[l]; ++j) {                                          \
                    T acc = (T)0;                                                         \
                    for (int c = 0; c < d[l - 1]; ++c) acc += cur[c] * w[(size_t)j * pin + c]; \
                    acc += bb[j];                                                         \
                    nxt[j] = acc > (T)0 ? acc : (T)0;                                     \
                }                                                                         \
                off += (size_t)d[l] * pin + pad8(d[l]);                                   \
                T *tmp = cur; cur = nxt; nxt = tmp;                                       \
            }                                                                             \
            T br = (T)0;                                                                  \
            for (int c = 0; c < d[nd - 1]; ++c) br += cur[c] * buf[off + c];              \
            out[r] = lin + br;                                                            \
        }                                                                                 \
        free(cur); free(nxt);                                                             \
    }

FALLBACK_KERNEL(fallback_kernel_f64, double)
FALLBACK_KERNEL(fallback_kernel_f32, float)

static int plan_is_fused(int nd, const int *d) { /* fused_inference.cpp:177-178 */
    for (int l = 0; l < nd; ++l)
        if (d[l] > 128) return 0;
    return 1;
}

void orc_fused_forward_f64(int nd, const int *d, const double *buf, int rows, const double *x,
                           double *out) {
    if (plan_is_fused(nd, d)) tile_kernel_f64(nd, d, buf, rows, x, out);
    else fallback_kernel_f64(nd, d, buf, rows, x, out);
}

void orc_fused_forward_f32(int nd, const int *d, const float *buf, int rows, const float *x,
                           float *out) {
    if (plan_is_fused(nd, d)) tile_kernel_f32(nd, d, buf, rows, x, out);
    else fallback_kernel_f32(nd, d, buf, rows, x, out);
}

static int cmp_double(const void *a, const void *b) {
    const double x = *(const double *)a, y = *(const double *)b;
    return x < y ? -1 : x > y;
}

double orc_bench_fused_ns(int nd, const int *d, const double *buf, int b, const double *x,
                          int repeats, double *out) { /* fused_inference.cpp:262-278 */
    double *ns = (double *)malloc(sizeof(double) * repeats);
    for (int i = 0; i < repeats; ++i) {
        struct timespec t0, t1;
        clock_gettime(CLOCK_MONOTONIC, &t0);
        orc_fused_forward_f64(nd, d, buf, b, x, out);
        clock_gettime(CLOCK_MONOTONIC, &t1);
        ns[i] = (t1.tv_sec - t0.tv_sec) * 1e9 + (t1.tv_nsec - t0.tv_nsec);
    }
    qsort(ns, repeats, sizeof(double), cmp_double);
    const double med = ns[repeats / 2];
    free(ns);
    return med / b;
}
