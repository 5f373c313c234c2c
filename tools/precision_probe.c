/* Diagnostics (not product, not a test): which FP32 stage of the device
 * training makes a 50-epoch training drift from the FP64 reference?
 *
 * Trains every user net of one slot (oracle synthesis, LLS, init, shuffles)
 * with one hidden layer, once in FP64 (the reference algorithm,
 * hybrid_nn.cpp:84-195) and once per precision variant, and prints the
 * decision flips and soft-output deviation of each variant against FP64.
 * Stages (bit flags): 1 forward in FP32, 2 gradients in FP32, 4 Adam state
 * and parameters in FP32, 8 residual through r0 = fl32(y - x w0) (the device
 * scheme), 16 FP64 with the minibatch rows summed in reverse order (a
 * reordering the reference's own Eigen build could make: rounding-level FP64
 * perturbation).  15 emulates the device kernels (up to summation order).
 *
 *   gcc -O2 -ffp-contract=off -I oracle tools/precision_probe.c oracle/orc_*.c -lm -lpthread
 *   ./a.out M K step_db seed variant...
 */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "noma_oracle.h"

typedef struct {
    int in, H, n, epochs, batch;
    const double *x, *y, *w0;
    uint64_t shuffle_seed;
    int flags;
} job;

static double r32(double v, int on) { return on ? (double)(float)v : v; }

/* theta layout (hybrid_nn.cpp flat order): W [H][in], b [H], final [H] */
static void train_mixed(const job *j, double *theta) {
    const int in = j->in, H = j->H, n = j->n, P = H * in + 2 * H;
    const int F = j->flags & 1, G = j->flags & 2, A = j->flags & 4, R = j->flags & 8;
    double *m = calloc(P, sizeof(double)), *v = calloc(P, sizeof(double)), *g = malloc(sizeof(double) * P);
    double *a = malloc(sizeof(double) * 128 * H), *dy = malloc(sizeof(double) * 128);
    double *r0 = malloc(sizeof(double) * n);
    int *idx = malloc(sizeof(int) * n);
    for (int r = 0; r < n; ++r) {
        double lin = 0.0;
        for (int c = 0; c < in; ++c) lin += j->x[(size_t)r * in + c] * j->w0[c];
        r0[r] = j->y[r] - lin;
    }
    if (A)
        for (int i = 0; i < P; ++i) theta[i] = (float)theta[i];
    long step = 0;
    for (int e = 0; e < j->epochs; ++e) {
        orc_shuffled_indices(n, j->shuffle_seed, e, idx);
        for (int start = 0; start < n; start += j->batch) {
            const int b = j->batch < n - start ? j->batch : n - start;
            const double *W = theta, *bb = theta + H * in, *wf = theta + H * in + H;
            for (int i = 0; i < b; ++i) {
                const int row = idx[start + i];
                const double *xr = j->x + (size_t)row * in;
                double br = 0.0;
                for (int h = 0; h < H; ++h) {
                    double z = r32(bb[h], F);
                    for (int c = 0; c < in; ++c) z = r32(z + r32(r32(W[h * in + c], F) * r32(xr[c], F), F), F);
                    a[i * H + h] = z > 0.0 ? z : 0.0;
                    br = r32(br + r32(a[i * H + h] * r32(wf[h], F), F), F);
                }
                double res;
                if (R) {
                    res = (double)((float)br - (float)r0[row]);
                } else {
                    double lin = 0.0;
                    for (int c = 0; c < in; ++c) lin += xr[c] * j->w0[c];
                    res = lin + br - j->y[row];
                }
                dy[i] = r32((2.0 / b) * res, G);
            }
            memset(g, 0, sizeof(double) * P);
            double *gW = g, *gb = g + H * in, *gf = g + H * in + H;
            for (int ii = 0; ii < b; ++ii) {
                const int i = (j->flags & 16) ? b - 1 - ii : ii;
                const int row = idx[start + i];
                const double *xr = j->x + (size_t)row * in;
                for (int h = 0; h < H; ++h) {
                    const double ah = a[i * H + h];
                    gf[h] = r32(gf[h] + r32(ah * dy[i], G), G);
                    const double dz = ah > 0.0 ? r32(dy[i] * r32(wf[h], G), G) : 0.0;
                    gb[h] = r32(gb[h] + dz, G);
                    for (int c = 0; c < in; ++c) gW[h * in + c] = r32(gW[h * in + c] + r32(dz * r32(xr[c], G), G), G);
                }
            }
            ++step;
            const double c1 = 1.0 - pow(0.9, (double)step), c2 = 1.0 - pow(0.999, (double)step);
            for (int i = 0; i < P; ++i) {
                m[i] = r32(r32(0.9 * m[i], A) + r32(0.1 * g[i], A), A);
                v[i] = r32(r32(0.999 * v[i], A) + r32(r32(0.001 * g[i], A) * g[i], A), A);
                const double upd = 0.005 * (m[i] / c1) / (sqrt(v[i] / c2) + 1e-8);
                theta[i] = r32(theta[i] - r32(upd, A), A);
            }
        }
    }
    free(m); free(v); free(g); free(a); free(dy); free(r0); free(idx);
}

int main(int argc, char **argv) {
    if (argc < 6) {
        fprintf(stderr, "usage: %s M K step_db seed variant...\n", argv[0]);
        return 1;
    }
    const int M = atoi(argv[1]), K = atoi(argv[2]);
    const double step_db = atof(argv[3]);
    const uint64_t seed = strtoull(argv[4], NULL, 10);
    const int NT = 685, ND = 3840, H = 64, in = 2 * M;
    orc_scenario sc = {K, M, NT, ND, step_db, 25.0, 0.05};
    uint64_t sb[3];
    orc_seed_bundle(seed, sb);
    double *chan = malloc(sizeof(double) * 2 * M * K), *pw = malloc(sizeof(double) * K), np;
    double *trx = malloc(sizeof(double) * 2 * NT * M), *tsym = malloc(sizeof(double) * 2 * NT * K);
    double *drx = malloc(sizeof(double) * 2 * ND * M), *dsym = malloc(sizeof(double) * 2 * ND * K);
    orc_synthesize(&sc, sb[0], sb[1], sb[2], chan, pw, trx, tsym, drx, dsym, &np);
    double *xt = malloc(sizeof(double) * 2 * NT * in), *xd = malloc(sizeof(double) * 2 * ND * in);
    orc_widen_design(NT, M, trx, xt);
    orc_widen_design(ND, M, drx, xd);
    const int dims[2] = {in, H};
    const int P = H * in + 2 * H;
    double *yt = malloc(sizeof(double) * 2 * NT), *w0 = malloc(sizeof(double) * in);
    double *th0 = malloc(sizeof(double) * P), *th = malloc(sizeof(double) * P), *thr = malloc(sizeof(double) * P);
    double *pr = malloc(sizeof(double) * 2 * ND), *pv = malloc(sizeof(double) * 2 * ND);
    const int nv = argc - 5;
    long flips[16] = {0};
    double sdev[16] = {0};
    for (int k = 0; k < K; ++k) {
        orc_widen_targets(NT, tsym + 2 * k, K, yt);
        double cond;
        if (orc_lls_fit(2 * NT, in, xt, yt, w0, &cond)) continue;
        orc_rng ir;
        orc_rng_seed(&ir, orc_substream_seed(seed, 0x1000u + (unsigned)(k + 1)));
        orc_init_params(2, dims, &ir, th0);
        job jb = {in, H, 2 * NT, 50, 128, xt, yt, w0, orc_substream_seed(seed, (unsigned)(k + 1)), 0};
        memcpy(thr, th0, sizeof(double) * P);
        train_mixed(&jb, thr);
        orc_forward(2, dims, w0, thr, 2 * ND, xd, pr);
        double scale = 1.0;
        for (int i = 0; i < 2 * ND; ++i) scale = fabs(pr[i]) > scale ? fabs(pr[i]) : scale;
        for (int vi = 0; vi < nv; ++vi) {
            jb.flags = atoi(argv[5 + vi]);
            memcpy(th, th0, sizeof(double) * P);
            train_mixed(&jb, th);
            orc_forward(2, dims, w0, th, 2 * ND, xd, pv);
            long f = 0;
            double dev = 0.0;
            for (int t = 0; t < ND; ++t) {
                const int a = (pr[2 * t] < 0) | ((pr[2 * t + 1] < 0) << 1);
                const int b = (pv[2 * t] < 0) | ((pv[2 * t + 1] < 0) << 1);
                f += a != b;
            }
            for (int i = 0; i < 2 * ND; ++i) dev = fabs(pv[i] - pr[i]) > dev ? fabs(pv[i] - pr[i]) : dev;
            flips[vi] += f;
            sdev[vi] = dev / scale > sdev[vi] ? dev / scale : sdev[vi];
            printf("user %2d variant %2d flips %5ld soft_dev %.3g\n", k + 1, jb.flags, f, dev / scale);
            fflush(stdout);
        }
    }
    for (int vi = 0; vi < nv; ++vi)
        printf("TOTAL variant %s flips %ld of %d soft_dev_max %.3g\n", argv[5 + vi], flips[vi], K * ND, sdev[vi]);
    return 0;
}
