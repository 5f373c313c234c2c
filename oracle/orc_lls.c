/*
 * TEST INFRASTRUCTURE ONLY -- FP64 CPU restatement (see noma_oracle.h).
 *
 * lls::fit (lls.cpp:10-54).  The reference calls Eigen 3.4 (JacobiSVD for
 * rank/condition, ColPivHouseholderQR for the solve).  Eigen is absent from
 * the image, so its published algorithms are restated: a one-sided (Hestenes)
 * Jacobi SVD giving the singular values (descending) with U and V, and a
 * Householder QR with column pivoting (max remaining column norm, as LAPACK
 * xGEQP3 / Eigen ColPivHouseholderQR) followed by back substitution.
 */
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "noma_oracle.h"

/* One-sided Jacobi: B = X (column-major copy), V = I; rotate column pairs
 * until mutually orthogonal.  sigma_j = ||B_j||, U_j = B_j / sigma_j.
 * Returns columns sorted by descending sigma. */
static void jacobi_svd(int rows, int cols, const double *x, double *sv, double *u /* cols x rows, col-major per column */,
                       double *v /* cols x cols, v[j*cols + i] = V(i, j) */) {
    double *b = (double *)malloc(sizeof(double) * (size_t)rows * cols);
    double *vv = (double *)calloc((size_t)cols * cols, sizeof(double));
    for (int j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) b[(size_t)j * rows + i] = x[(size_t)i * cols + j];
        vv[(size_t)j * cols + j] = 1.0;
    }
    for (int sweep = 0; sweep < 80; ++sweep) {
        int rotated = 0;
        for (int p = 0; p + 1 < cols; ++p) {
            for (int q = p + 1; q < cols; ++q) {
                double *bp = b + (size_t)p * rows, *bq = b + (size_t)q * rows;
                double app = 0, aqq = 0, apq = 0;
                for (int i = 0; i < rows; ++i) {
                    app += bp[i] * bp[i];
                    aqq += bq[i] * bq[i];
                    apq += bp[i] * bq[i];
                }
                if (apq == 0.0 || fabs(apq) <= DBL_EPSILON * sqrt(app * aqq)) continue;
                rotated = 1;
                const double zeta = (aqq - app) / (2.0 * apq);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + t * t);
                const double sn = cs * t;
                for (int i = 0; i < rows; ++i) {
                    const double xp = bp[i], xq = bq[i];
                    bp[i] = cs * xp - sn * xq;
                    bq[i] = sn * xp + cs * xq;
                }
                double *vp = vv + (size_t)p * cols, *vq = vv + (size_t)q * cols;
                for (int i = 0; i < cols; ++i) {
                    const double xp = vp[i], xq = vq[i];
                    vp[i] = cs * xp - sn * xq;
                    vq[i] = sn * xp + cs * xq;
                }
            }
        }
        if (!rotated) break;
    }
    /* norms and descending order */
    double *nrm = (double *)malloc(sizeof(double) * cols);
    int *ord = (int *)malloc(sizeof(int) * cols);
    for (int j = 0; j < cols; ++j) {
        double s = 0;
        const double *bj = b + (size_t)j * rows;
        for (int i = 0; i < rows; ++i) s += bj[i] * bj[i];
        nrm[j] = sqrt(s);
        ord[j] = j;
    }
    for (int i = 1; i < cols; ++i) { /* insertion sort, stable */
        int k = ord[i];
        int j = i - 1;
        while (j >= 0 && nrm[ord[j]] < nrm[k]) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = k;
    }
    for (int jj = 0; jj < cols; ++jj) {
        const int j = ord[jj];
        sv[jj] = nrm[j];
        if (u) {
            const double *bj = b + (size_t)j * rows;
            for (int i = 0; i < rows; ++i) u[(size_t)jj * rows + i] = nrm[j] > 0 ? bj[i] / nrm[j] : 0.0;
        }
        if (v) memcpy(v + (size_t)jj * cols, vv + (size_t)j * cols, sizeof(double) * cols);
    }
    free(nrm); free(ord); free(b); free(vv);
}

int orc_singular_values(int rows, int cols, const double *x, double *sv) {
    if (rows < cols) return ORC_ERR_DIMENSION;
    jacobi_svd(rows, cols, x, sv, NULL, NULL);
    return ORC_OK;
}

/* Householder QR with column pivoting, then solve R z = Q^T y, w[perm] = z. */
static void colpiv_qr_solve(int rows, int cols, const double *x, const double *y, double *w) {
    double *a = (double *)malloc(sizeof(double) * (size_t)rows * cols); /* column-major */
    double *rhs = (double *)malloc(sizeof(double) * rows);
    double *cn = (double *)malloc(sizeof(double) * cols);
    int *perm = (int *)malloc(sizeof(int) * cols);
    for (int j = 0; j < cols; ++j) {
        for (int i = 0; i < rows; ++i) a[(size_t)j * rows + i] = x[(size_t)i * cols + j];
        perm[j] = j;
    }
    memcpy(rhs, y, sizeof(double) * rows);
    for (int k = 0; k < cols; ++k) {
        /* pivot: largest remaining column norm (recomputed exactly) */
        int best = k;
        double bestn = -1.0;
        for (int j = k; j < cols; ++j) {
            double s = 0;
            const double *aj = a + (size_t)j * rows;
            for (int i = k; i < rows; ++i) s += aj[i] * aj[i];
            cn[j] = s;
            if (s > bestn) { bestn = s; best = j; }
        }
        if (best != k) {
            double *ak = a + (size_t)k * rows, *ab = a + (size_t)best * rows;
            for (int i = 0; i < rows; ++i) { double t = ak[i]; ak[i] = ab[i]; ab[i] = t; }
            int t = perm[k]; perm[k] = perm[best]; perm[best] = t;
        }
        double *ak = a + (size_t)k * rows;
        double alpha = sqrt(cn[best]);
        if (alpha == 0.0) continue;
        if (ak[k] > 0) alpha = -alpha;
        /* v = a_k - alpha e_k, stored in place (v_k = ak[k] - alpha) */
        const double vk = ak[k] - alpha;
        double vnorm2 = vk * vk;
        for (int i = k + 1; i < rows; ++i) vnorm2 += ak[i] * ak[i];
        ak[k] = vk;
        if (vnorm2 > 0) {
            for (int j = k + 1; j < cols; ++j) {
                double *aj = a + (size_t)j * rows;
                double d = 0;
                for (int i = k; i < rows; ++i) d += ak[i] * aj[i];
                const double f = 2.0 * d / vnorm2;
                for (int i = k; i < rows; ++i) aj[i] -= f * ak[i];
            }
            double d = 0;
            for (int i = k; i < rows; ++i) d += ak[i] * rhs[i];
            const double f = 2.0 * d / vnorm2;
            for (int i = k; i < rows; ++i) rhs[i] -= f * ak[i];
        }
        ak[k] = alpha; /* R(k,k); subdiagonal no longer needed below */
    }
    /* back substitution with R (upper triangle of a) */
    double *z = (double *)malloc(sizeof(double) * cols);
    for (int k = cols - 1; k >= 0; --k) {
        double s = rhs[k];
        for (int j = k + 1; j < cols; ++j) s -= a[(size_t)j * rows + k] * z[j];
        const double rkk = a[(size_t)k * rows + k];
        z[k] = rkk != 0.0 ? s / rkk : 0.0;
    }
    for (int k = 0; k < cols; ++k) w[perm[k]] = z[k];
    free(z); free(a); free(rhs); free(cn); free(perm);
}

int orc_lls_fit(int rows, int cols, const double *x, const double *y, double *w,
                double *gram_condition) {
    if (rows < cols) return ORC_ERR_DIMENSION; /* lls.cpp:11-12 */
    if (cols < 1) return ORC_ERR_DIMENSION;
    double *sv = (double *)malloc(sizeof(double) * cols);
    double *u = (double *)malloc(sizeof(double) * (size_t)rows * cols);
    double *v = (double *)malloc(sizeof(double) * (size_t)cols * cols);
    jacobi_svd(rows, cols, x, sv, u, v);
    const double smax = sv[0], smin = sv[cols - 1];
    const double rank_tol = smax * DBL_EPSILON * (double)(rows > cols ? rows : cols); /* :22-23 */
    int rank = 0;
    while (rank < cols && sv[rank] > rank_tol) ++rank;

    int st = ORC_OK;
    if (rank == cols) { /* :28-33 */
        colpiv_qr_solve(rows, cols, x, y, w);
        if (gram_condition) *gram_condition = (smax / smin) * (smax / smin);
    } else { /* :39-53, minimum-norm solution */
        double *coef = (double *)calloc(cols, sizeof(double));
        for (int i = 0; i < cols; ++i) {
            double d = 0;
            for (int r = 0; r < rows; ++r) d += u[(size_t)i * rows + r] * y[r];
            coef[i] = i < rank ? d / sv[i] : 0.0;
        }
        for (int j = 0; j < cols; ++j) {
            double s = 0;
            for (int i = 0; i < cols; ++i) s += v[(size_t)i * cols + j] * coef[i];
            w[j] = s;
        }
        double res = 0, yn = 0;
        for (int r = 0; r < rows; ++r) {
            double p = 0;
            for (int j = 0; j < cols; ++j) p += x[(size_t)r * cols + j] * w[j];
            res += (p - y[r]) * (p - y[r]);
            yn += y[r] * y[r];
        }
        res = sqrt(res);
        yn = sqrt(yn);
        if (res > 1e-8 * smax * (yn > 1.0 ? yn : 1.0)) { /* :43-49 */
            if (gram_condition)
                *gram_condition = smin > 0.0 ? (smax / smin) * (smax / smin) : INFINITY;
            st = ORC_ERR_ILL;
        } else if (gram_condition) {
            *gram_condition = (smax / sv[rank - 1]) * (smax / sv[rank - 1]); /* :51 */
        }
        free(coef);
    }
    free(sv); free(u); free(v);
    return st;
}
