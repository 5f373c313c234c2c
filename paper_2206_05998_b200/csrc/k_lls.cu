// LLS initialiser on sm_100a: replaces lls::fit (lls.cpp:10-54), batched.
//
// One CTA per design (slot).  All K users of a slot share the design, so the
// Gram matrix is accumulated once per slot (the reference refactorises the
// same design K times, eval.cpp:122).  For the IQ-widened design the real
// Gram X^T X = [[P, Q], [-Q, P]] is the real form of the complex Gram
// C = X^H X (M x M), and the widened LS solution is w0 = [Re c; -Im c] with
// c the complex LS solution -- so the kernel works on the M x M Hermitian
// problem: FP64 Gram accumulation, cyclic Jacobi eigensolve in shared memory
// (parallel round-robin ordering), pseudo-inverse solve for every user, then
// an FP64 residual pass that produces r0 = y - X w0 (the training targets of
// the frozen-branch formulation) and the rank-deficient
// consistency test of lls.cpp:43-49.
//
// Rank decision: the reference thresholds singular
// values of X at sigma_max * eps * max(rows, cols) (lls.cpp:22-25).  A Gram
// eigenvalue resolves sigma only down to ~sqrt(eps) sigma_max, so eigenvalues
// below 16 * eps * max(rows, cols) * lambda_max are treated as zero.  Exactly
// rank-deficient (noiseless under-loaded) and noisy full-rank designs are
// classified identically; only sigma in (~3e-13, ~2e-7) * sigma_max differ.
#include <float.h>
#include <math.h>

#include "kernels.cuh"

namespace noma_dev {

constexpr int kLlsMaxM = 64;     // complex columns (widened width <= 128)
constexpr int kLlsMaxE = 18;     // Gram/RHS entries per thread (registers)

__host__ __device__ inline int lls_chunk(int m) { return m <= 16 ? 64 : m <= 32 ? 32 : 16; }
// Gram row groups (a function of m only: see phase A)
__host__ __device__ inline int lls_row_groups(int m) { return m <= 16 ? 4 : m <= 32 ? 2 : 1; }

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One column's term of the widened prediction x_t . w0 (phase D and
// lls_r0_kernel: same rounding, so either pass gives the same r0 bits)
__device__ __forceinline__ double r0_even(double2 x, double w0a, double w1a) {
    return __fma_rn(x.x, w0a, __dmul_rn(x.y, w1a));
}
__device__ __forceinline__ double r0_odd(double2 x, double w0a, double w1a) {
    return __fma_rn(x.y, w0a, -__dmul_rn(x.x, w1a));
}

// Phase A register blocking: a thread accumulates 2 x 2 complex blocks
// (columns a, a+1 against columns b, b+1 of the design, or targets k, k+1) --
// four complex operands per row feed four MACs -- over the rows of its row
// group; MB = blocks per thread, row groups fill the CTA when blocks are few.
template <int MB>
__global__ void __launch_bounds__(kThreads) lls_kernel(LlsParams p) {
    extern __shared__ __align__(16) double smem[];
    const int m = p.m, K = p.K, d = blockIdx.x, tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int CH = lls_chunk(m);
    const bool cplx_layout = p.layout == NOMA_LAYOUT_WIDEN_COMPLEX;
    double *A = smem;                       // m*m complex (Gram -> eigenvalues)
    double *V = A + 2 * m * m;              // m*m complex eigenvectors
    double *D = V + 2 * m * m;              // m*K complex RHS X^H y, later the solutions c_k
    double *bufs = D + 2 * m * K;           // 2 x (CH rows of x | CH rows of y), complex
    const int bstride = 2 * CH * (m + 1) + 2 * CH * K;  // (+1: phase D's padded rows)
    double *rot = bufs + 2 * bstride;       // per pair: c, s, e_re, e_im
    double *lam = rot + 4 * (kLlsMaxM / 2 + 1);  // m eigenvalues
    double *red = lam + m;                  // 2 * kThreads reduction scratch
    double *U = bufs;                       // m*K complex: V^H d / lambda (reuses bufs)
    __shared__ int pair_p[kLlsMaxM / 2 + 1], pair_q[kLlsMaxM / 2 + 1];
    __shared__ int any_rot[2];    // by sweep parity; reset one sweep ahead
    __shared__ int round_rot[2];  // by round parity: some pair rotates
    __shared__ int chol_ok;       // fast path: every Cholesky pivot above the floor

    // Staging of CH rows of the design and the targets into buffer b with
    // cp.async (row-major complex rows are contiguous; REAL rows fill the Re
    // slots of zeroed buffers).
    for (int i = tid; i < 2 * bstride; i += kThreads) bufs[i] = 0.0;
    __syncthreads();
    const int nch = (p.nrow_c + CH - 1) / CH;
    auto issue = [&](int ch, int b) {
        const int t0 = ch * CH, tn = min(CH, p.nrow_c - t0);
        double *xb = bufs + b * bstride, *yb = xb + 2 * CH * m;
        if (cplx_layout) {
            const double *xs = p.design + ((size_t)d * p.nrow_c + t0) * m * 2;
            const double *ys = p.targets + ((size_t)d * p.nrow_c + t0) * K * 2;
            for (int i = tid; i < tn * m; i += kThreads) cp_async16(xb + 2 * i, xs + 2 * i);
            for (int i = tid; i < tn * K; i += kThreads) cp_async16(yb + 2 * i, ys + 2 * i);
        } else {
            const double *xs = p.design + ((size_t)d * p.nrow_c + t0) * m;
            for (int i = tid; i < tn * m; i += kThreads) cp_async8(xb + 2 * i, xs + i);
            for (int i = tid; i < tn * K; i += kThreads) {
                const int t = i / K, k = i - t * K;
                cp_async8(yb + 2 * i, p.targets + ((size_t)d * K + k) * p.rows + t0 + t);
            }
        }
        cp_async_commit();
    };

    const bool clk = NOMA_PROBE_ON(p.clocks && d == 0 && tid == 0);
    long long ck = clk ? clock64() : 0;
#define NOMA_LLS_CLK(I)                      \
    if (clk) {                               \
        const long long now = clock64();     \
        p.clocks[I] += now - ck;             \
        ck = now;                            \
    }
    // ---- phase A: Gram (upper 2x2 blocks) and RHS blocks in registers ------
    // Task = (row group g, block): rows t == g (mod RG) in order; the RG
    // partials are summed in group order.  RG depends on m only, so every
    // entry's arithmetic is independent of how many users share the fit --
    // batched and single-user fits agree bitwise (test_lls.cpp:120-134).
    const int nb = (m + 1) / 2, nk = (K + 1) / 2;
    const int ngb = nb * (nb + 1) / 2, nblk = ngb + nb * nk;
    const int RG = lls_row_groups(m);
    const int ntask = RG * nblk;
    int tg[MB], ba[MB], bb[MB];  // task row group, block coordinates (bb >= nb: targets)
    double acc[MB][4][2];
#pragma unroll
    for (int e = 0; e < MB; ++e) {
        const int task = tid + e * kThreads;
        tg[e] = ba[e] = bb[e] = -1;
        if (task < ntask) {
            const int g = task / nblk, id = task - g * nblk;
            tg[e] = g;
            if (id < ngb) {
                int A_ = 0, rem = id;
                while (rem >= nb - A_) { rem -= nb - A_; ++A_; }
                ba[e] = A_;
                bb[e] = A_ + rem;
            } else {
                ba[e] = (id - ngb) / nk;
                bb[e] = nb + (id - ngb) % nk;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[e][q][0] = acc[e][q][1] = 0.0;
    }
    long long wait_a = 0, wait_d = 0;  // probes: cycles thread 0 waits for staged rows
    issue(0, 0);
    for (int ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) issue(ch + 1, (ch + 1) & 1);
        const long long tw = clk ? clock64() : 0;
        if (ch + 1 < nch)
            cp_async_wait<1>();
        else
            cp_async_wait<0>();
        __syncthreads();
        if (clk) wait_a += clock64() - tw;
        const int t0 = ch * CH, tn = min(CH, p.nrow_c - t0);
        const double *xs = bufs + (ch & 1) * bstride, *ys = xs + 2 * CH * m;
        if (p.design32) {  // FP32 copy of the design for the training kernels
            for (int i = tid; i < tn * m; i += kThreads) {
                const int t = i / m, a = i - t * m;
                if (cplx_layout) {
                    float *o = p.design32 + ((size_t)d * p.nrow_c + t0 + t) * p.width;
                    o[a] = (float)xs[2 * i];
                    o[m + a] = (float)xs[2 * i + 1];
                } else {
                    p.design32[((size_t)d * p.nrow_c + t0 + t) * p.width + a] = (float)xs[2 * i];
                }
            }
        }
#pragma unroll
        for (int e = 0; e < MB; ++e) {
            if (tg[e] < 0) continue;
            const int a0 = 2 * ba[e], a1 = min(a0 + 1, m - 1);
            const bool rhs = bb[e] >= nb;
            const int c0 = rhs ? 2 * (bb[e] - nb) : 2 * bb[e];
            const int c1 = min(c0 + 1, (rhs ? K : m) - 1);
            const double *bp = rhs ? ys : xs;
            const int bst = rhs ? K : m;
            for (int t = tg[e]; t < tn; t += RG) {  // CH % RG == 0: global row parity kept
                const double2 x0 = *reinterpret_cast<const double2 *>(xs + 2 * (t * m + a0));
                const double2 x1 = *reinterpret_cast<const double2 *>(xs + 2 * (t * m + a1));
                const double2 y0 = *reinterpret_cast<const double2 *>(bp + 2 * (t * bst + c0));
                const double2 y1 = *reinterpret_cast<const double2 *>(bp + 2 * (t * bst + c1));
                // conj(x) * y: (xr yr + xi yi) + i (xr yi - xi yr)
                acc[e][0][0] += x0.x * y0.x + x0.y * y0.y;
                acc[e][0][1] += x0.x * y0.y - x0.y * y0.x;
                acc[e][1][0] += x0.x * y1.x + x0.y * y1.y;
                acc[e][1][1] += x0.x * y1.y - x0.y * y1.x;
                acc[e][2][0] += x1.x * y0.x + x1.y * y0.y;
                acc[e][2][1] += x1.x * y0.y - x1.y * y0.x;
                acc[e][3][0] += x1.x * y1.x + x1.y * y1.y;
                acc[e][3][1] += x1.x * y1.y - x1.y * y1.x;
            }
        }
        __syncthreads();  // buffer (ch & 1) is refilled by the next issue
    }
    NOMA_LLS_CLK(0)
    // group partials -> shared memory (bufs is free), summed in group order
    // (RG == 1: the thread's own sums are already final; stage them the same way
    // only when they fit, else write them directly below)
    double *part = bufs;  // [task][4][2]
    const bool staged = RG > 1 || (size_t)ntask * 8 <= (size_t)2 * bstride;
#pragma unroll
    for (int e = 0; e < MB; ++e)
        if (tg[e] >= 0 && staged)
            for (int q = 0; q < 4; ++q) {
                const int task = tid + e * kThreads;
                part[(task * 4 + q) * 2] = acc[e][q][0];
                part[(task * 4 + q) * 2 + 1] = acc[e][q][1];
            }
    __syncthreads();
    double fro = 0.0;  // squared Frobenius norm of the Gram (rotation invariant)
    // staged: thread -> blocks tid, tid + kThreads, ...; direct (RG == 1 and
    // too many blocks to stage): thread -> its own tasks (task == block).
#pragma unroll
    for (int e = 0; e < MB; ++e) {
    if (staged && e > 0) break;
    for (int id = staged ? tid : (tg[e] >= 0 ? tid + e * kThreads : nblk); id < nblk;
         id += staged ? kThreads : nblk) {
        int A_, B_;
        if (id < ngb) {
            int rem = id;
            A_ = 0;
            while (rem >= nb - A_) { rem -= nb - A_; ++A_; }
            B_ = A_ + rem;
        } else {
            A_ = (id - ngb) / nk;
            B_ = nb + (id - ngb) % nk;
        }
        const bool rhs = B_ >= nb;
        for (int q = 0; q < 4; ++q) {
            double sre = staged ? part[(id * 4 + q) * 2] : acc[e][q][0];
            double sim = staged ? part[(id * 4 + q) * 2 + 1] : acc[e][q][1];
            for (int g = 1; g < RG; ++g) {
                sre += part[((g * nblk + id) * 4 + q) * 2];
                sim += part[((g * nblk + id) * 4 + q) * 2 + 1];
            }
            const int a = 2 * A_ + (q >> 1);
            const int cidx = (rhs ? 2 * (B_ - nb) : 2 * B_) + (q & 1);
            if (a >= m) continue;
            if (rhs) {
                if (cidx < K) {
                    D[2 * (a * K + cidx)] = sre;
                    D[2 * (a * K + cidx) + 1] = sim;
                }
            } else if (cidx < m && cidx >= a) {
                A[2 * (a * m + cidx)] = sre;
                A[2 * (a * m + cidx) + 1] = cidx == a ? 0.0 : sim;
                A[2 * (cidx * m + a)] = sre;  // Hermitian mirror
                A[2 * (cidx * m + a) + 1] = cidx == a ? 0.0 : -sim;
                const double sq = sre * sre + (cidx == a ? 0.0 : sim * sim);
                fro += cidx == a ? sq : 2.0 * sq;
            }
        }
    }
    }
    for (int i = tid; i < m * m; i += kThreads) {
        V[2 * i] = (i / m == i % m) ? 1.0 : 0.0;
        V[2 * i + 1] = 0.0;
    }
    red[tid] = fro;
    __syncthreads();
    for (int s2 = kThreads / 2; s2 > 0; s2 >>= 1) {
        if (tid < s2) red[tid] += red[tid + s2];
        __syncthreads();
    }
    // Two-sided Jacobi leaves rounding-level off-diagonals of ~eps ||A||_F, so
    // that is the rotation threshold (a relative test against sqrt(a_pp a_qq)
    // never settles for the small noise eigenvalues of a near-far design).
    const double tol_rot = DBL_EPSILON * sqrt(red[0]);
    if (tid == 0) any_rot[0] = any_rot[1] = round_rot[0] = round_rot[1] = 0;
    __syncthreads();
    NOMA_LLS_CLK(1)

    // ---- fast path (mode 1): Cholesky of the Hermitian Gram C = L L^H in the
    // idle staging buffer, then L y = d, L^H c = y for every user in place.
    // A pivot below 1e-10 ||C||_F -- far above the rank threshold of phase C --
    // sends the slot down the Jacobi path instead, so the rank / status
    // decisions are those of the Jacobi path; the full-rank solution agrees
    // with the pseudo-inverse one to rounding.  The condition number is left
    // to a mode-2 launch (off the critical path).
    bool fast = false;
    const int ms = m + 1;  // padded row stride: column reads hit distinct banks
    if (p.mode == 1 && 4 * m * ms + m <= 2 * bstride) {
        // Right-looking, one barrier per pivot: step k reads column k of the
        // working matrix W (final after step k-1), updates W's trailing
        // lower triangle with the column scaled on the fly, and stores the
        // scaled column in the factor F -- F and W are separate, so no
        // thread writes what another reads within a step.
        double *W = bufs;              // m x m complex, lower triangle
        double *F = W + 2 * m * ms;    // the factor L (lower triangle)
        double *ilv = F + 2 * m * ms;  // 1 / L[k][k]
        for (int i = tid; i < m * m; i += kThreads) {
            W[2 * (i + i / m)] = A[2 * i];
            W[2 * (i + i / m) + 1] = A[2 * i + 1];
        }
        if (tid == 0) chol_ok = 1;
        const double floor_piv = 1e-10 * sqrt(red[0]);
        int msh = 0;  // trailing-block grid width 2^msh >= m - 1
        while ((1 << msh) < m - 1) ++msh;
        __syncthreads();
        for (int k = 0; k < m; ++k) {
            const double dkk = W[2 * (k * ms + k)];
            if (!(dkk > floor_piv)) {  // uniform: every thread read the same pivot
                if (tid == 0) chol_ok = 0;
                break;
            }
            // 1/sqrt by rsqrt + one Newton step (~1 ulp; an IEEE sqrt and
            // divide per pivot were the serial chain of this phase)
            double il = rsqrt(dkk);
            il = il * fma(-0.5 * dkk, il * il, 1.5);
            const double lkk = dkk * il;
            const int nt = m - k - 1;  // W[i][j] -= L[i][k] conj(L[j][k]), k < j <= i
            for (int t = tid; t < (nt << msh); t += kThreads) {
                const int i = k + 1 + (t >> msh), j = k + 1 + (t & ((1 << msh) - 1));
                if (j <= i) {
                    const double ar = W[2 * (i * ms + k)] * il, ai = W[2 * (i * ms + k) + 1] * il;
                    const double br = W[2 * (j * ms + k)] * il, bi = W[2 * (j * ms + k) + 1] * il;
                    W[2 * (i * ms + j)] -= ar * br + ai * bi;
                    W[2 * (i * ms + j) + 1] -= ai * br - ar * bi;
                }
            }
            for (int i = k + 1 + tid; i < m; i += kThreads) {
                F[2 * (i * ms + k)] = W[2 * (i * ms + k)] * il;
                F[2 * (i * ms + k) + 1] = W[2 * (i * ms + k) + 1] * il;
            }
            if (tid == 0) {
                F[2 * (k * ms + k)] = lkk;
                ilv[k] = il;
            }
            __syncthreads();
        }
        __syncthreads();
        fast = chol_ok != 0;
        if (fast) {
            // L y = d, then L^H c = y: one warp per user, lane a holds rows
            // a and a + 32 of the right-hand side in registers; each step
            // broadcasts the finished entry by shuffle (no block barriers)
            for (int k = warp; k < K; k += kThreads / 32) {
                double yr[2], yi[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int a = lane + 32 * h;
                    yr[h] = a < m ? D[2 * (a * K + k)] : 0.0;
                    yi[h] = a < m ? D[2 * (a * K + k) + 1] : 0.0;
                }
                for (int j = 0; j < m; ++j) {  // forward
                    const int hj = j >> 5;
                    double cr = __shfl_sync(0xffffffffu, hj ? yr[1] : yr[0], j & 31);
                    double ci = __shfl_sync(0xffffffffu, hj ? yi[1] : yi[0], j & 31);
                    cr *= ilv[j];
                    ci *= ilv[j];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = lane + 32 * h;
                        if (i == j) {
                            yr[h] = cr;
                            yi[h] = ci;
                        } else if (i > j && i < m) {
                            const double lr = F[2 * (i * ms + j)], li = F[2 * (i * ms + j) + 1];
                            yr[h] -= lr * cr - li * ci;
                            yi[h] -= lr * ci + li * cr;
                        }
                    }
                }
                for (int j = m - 1; j >= 0; --j) {  // backward: c_i -= conj(L[j][i]) c_j
                    const int hj = j >> 5;
                    double cr = __shfl_sync(0xffffffffu, hj ? yr[1] : yr[0], j & 31);
                    double ci = __shfl_sync(0xffffffffu, hj ? yi[1] : yi[0], j & 31);
                    cr *= ilv[j];
                    ci *= ilv[j];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int i = lane + 32 * h;
                        if (i == j) {
                            yr[h] = cr;
                            yi[h] = ci;
                        } else if (i < j) {
                            const double lr = F[2 * (j * ms + i)], li = -F[2 * (j * ms + i) + 1];
                            yr[h] -= lr * cr - li * ci;
                            yi[h] -= lr * ci + li * cr;
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {  // w0, as phase C
                    const int a = lane + 32 * h;
                    if (a >= m) continue;
                    D[2 * (a * K + k)] = yr[h];
                    D[2 * (a * K + k) + 1] = yi[h];
                    double *w = p.w0 + ((size_t)d * K + k) * p.width;
                    float *pw = p.plans ? p.plans + ((size_t)d * K + k) * p.plan_total : nullptr;
                    if (cplx_layout) {
                        w[a] = yr[h];
                        w[m + a] = -yi[h];
                        if (pw) {
                            pw[a] = (float)yr[h];
                            pw[m + a] = (float)(-yi[h]);
                        }
                    } else {
                        w[a] = yr[h];
                        if (pw) pw[a] = (float)yr[h];
                    }
                }
            }
            __syncthreads();
        }
    }
    double lmax = 0.0, lmin = INFINITY, lkeep = INFINITY;
    int rank = m;
    if (!fast) {
    // ---- phase B: cyclic Jacobi, round-robin pairs (circle method); each
    // round applies A <- U^H A U as independent 2x2 blocks (in place) and
    // V <- V U, two barriers per round.
    const int mm = m + (m & 1);
    const int npairs = mm / 2;
    // round_rot alternates by a round counter that runs across sweeps: the
    // last round of a sweep and the first of the next must not share a slot
    // (an identity round skips the second barrier, so a fast thread's write
    // for the next round could reach the slot a slow thread is still testing)
    int gr = 0;
    for (int sweep = 0; sweep < 30; ++sweep) {
        for (int r = 0; r < mm - 1; ++r, ++gr) {
            if (tid < npairs) {
                const int i = tid;
                const int pi = (i == 0) ? 0 : ((i - 1 + r) % (mm - 1)) + 1;
                const int j = mm - 1 - i;
                const int qi = (j == 0) ? 0 : ((j - 1 + r) % (mm - 1)) + 1;
                int pp = min(pi, qi), qq = max(pi, qi);
                double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
                if (qq < m) {
                    const double a = A[2 * (pp * m + pp)], b = A[2 * (qq * m + qq)];
                    const double hr = A[2 * (pp * m + qq)], hi = A[2 * (pp * m + qq) + 1];
                    const double h2 = hr * hr + hi * hi;
                    if (h2 > tol_rot * tol_rot) {
                        // short dependent chain of FP64 special functions:
                        // e = h/|h|, th = (b-a)/(2|h|), t = sgn/(|th|+sqrt(th^2+1)),
                        // c = 1/sqrt(1+t^2), s = t c
                        const double ih = rsqrt(h2);
                        er = hr * ih;
                        ei = hi * ih;
                        const double th = 0.5 * (b - a) * ih;
                        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(fma(th, th, 1.0)));
                        c = rsqrt(fma(t, t, 1.0));
                        s = t * c;
                        any_rot[sweep & 1] = 1;
                        round_rot[gr & 1] = 1;
                    }
                }
                pair_p[i] = pp;
                pair_q[i] = qq;  // qq == m: p is unpaired this round (m odd)
                rot[4 * i] = c;
                rot[4 * i + 1] = s;
                rot[4 * i + 2] = er;
                rot[4 * i + 3] = ei;
            }
            __syncthreads();
            // every thread has passed the previous sweep's break test
            if (r == 0 && tid == 0) any_rot[(sweep + 1) & 1] = 0;
            if (!round_rot[gr & 1]) continue;  // no pair rotates: identity round
            __syncthreads();
            if (tid == 0) round_rot[gr & 1] = 0;  // reset for round gr + 2
            // A block (row pair I, column pair J): rows get U^H, columns U
            for (int it = tid; it < npairs * npairs + npairs * m; it += kThreads) {
                if (it < npairs * npairs) {
                    const int I = it / npairs, J = it - I * npairs;
                    const int r0 = pair_p[I], r1 = pair_q[I], c0 = pair_p[J], c1 = pair_q[J];
                    const double ci = rot[4 * I], si = rot[4 * I + 1], eri = rot[4 * I + 2], eii = rot[4 * I + 3];
                    const double cj = rot[4 * J], sj = rot[4 * J + 1], erj = rot[4 * J + 2], eij = -rot[4 * J + 3];
                    if (si == 0.0 && sj == 0.0) continue;  // both rotations identity
                    const bool h1 = r1 < m, k1 = c1 < m;
                    double x[2][2][2];  // [row][col][re/im]
                    x[0][0][0] = A[2 * (r0 * m + c0)];
                    x[0][0][1] = A[2 * (r0 * m + c0) + 1];
                    x[0][1][0] = k1 ? A[2 * (r0 * m + c1)] : 0.0;
                    x[0][1][1] = k1 ? A[2 * (r0 * m + c1) + 1] : 0.0;
                    x[1][0][0] = h1 ? A[2 * (r1 * m + c0)] : 0.0;
                    x[1][0][1] = h1 ? A[2 * (r1 * m + c0) + 1] : 0.0;
                    x[1][1][0] = h1 && k1 ? A[2 * (r1 * m + c1)] : 0.0;
                    x[1][1][1] = h1 && k1 ? A[2 * (r1 * m + c1) + 1] : 0.0;
                    // rows: (x0, x1) <- (c x0 - s e x1, s x0 + c e x1), e = e^{+i phi_I}
                    double y[2][2][2];
                    for (int cc = 0; cc < 2; ++cc) {
                        const double zr = eri * x[1][cc][0] - eii * x[1][cc][1];
                        const double zi = eri * x[1][cc][1] + eii * x[1][cc][0];
                        y[0][cc][0] = ci * x[0][cc][0] - si * zr;
                        y[0][cc][1] = ci * x[0][cc][1] - si * zi;
                        y[1][cc][0] = si * x[0][cc][0] + ci * zr;
                        y[1][cc][1] = si * x[0][cc][1] + ci * zi;
                    }
                    // columns: (y0, y1) <- (c y0 - s e' y1, s y0 + c e' y1), e' = e^{-i phi_J}
                    for (int rr = 0; rr < 2; ++rr) {
                        const double zr = erj * y[rr][1][0] - eij * y[rr][1][1];
                        const double zi = erj * y[rr][1][1] + eij * y[rr][1][0];
                        x[rr][0][0] = cj * y[rr][0][0] - sj * zr;
                        x[rr][0][1] = cj * y[rr][0][1] - sj * zi;
                        x[rr][1][0] = sj * y[rr][0][0] + cj * zr;
                        x[rr][1][1] = sj * y[rr][0][1] + cj * zi;
                    }
                    A[2 * (r0 * m + c0)] = x[0][0][0];
                    A[2 * (r0 * m + c0) + 1] = x[0][0][1];
                    if (k1) {
                        A[2 * (r0 * m + c1)] = x[0][1][0];
                        A[2 * (r0 * m + c1) + 1] = x[0][1][1];
                    }
                    if (h1) {
                        A[2 * (r1 * m + c0)] = x[1][0][0];
                        A[2 * (r1 * m + c0) + 1] = x[1][0][1];
                    }
                    if (h1 && k1) {
                        A[2 * (r1 * m + c1)] = x[1][1][0];
                        A[2 * (r1 * m + c1) + 1] = x[1][1][1];
                    }
                } else {  // V <- V U on row `row`, column pair i
                    const int rem = it - npairs * npairs;
                    const int i = rem / m, row = rem - i * m;
                    const int pp = pair_p[i], qq = pair_q[i];
                    if (qq >= m) continue;
                    const double c = rot[4 * i], s = rot[4 * i + 1];
                    if (s == 0.0) continue;
                    const double er = rot[4 * i + 2], ei = -rot[4 * i + 3];  // e^{-i phi}
                    const double xr = V[2 * (row * m + pp)], xi = V[2 * (row * m + pp) + 1];
                    const double yr = V[2 * (row * m + qq)], yi = V[2 * (row * m + qq) + 1];
                    const double zr = er * yr - ei * yi, zi = er * yi + ei * yr;
                    V[2 * (row * m + pp)] = c * xr - s * zr;
                    V[2 * (row * m + pp) + 1] = c * xi - s * zi;
                    V[2 * (row * m + qq)] = s * xr + c * zr;
                    V[2 * (row * m + qq) + 1] = s * xi + c * zi;
                }
            }
            __syncthreads();
        }
        if (clk) p.clocks[5] = sweep + 1;
        if (!any_rot[sweep & 1]) break;
    }
    NOMA_LLS_CLK(2)

    // ---- phase C: eigenvalues, rank, pseudo-inverse solve.
    for (int i = tid; i < m; i += kThreads) lam[i] = A[2 * (i * m + i)];
    __syncthreads();
    for (int i = 0; i < m; ++i) {
        lmax = fmax(lmax, lam[i]);
        lmin = fmin(lmin, lam[i]);
    }
    const int big = p.rows > p.width ? p.rows : p.width;
    const double tol = lmax * 16.0 * DBL_EPSILON * (double)big;
    rank = 0;
    for (int i = 0; i < m; ++i)
        if (lam[i] > tol) {
            ++rank;
            lkeep = fmin(lkeep, lam[i]);
        }
    if (p.mode == 2) {  // condition numbers only: full-rank nets (the others get
                        // theirs from the solving launch, which takes this path)
        if (rank == m && p.cond)
            for (int k = tid; k < K; k += kThreads) p.cond[(size_t)d * K + k] = lmax / lmin;
        return;
    }
    // U[i][k] = (V_i^H d_k) / lambda_i for kept i, else 0
    for (int it = tid; it < m * K; it += kThreads) {
        const int i = it / K, k = it % K;
        double sr = 0.0, si = 0.0;
        if (lam[i] > tol) {
            for (int a = 0; a < m; ++a) {
                const double vr = V[2 * (a * m + i)], vi = V[2 * (a * m + i) + 1];
                const double dr = D[2 * (a * K + k)], di = D[2 * (a * K + k) + 1];
                sr += vr * dr + vi * di;  // conj(v) d
                si += vr * di - vi * dr;
            }
            sr /= lam[i];
            si /= lam[i];
        }
        U[2 * it] = sr;
        U[2 * it + 1] = si;
    }
    __syncthreads();
    // c_k[a] = sum_i V[a][i] U[i][k] -> D (complex), w0 written FP64
    for (int it = tid; it < m * K; it += kThreads) {
        const int a = it / K, k = it % K;
        double sr = 0.0, si = 0.0;
        for (int i = 0; i < m; ++i) {
            const double vr = V[2 * (a * m + i)], vi = V[2 * (a * m + i) + 1];
            const double ur = U[2 * (i * K + k)], ui = U[2 * (i * K + k) + 1];
            sr += vr * ur - vi * ui;
            si += vr * ui + vi * ur;
        }
        D[2 * it] = sr;
        D[2 * it + 1] = si;
        double *w = p.w0 + ((size_t)d * K + k) * p.width;
        float *pw = p.plans ? p.plans + ((size_t)d * K + k) * p.plan_total : nullptr;
        if (cplx_layout) {
            w[a] = sr;
            w[m + a] = -si;
            if (pw) {
                pw[a] = (float)sr;
                pw[m + a] = (float)(-si);
            }
        } else {
            w[a] = sr;
            if (pw) pw[a] = (float)sr;
        }
    }
    __syncthreads();
    }  // !fast
    NOMA_LLS_CLK(3)

    // a Cholesky-path design is full rank: status OK, and with p.fast its
    // residuals come from lls_r0_kernel (spread over many CTAs)
    if (p.fast && cplx_layout) {
        if (tid == 0) p.fast[d] = fast ? 1 : 0;
        if (fast) {
            for (int k = tid; k < K; k += kThreads)
                if (p.status) p.status[(size_t)d * K + k] = NOMA_OK;
            return;
        }
    }
    // ---- phase D: residuals r0 = y - X w0 (FP64) and their norms (status of
    // rank-deficient designs, lls.cpp:43-49)
    auto decide = [&](int k, double sr, double sy) {
        const double res = sqrt(sr), ynorm = sqrt(sy);
        const size_t net = (size_t)d * K + k;
        int st = NOMA_OK;
        double cond;
        if (rank == m) {
            cond = lmax / lmin;
        } else if (rank > 0 && res <= 1e-8 * sqrt(lmax) * fmax(1.0, ynorm)) {
            cond = lmax / lkeep;
        } else {
            st = NOMA_ERR_ILL_CONDITIONED;
            cond = lmin > 0.0 ? lmax / lmin : INFINITY;
        }
        if (p.cond && !fast) p.cond[net] = cond;
        if (p.status) p.status[net] = st;
    };
    if (cplx_layout) {
        // Rows staged by cp.async in chunks again (row stride m + 1 complex,
        // so a warp reading one column of 32 rows hits distinct banks);
        // TPU threads per user, each a row of the chunk at a time; per-user
        // sums over the threads in fixed order.
        const int TPU = kThreads / K, uk = tid / TPU, slot = tid - uk * TPU;
        const bool act = uk < K;
        const int ms1 = m + 1;
        auto issue_pad = [&](int ch, int b) {
            const int t0 = ch * CH, tn = min(CH, p.nrow_c - t0);
            double *xb = bufs + b * bstride, *yb = xb + 2 * CH * ms1;
            const double *xs = p.design + ((size_t)d * p.nrow_c + t0) * m * 2;
            const double *ys = p.targets + ((size_t)d * p.nrow_c + t0) * K * 2;
            for (int i = tid; i < tn * m; i += kThreads) cp_async16(xb + 2 * (i + i / m), xs + 2 * i);
            for (int i = tid; i < tn * K; i += kThreads) cp_async16(yb + 2 * i, ys + 2 * i);
            cp_async_commit();
        };
        __syncthreads();  // the factor / eigenvectors in bufs are dead
        double rr = 0.0, yy = 0.0;
        issue_pad(0, 0);
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) issue_pad(ch + 1, (ch + 1) & 1);
            const long long tw = clk ? clock64() : 0;
            if (ch + 1 < nch)
                cp_async_wait<1>();
            else
                cp_async_wait<0>();
            __syncthreads();
            if (clk) wait_d += clock64() - tw;
            const int t0 = ch * CH, tn = min(CH, p.nrow_c - t0);
            const double *xs = bufs + (ch & 1) * bstride, *ys = xs + 2 * CH * ms1;
            if (act) {
                const size_t net = (size_t)d * K + uk;
                // two rows at a time (independent chains), columns unrolled so
                // the operand loads run ahead; each sum keeps the column order
                for (int t = slot; t < tn; t += 2 * TPU) {
                    const int t2 = t + TPU < tn ? t + TPU : t;
                    double pe0 = 0.0, po0 = 0.0, pe1 = 0.0, po1 = 0.0;
#pragma unroll 8
                    for (int a = 0; a < m; ++a) {
                        const double2 x0 = *reinterpret_cast<const double2 *>(xs + 2 * (t * ms1 + a));
                        const double2 x1 = *reinterpret_cast<const double2 *>(xs + 2 * (t2 * ms1 + a));
                        const double w0a = D[2 * (a * K + uk)], w1a = -D[2 * (a * K + uk) + 1];
                        pe0 = __dadd_rn(pe0, r0_even(x0, w0a, w1a));  // row 2t = [Re x; Im x]
                        po0 = __dadd_rn(po0, r0_odd(x0, w0a, w1a));   // row 2t+1 = [Im x; -Re x]
                        pe1 = __dadd_rn(pe1, r0_even(x1, w0a, w1a));
                        po1 = __dadd_rn(po1, r0_odd(x1, w0a, w1a));
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        if (h == 1 && t2 == t) break;
                        const int tt = h ? t2 : t;
                        const double pe = h ? pe1 : pe0, po = h ? po1 : po0;
                        const double2 y = *reinterpret_cast<const double2 *>(ys + 2 * (tt * K + uk));
                        const double r_e = y.x - pe, r_o = y.y - po;
                        rr += r_e * r_e + r_o * r_o;
                        yy += y.x * y.x + y.y * y.y;
                        if (p.r0) {
                            p.r0[net * p.rows + 2 * (t0 + tt)] = (float)r_e;
                            p.r0[net * p.rows + 2 * (t0 + tt) + 1] = (float)r_o;
                        }
                    }
                }
            }
            __syncthreads();  // buffer (ch & 1) is refilled by the next issue
        }
        red[2 * tid] = rr;
        red[2 * tid + 1] = yy;
        __syncthreads();
        if (tid < K) {
            double sr = 0.0, sy = 0.0;
            for (int q = 0; q < TPU; ++q) {
                sr += red[2 * (tid * TPU + q)];
                sy += red[2 * (tid * TPU + q) + 1];
            }
            decide(tid, sr, sy);
        }
    } else {
        double *sums = red;  // [8 warps][8 users][2]
        for (int k0 = 0; k0 < K; k0 += 8) {
            const int kn = min(8, K - k0);
            double rr[8], yy[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) rr[k] = yy[k] = 0.0;
            for (int t = tid; t < p.nrow_c; t += kThreads) {
                double pe[8], po[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) pe[k] = po[k] = 0.0;
                // the row's samples are loaded four at a time, all in flight
                // before the FMAs (one dependent L2 load per column made this
                // phase latency-bound); the sums keep the column order
                for (int a0 = 0; a0 < m; a0 += 4) {
                    double2 xv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int a = a0 + u;
                        xv[u] = a >= m ? make_double2(0.0, 0.0)
                                : cplx_layout
                                    ? *reinterpret_cast<const double2 *>(p.design + (((size_t)d * p.nrow_c + t) * m + a) * 2)
                                    : make_double2(p.design[((size_t)d * p.nrow_c + t) * m + a], 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int a = a0 + u;
                        if (a >= m) break;
                        const double xr = xv[u].x, xi = xv[u].y;
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            if (k < kn) {
                                const double w0a = D[2 * (a * K + k0 + k)], w1a = -D[2 * (a * K + k0 + k) + 1];
                                pe[k] += xr * w0a + xi * w1a;  // row 2t = [Re x; Im x]
                                po[k] += xi * w0a - xr * w1a;  // row 2t+1 = [Im x; -Re x]
                            }
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (k >= kn) continue;
                    const size_t net = (size_t)d * K + k0 + k;
                    if (cplx_layout) {
                        const double2 y = *reinterpret_cast<const double2 *>(p.targets + (((size_t)d * p.nrow_c + t) * K + k0 + k) * 2);
                        const double r_e = y.x - pe[k], r_o = y.y - po[k];
                        rr[k] += r_e * r_e + r_o * r_o;
                        yy[k] += y.x * y.x + y.y * y.y;
                        if (p.r0) {
                            p.r0[net * p.rows + 2 * t] = (float)r_e;
                            p.r0[net * p.rows + 2 * t + 1] = (float)r_o;
                        }
                    } else {
                        const double y = p.targets[((size_t)d * K + k0 + k) * p.rows + t];
                        const double r_e = y - pe[k];
                        rr[k] += r_e * r_e;
                        yy[k] += y * y;
                        if (p.r0) p.r0[net * p.rows + t] = (float)r_e;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    rr[k] += __shfl_xor_sync(0xffffffffu, rr[k], o);
                    yy[k] += __shfl_xor_sync(0xffffffffu, yy[k], o);
                }
            if (lane == 0)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    sums[(warp * 8 + k) * 2] = rr[k];
                    sums[(warp * 8 + k) * 2 + 1] = yy[k];
                }
            __syncthreads();
            if (tid < kn) {
                double sr = 0.0, sy = 0.0;
                for (int w = 0; w < kThreads / 32; ++w) {
                    sr += sums[(w * 8 + tid) * 2];
                    sy += sums[(w * 8 + tid) * 2 + 1];
                }
                decide(k0 + tid, sr, sy);
            }
            __syncthreads();
        }
    }
    NOMA_LLS_CLK(4)
#undef NOMA_LLS_CLK
    if (clk) {
        p.clocks[6] = wait_a;
        p.clocks[7] = wait_d;
    }
}

// lls::predict (lls.cpp:62-66): yhat = narrow(X_widened w0), FP64, one thread
// per (net, row).  WIDEN: the widened rows 2t / 2t+1 of complex row t give
// Re / Im of the prediction directly.
__global__ void lls_predict_kernel(int layout, int S, int K, int rows, int width,
                                   const double *data, const double *w0, double *out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)S * K * rows) return;
    const int t = (int)(i % rows);
    const size_t net = i / rows;
    const int d = (int)(net / K);
    const double *w = w0 + net * width;
    if (layout == NOMA_LAYOUT_WIDEN_COMPLEX) {
        const int m = width / 2;
        const double *x = data + ((size_t)d * rows + t) * m * 2;
        double pe = 0.0, po = 0.0;
        for (int a = 0; a < m; ++a) {
            const double xr = x[2 * a], xi = x[2 * a + 1];
            pe += xr * w[a] + xi * w[m + a];
            po += xi * w[a] - xr * w[m + a];
        }
        out[2 * i] = pe;
        out[2 * i + 1] = po;
    } else {
        const double *x = data + ((size_t)d * rows + t) * width;
        double s = 0.0;
        for (int c = 0; c < width; ++c) s += x[c] * w[c];
        out[i] = s;
    }
}

int lls_predict_launch(int layout, int S, int K, int rows, int width, const double *data,
                       const double *w0, double *out, cudaStream_t st) {
    const size_t n = (size_t)S * K * rows;
    if (n == 0) return NOMA_OK;
    lls_predict_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(layout, S, K, rows, width,
                                                                     data, w0, out);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

// r0 = y - X w0 of the Cholesky-path designs (WIDEN layout), one thread per
// (design, user, complex row); phase D's arithmetic, column order.
__global__ void lls_r0_kernel(LlsParams p) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int m = p.m, K = p.K, nr = p.nrow_c;
    if (i >= (size_t)p.n_designs * K * nr) return;
    const int t = (int)(i % nr);
    const size_t net = i / nr;
    const int d = (int)(net / K);
    if (!p.fast[d]) return;
    const double *w = p.w0 + net * p.width;
    const double2 *x = reinterpret_cast<const double2 *>(p.design + ((size_t)d * nr + t) * m * 2);
    double pe = 0.0, po = 0.0;
    for (int a = 0; a < m; ++a) {
        const double2 xv = x[a];
        const double w0a = w[a], w1a = w[m + a];
        pe = __dadd_rn(pe, r0_even(xv, w0a, w1a));
        po = __dadd_rn(po, r0_odd(xv, w0a, w1a));
    }
    const double2 y = *reinterpret_cast<const double2 *>(p.targets + (((size_t)d * nr + t) * K + (net - (size_t)d * K)) * 2);
    p.r0[net * p.rows + 2 * t] = (float)(y.x - pe);
    p.r0[net * p.rows + 2 * t + 1] = (float)(y.y - po);
}

int lls_r0_launch(const LlsParams &p, cudaStream_t st) {
    const size_t n = (size_t)p.n_designs * p.K * p.nrow_c;
    if (!p.fast || !p.r0 || n == 0) return NOMA_OK;
    lls_r0_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

size_t lls_smem_bytes(int m, int K) {
    const size_t bstride = 2 * (size_t)lls_chunk(m) * (m + 1) + 2 * (size_t)lls_chunk(m) * K;
    size_t n = 2 * (size_t)m * m * 2 + 2 * (size_t)m * K + 2 * bstride + 4 * (kLlsMaxM / 2 + 1) + m +
               2 * kThreads;
    return n * sizeof(double);
}

int lls_launch(const LlsParams &p, cudaStream_t st) {
    if (p.m < 1 || p.m > kLlsMaxM) return NOMA_ERR_UNSUPPORTED;
    const int nent = p.m * (p.m + 1) / 2 + p.m * p.K;
    if (nent > kLlsMaxE * kThreads || p.K > kThreads) return NOMA_ERR_UNSUPPORTED;
    if (2 * p.m * p.K > 2 * (2 * lls_chunk(p.m) * (p.m + 1) + 2 * lls_chunk(p.m) * p.K)) return NOMA_ERR_UNSUPPORTED;
    const size_t smem = lls_smem_bytes(p.m, p.K);
    if (smem > 227 * 1024) return NOMA_ERR_UNSUPPORTED;
    const int nb = (p.m + 1) / 2, nk = (p.K + 1) / 2;
    const int nblk = nb * (nb + 1) / 2 + nb * nk;
    const int ntask = lls_row_groups(p.m) * nblk;
    const int mb = (ntask + kThreads - 1) / kThreads;
    if (mb > 8) return NOMA_ERR_UNSUPPORTED;
    // task partials [task][4][2] reuse the staging buffers when RG > 1
    if (lls_row_groups(p.m) > 1 &&
        (size_t)ntask * 8 > (size_t)2 * (2 * lls_chunk(p.m) * (p.m + 1) + 2 * lls_chunk(p.m) * p.K))
        return NOMA_ERR_UNSUPPORTED;
    // the shared-memory opt-in is raised once per device and kernel (a host
    // call per launch delayed the single-slot pipeline's critical path)
    static int smem_set[64][4] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    auto go = [&](auto kern, int ki) {
        int *have = dev >= 0 && dev < 64 ? &smem_set[dev][ki] : nullptr;
        if (!have || *have < (int)smem) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (have) *have = (int)smem;
        }
        kern<<<p.n_designs, kThreads, smem, st>>>(p);
    };
    if (mb == 1) go(lls_kernel<1>, 0);
    else if (mb == 2) go(lls_kernel<2>, 1);
    else if (mb <= 4) go(lls_kernel<4>, 2);
    else go(lls_kernel<8>, 3);
    return cudaGetLastError() == cudaSuccess ? NOMA_OK : NOMA_ERR_CUDA;
}

}  // namespace noma_dev
