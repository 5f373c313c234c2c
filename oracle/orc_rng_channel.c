/*
 * TEST INFRASTRUCTURE ONLY -- FP64 CPU restatement (see noma_oracle.h).
 *
 * RNG (rng.hpp:10-67), seed mixing (eval.cpp:77-84), channel synthesis
 * (channel_sim.cpp:9-117) and IQ widening (iq_transform.cpp:7-54).
 *
 * Argument-evaluation order: the reference builds complex draws as
 * `cplx(rng.gaussian() * s, rng.gaussian() * s)` (channel_sim.cpp:56, :71).
 * C++ leaves the order of constructor arguments unspecified; g++ (the
 * reference's recorded Linux build, test_output.txt:1) evaluates them right to
 * left, so the FIRST draw lands in the IMAGINARY part.  This is pinned by
 * tests/golden/probe_eval_order.cpp and restated here explicitly.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "noma_oracle.h"

static const double kPi = 3.141592653589793238462643383279502884; /* std::numbers::pi */

uint64_t orc_splitmix64(uint64_t *state) { /* rng.hpp:10-15 */
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t orc_substream_seed(uint64_t master, uint64_t tag) { /* rng.hpp:18-23 */
    uint64_t s = master;
    uint64_t a = orc_splitmix64(&s);
    s = a ^ (tag * 0xD1B54A32D192ED03ULL + 0x8BB84B93962EACC9ULL);
    return orc_splitmix64(&s);
}

/* eval.cpp:77-84.  `s ^= splitmix64(s) + b` -- C++17 sequences the right
 * operand first, so the xor uses the advanced s. */
uint64_t orc_mix_tag(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    uint64_t s = a * 0x9E3779B97F4A7C15ULL + 1;
    uint64_t t;
    t = orc_splitmix64(&s) + b; s ^= t;
    t = orc_splitmix64(&s) + c; s ^= t;
    t = orc_splitmix64(&s) + d; s ^= t;
    return orc_splitmix64(&s);
}

void orc_rng_seed(orc_rng *r, uint64_t seed) { /* rng.hpp:30-33 */
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = orc_splitmix64(&sm);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

uint64_t orc_rng_next(orc_rng *r) { /* rng.hpp:35-45, xoshiro256++ */
    uint64_t *s = r->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

double orc_rng_uniform(orc_rng *r) { /* rng.hpp:48 */
    return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
}

uint64_t orc_rng_below(orc_rng *r, uint64_t bound) { /* rng.hpp:51-54 */
    return (uint64_t)(((unsigned __int128)orc_rng_next(r) * bound) >> 64);
}

double orc_rng_gaussian(orc_rng *r) { /* rng.hpp:58-62, Box-Muller cosine half */
    double u1 = 1.0 - orc_rng_uniform(r);
    double u2 = orc_rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

void orc_rng_fill_u64(uint64_t seed, int n, uint64_t *out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = orc_rng_next(&r);
}

void orc_rng_fill_gaussian(uint64_t seed, int n, double *out) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int i = 0; i < n; ++i) out[i] = orc_rng_gaussian(&r);
}

/* ------------------------------------------------------------------ */

int orc_scenario_validate(const orc_scenario *c) { /* channel_sim.cpp:9-21 */
    if (c->num_users < 1) return ORC_ERR_CONFIG;
    if (c->num_antennas < 1) return ORC_ERR_CONFIG;
    if (c->train_symbols < 1 || c->data_symbols < 1) return ORC_ERR_CONFIG;
    if (c->train_symbols < 2 * c->num_antennas) return ORC_ERR_CONFIG;
    if (c->power_step_db < 0.0) return ORC_ERR_CONFIG;
    if (c->rx_nonlinearity_gain < 0.0) return ORC_ERR_CONFIG;
    if (isnan(c->snr_db)) return ORC_ERR_CONFIG;
    return ORC_OK;
}

void orc_power_profile(int num_users, double step_db, double *p) { /* :23-28 */
    for (int k = 0; k < num_users; ++k) p[k] = pow(10.0, (double)(-k) * step_db / 10.0);
}

int orc_gen_symbols(int K, int N, orc_rng *r, double *out) { /* :30-47 */
    if (K < 1 || N < 1) return ORC_ERR_DIMENSION;
    const double a = 1.0 / sqrt(2.0);
    for (int t = 0; t < N; ++t) {
        for (int k = 0; k < K; ++k) { /* row-major draw order */
            uint64_t bits = orc_rng_below(r, 4);
            out[((size_t)t * K + k) * 2 + 0] = (bits & 1) ? -a : a;
            out[((size_t)t * K + k) * 2 + 1] = (bits & 2) ? -a : a;
        }
    }
    return ORC_OK;
}

int orc_gen_channel(int K, int M, orc_rng *r, double *h) { /* :49-58 */
    if (K < 1 || M < 1) return ORC_ERR_DIMENSION;
    const double s = 1.0 / sqrt(2.0);
    for (int k = 0; k < K; ++k) {
        for (int m = 0; m < M; ++m) {
            /* g++ right-to-left argument evaluation: imaginary part first */
            double im = orc_rng_gaussian(r) * s;
            double re = orc_rng_gaussian(r) * s;
            h[((size_t)m * K + k) * 2 + 0] = re;
            h[((size_t)m * K + k) * 2 + 1] = im;
        }
    }
    return ORC_OK;
}

void orc_seed_bundle(uint64_t master, uint64_t out3[3]) { /* channel_sim.hpp:38-41 */
    out3[0] = orc_substream_seed(master, 1);
    out3[1] = orc_substream_seed(master, 2);
    out3[2] = orc_substream_seed(master, 3);
}

/* X = B diag(sqrt p) H^T, row t: x(t,m) = sum_k b(t,k) * (h(m,k) sqrt(p_k)) */
static void superpose(int N, int M, int K, const double *sym, const double *scaled,
                      double *x) {
    for (int t = 0; t < N; ++t) {
        for (int m = 0; m < M; ++m) {
            double re = 0.0, im = 0.0;
            for (int k = 0; k < K; ++k) {
                const double a = sym[((size_t)t * K + k) * 2], b = sym[((size_t)t * K + k) * 2 + 1];
                const double c = scaled[((size_t)m * K + k) * 2], d = scaled[((size_t)m * K + k) * 2 + 1];
                re += a * c - b * d;
                im += a * d + b * c;
            }
            x[((size_t)t * M + m) * 2] = re;
            x[((size_t)t * M + m) * 2 + 1] = im;
        }
    }
}

static void cubic_distortion(size_t n, double *x, double gain) { /* :62-65 */
    if (gain <= 0.0) return;
    for (size_t i = 0; i < n; ++i) {
        const double re = x[2 * i], im = x[2 * i + 1];
        const double nrm = re * re + im * im; /* std::norm */
        x[2 * i] = re + (gain * re) * nrm;    /* u + (gain*u)*norm(u) */
        x[2 * i + 1] = im + (gain * im) * nrm;
    }
}

static void add_noise(size_t rows, int M, double *x, double sigma2, orc_rng *r) { /* :67-72 */
    const double s = sqrt(sigma2 / 2.0);
    for (size_t t = 0; t < rows; ++t)
        for (int m = 0; m < M; ++m) {
            double im = orc_rng_gaussian(r) * s; /* right-to-left, see header */
            double re = orc_rng_gaussian(r) * s;
            x[(t * M + m) * 2] += re;
            x[(t * M + m) * 2 + 1] += im;
        }
}

int orc_synthesize(const orc_scenario *sc, uint64_t sym_seed, uint64_t chan_seed,
                   uint64_t noise_seed, double *channel, double *powers, double *train_rx,
                   double *train_sym, double *data_rx, double *data_sym, double *noise_power) {
    int st = orc_scenario_validate(sc);
    if (st) return st;
    const int K = sc->num_users, M = sc->num_antennas;
    const int NT = sc->train_symbols, ND = sc->data_symbols;
    orc_rng sym_rng, chan_rng, noise_rng;
    orc_rng_seed(&sym_rng, sym_seed);
    orc_rng_seed(&chan_rng, chan_seed);
    orc_rng_seed(&noise_rng, noise_seed);

    orc_power_profile(K, sc->power_step_db, powers);
    orc_gen_channel(K, M, &chan_rng, channel);
    orc_gen_symbols(K, NT, &sym_rng, train_sym);
    orc_gen_symbols(K, ND, &sym_rng, data_sym);

    double *scaled = (double *)malloc(sizeof(double) * 2 * (size_t)M * K);
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) {
            const double sp = sqrt(powers[k]);
            scaled[((size_t)m * K + k) * 2] = channel[((size_t)m * K + k) * 2] * sp;
            scaled[((size_t)m * K + k) * 2 + 1] = channel[((size_t)m * K + k) * 2 + 1] * sp;
        }
    superpose(NT, M, K, train_sym, scaled, train_rx);
    superpose(ND, M, K, data_sym, scaled, data_rx);
    free(scaled);

    cubic_distortion((size_t)NT * M, train_rx, sc->rx_nonlinearity_gain);
    cubic_distortion((size_t)ND * M, data_rx, sc->rx_nonlinearity_gain);

    if (isinf(sc->snr_db)) {
        *noise_power = 0.0;
    } else {
        double sig = 0.0;
        for (int k = 0; k < K; ++k) {
            double nrm = 0.0; /* squaredNorm of column k */
            for (int m = 0; m < M; ++m) {
                const double re = channel[((size_t)m * K + k) * 2], im = channel[((size_t)m * K + k) * 2 + 1];
                nrm += re * re + im * im;
            }
            sig += powers[k] * nrm;
        }
        const double np = sig / (M * pow(10.0, sc->snr_db / 10.0));
        *noise_power = np;
        add_noise((size_t)NT, M, train_rx, np, &noise_rng);
        add_noise((size_t)ND, M, data_rx, np, &noise_rng);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */

int orc_widen_design(int n, int m, const double *x, double *out) { /* iq_transform.cpp:7-24 */
    if (n == 0 || m == 0) return ORC_ERR_DIMENSION;
    const int w = 2 * m;
    for (int t = 0; t < n; ++t)
        for (int j = 0; j < m; ++j) {
            const double re = x[((size_t)t * m + j) * 2], im = x[((size_t)t * m + j) * 2 + 1];
            out[(size_t)(2 * t) * w + j] = re;
            out[(size_t)(2 * t) * w + m + j] = im;
            out[(size_t)(2 * t + 1) * w + j] = im;
            out[(size_t)(2 * t + 1) * w + m + j] = -re;
        }
    return ORC_OK;
}

void orc_widen_targets(int n, const double *y, int stride, double *out) { /* :26-33 */
    for (int t = 0; t < n; ++t) {
        out[2 * t] = y[(size_t)t * stride * 2];
        out[2 * t + 1] = y[(size_t)t * stride * 2 + 1];
    }
}

int orc_narrow_predictions(int n2, const double *yhat, double *out) { /* :47-54 */
    if (n2 % 2 != 0) return ORC_ERR_DIMENSION;
    memcpy(out, yhat, sizeof(double) * (size_t)n2);
    return ORC_OK;
}

/* eval.cpp:38-45: bit = (x < 0); 0, -0 and NaN decide to bit 0 */
void orc_hard_decision_qpsk(int n, const double *sym, int stride, uint8_t *bits) {
    for (int t = 0; t < n; ++t) {
        bits[2 * t] = sym[(size_t)t * stride * 2] < 0.0 ? 1 : 0;
        bits[2 * t + 1] = sym[(size_t)t * stride * 2 + 1] < 0.0 ? 1 : 0;
    }
}

long orc_bit_errors(int n2, const uint8_t *a, const uint8_t *b) { /* eval.cpp:56-65 */
    long e = 0;
    for (int i = 0; i < n2; ++i) e += a[i] != b[i];
    return e;
}
