/*
 * TEST INFRASTRUCTURE ONLY -- FP64 CPU restatement (see noma_oracle.h).
 *
 * One slot end to end, composed the way the reference's callers compose the
 * hot path: noma_cli.cpp:86-160 (train + detect per user, seed conventions
 * :97 and :103) and eval.cpp:228-241 (users run sequentially).  The threaded
 * variant spreads independent slots over pthreads for the CPU baseline
 * (per-user trainings are independent).
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "noma_oracle.h"

int orc_slot_run(const orc_slot_cfg *cfg, uint64_t seed, double *w0_out, double *cond_out,
                 int *status_out, double *plan_out, double *trace_out, double *soft_out,
                 long *err_out) {
    const orc_scenario *sc = &cfg->sc;
    const int K = sc->num_users, M = sc->num_antennas;
    const int NT = sc->train_symbols, ND = sc->data_symbols;
    const int nd = cfg->ndims;
    const int *d = cfg->dims;
    if (d[0] != 2 * M) return ORC_ERR_DIMENSION;
    int st = orc_scenario_validate(sc);
    if (st) return st;

    uint64_t sb[3];
    orc_seed_bundle(seed, sb);
    double *chan = malloc(sizeof(double) * 2 * M * K), *pw = malloc(sizeof(double) * K);
    double *trx = malloc(sizeof(double) * 2 * (size_t)NT * M);
    double *tsym = malloc(sizeof(double) * 2 * (size_t)NT * K);
    double *drx = malloc(sizeof(double) * 2 * (size_t)ND * M);
    double *dsym = malloc(sizeof(double) * 2 * (size_t)ND * K);
    double np;
    orc_synthesize(sc, sb[0], sb[1], sb[2], chan, pw, trx, tsym, drx, dsym, &np);

    const int w = 2 * M;
    double *xt = malloc(sizeof(double) * (size_t)2 * NT * w);
    double *xd = malloc(sizeof(double) * (size_t)2 * ND * w);
    orc_widen_design(NT, M, trx, xt);
    orc_widen_design(ND, M, drx, xd);
    double *yt = malloc(sizeof(double) * 2 * NT);
    const int P = orc_param_count(nd, d), PS = orc_plan_size(nd, d);
    double *theta = malloc(sizeof(double) * P);
    double *w0 = malloc(sizeof(double) * w);
    double *pred = malloc(sizeof(double) * 2 * (size_t)ND);
    uint8_t *bits = malloc(2 * (size_t)ND), *truth = malloc(2 * (size_t)ND);

    for (int k = 0; k < K; ++k) {
        const int user = k + 1;
        orc_widen_targets(NT, tsym + 2 * k, K, yt);
        double cond = 0.0;
        int s = orc_lls_fit(2 * NT, w, xt, yt, w0, &cond);
        if (status_out) status_out[k] = s;
        if (cond_out) cond_out[k] = cond;
        if (s != ORC_OK) {
            if (err_out) err_out[k] = -1;
            continue;
        }
        if (w0_out) memcpy(w0_out + (size_t)k * w, w0, sizeof(double) * w);
        orc_rng init_rng;
        orc_rng_seed(&init_rng, orc_substream_seed(seed, 0x1000u + (unsigned)user));
        orc_init_params(nd, d, &init_rng, theta);
        orc_train(nd, d, w0, theta, 2 * NT, xt, yt, cfg->epochs, cfg->batch, cfg->lr,
                  orc_substream_seed(seed, (unsigned)user),
                  trace_out ? trace_out + (size_t)k * cfg->epochs : NULL);
        if (plan_out) orc_build_plan(nd, d, w0, theta, plan_out + (size_t)k * PS);
        orc_forward(nd, d, w0, theta, 2 * ND, xd, pred);
        if (soft_out) memcpy(soft_out + (size_t)k * 2 * ND, pred, sizeof(double) * 2 * ND);
        orc_hard_decision_qpsk(ND, pred, 1, bits);
        orc_hard_decision_qpsk(ND, dsym + 2 * k, K, truth);
        if (err_out) err_out[k] = orc_bit_errors(2 * ND, bits, truth);
    }
    free(chan); free(pw); free(trx); free(tsym); free(drx); free(dsym);
    free(xt); free(xd); free(yt); free(theta); free(w0); free(pred); free(bits); free(truth);
    return ORC_OK;
}

typedef struct {
    const orc_slot_cfg *cfg;
    int S;
    const uint64_t *seeds;
    int *next;
    pthread_mutex_t *mu;
    double *w0, *cond, *plan, *trace, *soft;
    int *status;
    long *err;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    const orc_slot_cfg *c = j->cfg;
    const int K = c->sc.num_users, w = c->dims[0], PS = orc_plan_size(c->ndims, c->dims);
    for (;;) {
        pthread_mutex_lock(j->mu);
        const int s = (*j->next)++;
        pthread_mutex_unlock(j->mu);
        if (s >= j->S) break;
        orc_slot_run(c, j->seeds[s], j->w0 ? j->w0 + (size_t)s * K * w : NULL,
                     j->cond ? j->cond + (size_t)s * K : NULL,
                     j->status ? j->status + (size_t)s * K : NULL,
                     j->plan ? j->plan + (size_t)s * K * PS : NULL,
                     j->trace ? j->trace + (size_t)s * K * c->epochs : NULL,
                     j->soft ? j->soft + (size_t)s * K * 2 * c->sc.data_symbols : NULL,
                     j->err ? j->err + (size_t)s * K : NULL);
    }
    return NULL;
}

int orc_slots_run_threaded(const orc_slot_cfg *cfg, int S, const uint64_t *seeds, int threads,
                           double *w0, double *cond, int *status, double *plan, double *trace,
                           double *soft, long *err) {
    if (threads < 1) threads = 1;
    int next = 0;
    pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
    job_t job = {cfg, S, seeds, &next, &mu, w0, cond, plan, trace, soft, status, err};
    pthread_t *th = malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &job);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
    return ORC_OK;
}
