/*
 * heat_oracle.c — CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as
 * the checker or the timed CPU baseline.  The product path never calls it.
 *
 * What it restates (all paths under /root/reference/pkg/src/heatcf/):
 *   - SplitMix64 streams            rng.py:26-39 (mix64, derive_stream),
 *                                   rng.py:63-76 (rng_next, rng_below)
 *   - the per-pair SGD loop         trainer.py:103-331, the branch with
 *                                   tiled=False, agg_on=False, for both
 *                                   use_cosine=True and use_cosine=False
 *   - the threaded epoch driver     trainer.py:385-466 (chunk claiming from a
 *                                   shared counter, per-thread streams salted
 *                                   with (0x45504F43, epoch, tid))
 *
 * Arithmetic contract: every expression below is evaluated in the same order
 * and with the same roundings as the reference's JIT code — IEEE binary64,
 * no FMA contraction (build with -ffp-contract=off), correctly rounded sqrt
 * and division, float32 rounding on store.  tests/test_oracle_golden.py pins
 * this file bit-for-bit against vectors produced by the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define HO_GAMMA 0x9E3779B97F4A7C15ULL
#define HO_MIX1 0xBF58476D1CE4E5B9ULL
#define HO_MIX2 0x94D049BB133111EBULL

/* rng.py:26-31 */
uint64_t ho_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * HO_MIX1;
    x = (x ^ (x >> 27)) * HO_MIX2;
    return x ^ (x >> 31);
}

/* rng.py:34-39 */
uint64_t ho_derive_stream(uint64_t seed, const uint64_t *words, int nwords) {
    uint64_t state = ho_mix64(seed);
    for (int i = 0; i < nwords; ++i) state = ho_mix64(state + HO_GAMMA + words[i]);
    return state;
}

/* rng.py:63-70: advance in place, return the draw */
static inline uint64_t rng_next(uint64_t *state) {
    *state += HO_GAMMA;
    return ho_mix64(*state);
}

/* rng.py:73-76 */
static inline int64_t rng_below(uint64_t *state, int64_t n) {
    return (int64_t)(rng_next(state) % (uint64_t)n);
}

/* Fill out[p*n_neg + j] with the negatives the reference draws for the
 * pairs [0, npairs) of one sequential stream starting at *state
 * (trainer.py:135-139).  Advances *state. */
void ho_sample_negatives(uint64_t *state, int64_t npairs, int n_neg, int64_t num_items,
                         int32_t *out) {
    for (int64_t i = 0; i < npairs * (int64_t)n_neg; ++i) out[i] = (int32_t)rng_below(state, num_items);
}

typedef struct {
    /* per-thread scratch, trainer.py:334-363 (tile buffers dropped) */
    int K, n_neg;
    double *ubuf, *ugrad, *tts, *sts, *sims, *dnegs, *pooled, *wh;
    float *pos_buf, *neg_buf;
    int32_t *neg_ids;
} ho_scratch;

/* Behaviour aggregation (aggregator.py:30-113, in-loop copy trainer.py:148-173
 * and 299-331).  accu (K*K f64) and counter are the per-thread state that
 * persists across chunks of an epoch (_ThreadState.agg_accu / agg_ctr). */
typedef struct {
    int on;
    float *W;                 /* K x K, input-major: W[k*K + j] */
    const int64_t *tr_offsets;
    const int32_t *tr_items;
    double gamma, lr;
    int64_t mb_size, max_history;
    int hist_prop;
    double *accu;
    int64_t *counter;
} ho_agg;

static int scratch_init(ho_scratch *s, int K, int n_neg) {
    s->K = K;
    s->n_neg = n_neg;
    s->ubuf = calloc((size_t)K, sizeof(double));
    s->pooled = calloc((size_t)K, sizeof(double));
    s->wh = calloc((size_t)K, sizeof(double));
    s->ugrad = calloc((size_t)K, sizeof(double));
    s->tts = calloc((size_t)n_neg, sizeof(double));
    s->sts = calloc((size_t)n_neg, sizeof(double));
    s->sims = calloc((size_t)n_neg, sizeof(double));
    s->dnegs = calloc((size_t)n_neg, sizeof(double));
    s->pos_buf = calloc((size_t)K, sizeof(float));
    s->neg_buf = calloc((size_t)n_neg * K, sizeof(float));
    s->neg_ids = calloc((size_t)n_neg, sizeof(int32_t));
    return s->ubuf && s->pooled && s->wh && s->ugrad && s->tts && s->sts && s->sims && s->dnegs && s->pos_buf &&
                   s->neg_buf && s->neg_ids
               ? 0
               : -1;
}

static void scratch_free(ho_scratch *s) {
    free(s->ubuf); free(s->pooled); free(s->wh); free(s->ugrad); free(s->tts); free(s->sts); free(s->sims);
    free(s->dnegs); free(s->pos_buf); free(s->neg_buf); free(s->neg_ids);
}

/* The per-pair loop of trainer.py:114-297 for tiled=False, agg_on=False.
 * S is (S_rows, K) and T is (num_items, K), both float32 row-major.
 * loss_out/degen_out accumulate like the reference's per-thread outputs;
 * active_out counts negatives with dnegs[j] != 0 (our telemetry, not the
 * reference's).  The last pair's negative ids stay in s->neg_ids. */
static void train_chunk(float *S, float *T, const int32_t *ep_users, const int32_t *ep_items,
                        int64_t start, int64_t stop, int64_t num_items, uint64_t *rng_state,
                        int use_cosine, int n_neg, double lr, double l2, double mu, double theta,
                        const ho_agg *ag, ho_scratch *s, double *loss_out, int64_t *degen_out,
                        int64_t *active_out) {
    const int K = s->K;
    const double inv_n = 1.0 / n_neg;
    double *ubuf = s->ubuf, *ugrad = s->ugrad, *tts = s->tts, *sts = s->sts, *sims = s->sims,
           *dnegs = s->dnegs;
    float *pos_buf = s->pos_buf, *neg_buf = s->neg_buf;
    int32_t *neg_ids = s->neg_ids;
    for (int64_t i = start; i < stop; ++i) {
        const int64_t u = ep_users[i];
        const int64_t pos = ep_items[i];
        /* read: trainer.py:121-142 */
        for (int k = 0; k < K; ++k) pos_buf[k] = T[pos * K + k];
        for (int j = 0; j < n_neg; ++j) {
            int64_t nid = rng_below(rng_state, num_items);
            neg_ids[j] = (int32_t)nid;
            for (int k = 0; k < K; ++k) neg_buf[(int64_t)j * K + k] = T[nid * K + k];
        }
        if (!ag->on) {
            for (int k = 0; k < K; ++k) ubuf[k] = (double)S[u * K + k];
        }

        /* aggregate forward: trainer.py:150-169 */
        int64_t hb = 0, hist_len = 0;
        double *pooled = s->pooled;
        if (ag->on) {
            hb = ag->tr_offsets[u];
            int64_t he = ag->tr_offsets[u + 1];
            if (he - hb > ag->max_history) he = hb + ag->max_history;
            hist_len = he - hb;
            for (int k = 0; k < K; ++k) pooled[k] = 0.0;
            for (int64_t idx = hb; idx < he; ++idx) {
                const int64_t hid = ag->tr_items[idx];
                for (int k = 0; k < K; ++k) pooled[k] += (double)T[hid * K + k];
            }
            if (hist_len > 0)
                for (int k = 0; k < K; ++k) pooled[k] /= (double)hist_len;
            for (int j = 0; j < K; ++j) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc += pooled[k] * (double)ag->W[k * K + j];
                ubuf[j] = ag->gamma * (double)S[u * K + j] + (1.0 - ag->gamma) * acc;
            }
        }

        /* similarity: trainer.py:176-207 */
        double ss = 0.0;
        for (int k = 0; k < K; ++k) ss += ubuf[k] * ubuf[k];
        double tt_p = 0.0, st_p = 0.0;
        for (int k = 0; k < K; ++k) {
            tt_p += (double)pos_buf[k] * (double)pos_buf[k];
            st_p += ubuf[k] * (double)pos_buf[k];
        }
        double sim_p;
        if (use_cosine) {
            if (ss <= 0.0 || tt_p <= 0.0) {
                sim_p = 0.0;
                degen_out[0] += 1;
            } else {
                sim_p = st_p / (sqrt(ss) * sqrt(tt_p));
            }
        } else {
            sim_p = st_p;
        }
        for (int j = 0; j < n_neg; ++j) {
            const float *nb = neg_buf + (int64_t)j * K;
            double tt = 0.0, st = 0.0;
            for (int k = 0; k < K; ++k) {
                tt += (double)nb[k] * (double)nb[k];
                st += ubuf[k] * (double)nb[k];
            }
            tts[j] = tt;
            sts[j] = st;
            if (use_cosine) {
                if (ss <= 0.0 || tt <= 0.0) {
                    sims[j] = 0.0;
                    degen_out[0] += 1;
                } else {
                    sims[j] = st / (sqrt(ss) * sqrt(tt));
                }
            } else {
                sims[j] = st;
            }
        }

        /* loss: trainer.py:214-223 */
        double hinge = 0.0;
        for (int j = 0; j < n_neg; ++j) {
            double d = sims[j] - theta;
            if (d > 0.0) {
                hinge += d;
                dnegs[j] = mu * inv_n;
            } else {
                dnegs[j] = 0.0;
            }
            if (dnegs[j] != 0.0) active_out[0] += 1;
        }
        loss_out[0] += (1.0 - sim_p) + mu * inv_n * hinge;
        const double dpos = -1.0;

        /* gradient: trainer.py:230-251 */
        const double rs = ss > 0.0 ? sqrt(ss) : 0.0;
        for (int k = 0; k < K; ++k) ugrad[k] = 0.0;
        if (use_cosine) {
            if (ss > 0.0 && tt_p > 0.0) {
                double denom = ss * rs * sqrt(tt_p);
                for (int k = 0; k < K; ++k)
                    ugrad[k] += dpos * ((double)pos_buf[k] * ss - st_p * ubuf[k]) / denom;
            }
            for (int j = 0; j < n_neg; ++j) {
                if (dnegs[j] != 0.0 && ss > 0.0 && tts[j] > 0.0) {
                    double denom = ss * rs * sqrt(tts[j]);
                    double wj = dnegs[j];
                    const float *nb = neg_buf + (int64_t)j * K;
                    for (int k = 0; k < K; ++k)
                        ugrad[k] += wj * ((double)nb[k] * ss - sts[j] * ubuf[k]) / denom;
                }
            }
        } else {
            for (int k = 0; k < K; ++k) ugrad[k] += dpos * (double)pos_buf[k];
            for (int j = 0; j < n_neg; ++j) {
                if (dnegs[j] != 0.0) {
                    double wj = dnegs[j];
                    const float *nb = neg_buf + (int64_t)j * K;
                    for (int k = 0; k < K; ++k) ugrad[k] += wj * (double)nb[k];
                }
            }
        }

        /* update: trainer.py:259-293 */
        float *tp = T + pos * K;
        if (use_cosine) {
            if (ss > 0.0 && tt_p > 0.0) {
                double denom = tt_p * sqrt(tt_p) * rs;
                for (int k = 0; k < K; ++k) {
                    double g = dpos * (ubuf[k] * tt_p - st_p * (double)pos_buf[k]) / denom;
                    tp[k] = (float)((double)tp[k] - lr * (g + l2 * (double)tp[k]));
                }
            } else if (l2 != 0.0) {
                for (int k = 0; k < K; ++k) tp[k] = (float)((double)tp[k] - lr * l2 * (double)tp[k]);
            }
        } else {
            for (int k = 0; k < K; ++k) {
                double g = dpos * ubuf[k];
                tp[k] = (float)((double)tp[k] - lr * (g + l2 * (double)tp[k]));
            }
        }
        for (int j = 0; j < n_neg; ++j) {
            float *tn = T + (int64_t)neg_ids[j] * K;
            const float *nb = neg_buf + (int64_t)j * K;
            if (dnegs[j] != 0.0) {
                if (use_cosine) {
                    if (ss > 0.0 && tts[j] > 0.0) {
                        double denom = tts[j] * sqrt(tts[j]) * rs;
                        double wj = dnegs[j];
                        for (int k = 0; k < K; ++k) {
                            double g = wj * (ubuf[k] * tts[j] - sts[j] * (double)nb[k]) / denom;
                            tn[k] = (float)((double)tn[k] - lr * (g + l2 * (double)tn[k]));
                        }
                    }
                } else {
                    double wj = dnegs[j];
                    for (int k = 0; k < K; ++k) {
                        double g = wj * ubuf[k];
                        tn[k] = (float)((double)tn[k] - lr * (g + l2 * (double)tn[k]));
                    }
                }
            } else if (l2 != 0.0) {
                for (int k = 0; k < K; ++k) tn[k] = (float)((double)tn[k] - lr * l2 * (double)tn[k]);
            }
        }
        float *su = S + u * K;
        if (!ag->on) {
            for (int k = 0; k < K; ++k)
                su[k] = (float)((double)su[k] - lr * (ugrad[k] + l2 * (double)su[k]));
        } else {
            /* aggregate backward: trainer.py:301-328 */
            const double gamma = ag->gamma;
            for (int k = 0; k < K; ++k)
                su[k] = (float)((double)su[k] - lr * (gamma * ugrad[k] + l2 * (double)su[k]));
            for (int a = 0; a < K; ++a) {
                const double pa = (1.0 - gamma) * pooled[a];
                if (pa != 0.0)
                    for (int b = 0; b < K; ++b) ag->accu[a * K + b] += pa * ugrad[b];
            }
            ag->counter[0] += 1;
            if (ag->counter[0] >= ag->mb_size) {
                const double inv_m = 1.0 / (double)ag->mb_size;
                for (int a = 0; a < K; ++a)
                    for (int b = 0; b < K; ++b) {
                        float *wab = ag->W + a * K + b;
                        *wab = (float)((double)*wab - ag->lr * ag->accu[a * K + b] * inv_m);
                        ag->accu[a * K + b] = 0.0;
                    }
                ag->counter[0] = 0;
            }
            if (ag->hist_prop && hist_len > 0) {
                const double scale = (1.0 - gamma) / (double)hist_len;
                double *wh = s->wh;
                for (int k = 0; k < K; ++k) {
                    double acc = 0.0;
                    for (int b = 0; b < K; ++b) acc += (double)ag->W[k * K + b] * ugrad[b];
                    wh[k] = scale * acc;
                }
                for (int64_t idx = hb; idx < hb + hist_len; ++idx) {
                    float *th = T + (int64_t)ag->tr_items[idx] * K;
                    for (int k = 0; k < K; ++k)
                        th[k] = (float)((double)th[k] - lr * (wh[k] + l2 * (double)th[k]));
                }
            }
        }
    }
}

/* Sequential range [start, stop) on one stream; the single-thread epoch is
 * this over [0, P) with *rng_state = derive_stream(seed, 0x45504F43, epoch, 0)
 * (trainer.py:398-429 with num_threads=1).  last_neg_ids (optional, n_neg
 * entries) receives the final pair's negatives.  Returns 0, or -1 on OOM. */
int ho_train_range(float *S, float *T, int64_t num_items, int K, const int32_t *ep_users,
                   const int32_t *ep_items, int64_t start, int64_t stop, uint64_t *rng_state,
                   int use_cosine, int n_neg, double lr, double l2, double mu, double theta,
                   double *loss_out, int64_t *degen_out, int64_t *active_out,
                   int32_t *last_neg_ids, float *agg_W, const int64_t *tr_offsets,
                   const int32_t *tr_items, double gamma, double agg_lr, int64_t mb_size,
                   int64_t max_history, int hist_prop, double *agg_accu, int64_t *agg_counter) {
    ho_agg ag = {agg_W != NULL, agg_W, tr_offsets, tr_items, gamma, agg_lr, mb_size, max_history,
                 hist_prop, agg_accu, agg_counter};
    ho_scratch s;
    if (scratch_init(&s, K, n_neg)) {
        scratch_free(&s);
        return -1;
    }
    train_chunk(S, T, ep_users, ep_items, start, stop, num_items, rng_state, use_cosine, n_neg, lr,
                l2, mu, theta, &ag, &s, loss_out, degen_out, active_out);
    if (last_neg_ids) memcpy(last_neg_ids, s.neg_ids, sizeof(int32_t) * (size_t)n_neg);
    scratch_free(&s);
    return 0;
}

/* ---- threaded Hogwild epoch: trainer.py:398-447 ------------------------ */
typedef struct {
    float *S, *T;
    const int32_t *ep_users, *ep_items;
    int64_t npairs, chunk, nchunks, num_items;
    int K, n_neg, use_cosine;
    double lr, l2, mu, theta;
    pthread_mutex_t lock;
    int64_t next_chunk;
} ho_epoch_shared;

typedef struct {
    ho_epoch_shared *sh;
    uint64_t rng_state;
    double loss;
    int64_t degen, active;
    int err;
} ho_worker;

static void *worker_main(void *arg) {
    ho_worker *w = (ho_worker *)arg;
    ho_epoch_shared *sh = w->sh;
    ho_scratch s;
    if (scratch_init(&s, sh->K, sh->n_neg)) {
        scratch_free(&s);
        w->err = -1;
        return NULL;
    }
    for (;;) {
        pthread_mutex_lock(&sh->lock);
        int64_t c = sh->next_chunk++;
        pthread_mutex_unlock(&sh->lock);
        if (c >= sh->nchunks) break;
        int64_t start = c * sh->chunk;
        int64_t stop = start + sh->chunk < sh->npairs ? start + sh->chunk : sh->npairs;
        const ho_agg off = {0, NULL, NULL, NULL, 0.0, 0.0, 1, 0, 0, NULL, NULL};
        train_chunk(sh->S, sh->T, sh->ep_users, sh->ep_items, start, stop, sh->num_items,
                    &w->rng_state, sh->use_cosine, sh->n_neg, sh->lr, sh->l2, sh->mu, sh->theta,
                    &off, &s, &w->loss, &w->degen, &w->active);
    }
    scratch_free(&s);
    return NULL;
}

/* One epoch with num_threads workers, per-thread streams
 * derive_stream(seed, 0x45504F43, epoch, tid), dynamic chunk_pairs chunks.
 * Per-thread outputs are reduced in thread order like trainer.py:450-451. */
int ho_train_epoch_threads(float *S, float *T, int64_t num_items, int K, const int32_t *ep_users,
                           const int32_t *ep_items, int64_t npairs, uint64_t seed, int64_t epoch,
                           int num_threads, int64_t chunk_pairs, int use_cosine, int n_neg,
                           double lr, double l2, double mu, double theta, double *loss_out,
                           int64_t *degen_out, int64_t *active_out) {
    if (num_threads < 1 || npairs < 1) return -2;
    ho_epoch_shared sh;
    sh.S = S; sh.T = T; sh.ep_users = ep_users; sh.ep_items = ep_items;
    sh.npairs = npairs;
    sh.chunk = chunk_pairs < npairs ? (chunk_pairs > 0 ? chunk_pairs : 1) : npairs;
    sh.nchunks = (npairs + sh.chunk - 1) / sh.chunk;
    sh.num_items = num_items; sh.K = K; sh.n_neg = n_neg; sh.use_cosine = use_cosine;
    sh.lr = lr; sh.l2 = l2; sh.mu = mu; sh.theta = theta;
    sh.next_chunk = 0;
    pthread_mutex_init(&sh.lock, NULL);
    ho_worker *ws = calloc((size_t)num_threads, sizeof(ho_worker));
    pthread_t *th = calloc((size_t)num_threads, sizeof(pthread_t));
    if (!ws || !th) { free(ws); free(th); return -1; }
    for (int t = 0; t < num_threads; ++t) {
        uint64_t words[3] = {0x45504F43ULL, (uint64_t)epoch, (uint64_t)t};
        ws[t].sh = &sh;
        ws[t].rng_state = ho_derive_stream(seed, words, 3);
    }
    int rc = 0;
    if (num_threads == 1) {
        worker_main(&ws[0]);
    } else {
        for (int t = 0; t < num_threads; ++t) pthread_create(&th[t], NULL, worker_main, &ws[t]);
        for (int t = 0; t < num_threads; ++t) pthread_join(th[t], NULL);
    }
    double loss = 0.0;
    int64_t degen = 0, active = 0;
    for (int t = 0; t < num_threads; ++t) {
        if (ws[t].err) rc = ws[t].err;
        loss += ws[t].loss;
        degen += ws[t].degen;
        active += ws[t].active;
    }
    *loss_out = loss;
    *degen_out = degen;
    *active_out = active;
    pthread_mutex_destroy(&sh.lock);
    free(ws);
    free(th);
    return rc;
}
