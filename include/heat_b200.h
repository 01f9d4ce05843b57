/*
 * heat_b200.h — C ABI of the B200 SimpleX-MF-CCL training path.
 *
 * Plain pointers and sizes only (no torch types).  All table / index
 * pointers are DEVICE pointers owned by the caller; `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  Every entry
 * point validates its arguments on the host, launches asynchronously on
 * `stream`, and returns a status code; heat_last_error() returns the
 * message of the last failure on the calling thread.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/heatcf):
 *   heat_train_range       <- trainer._train_chunk           trainer.py:103-331
 *                             (uniform sampler, no aggregator; cosine or dot)
 *                             driven per epoch by train_epoch trainer.py:385-466
 *   heat_sample_negatives  <- rng_below loop of _train_chunk trainer.py:135-139,
 *                             rng.rng_next / rng_below     rng.py:63-76
 *   heat_eval_users        <- evaluator.evaluate scoring + top-k + hits
 *                             evaluator.py:140-172, _topk_from_scores 61-73
 *   heat_apply_row_deltas  <- (new) multi-GPU item-delta exchange, SURVEY.md §8(e)
 *   heat_apply_row_deltas_fixed <- (new) same, order-independent (pipelined exchange)
 *   heat_shard_*           <- (new) per-rank step scheduler of the sharded epoch;
 *                             the reference's thread pool  trainer.py:398-447
 *   heat_epoch_pairs       <- dataset.epoch_pairs (host)    dataset.py:146-158
 *   heat_aggregate_users   <- evaluator._aggregated_user_vectors evaluator.py:91-110
 *   heat_train_range(agg)  <- _train_chunk agg_on branch     trainer.py:148-173, 299-331
 *   heat_phase_collect/_read <- collect_phases cycle counters trainer.py:120-331, 452-457;
 *                             timing.py:20-53
 *   heat_agg_scratch_bytes <- _ThreadState agg buffers      trainer.py:334-363
 */
#ifndef HEAT_B200_H
#define HEAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEAT_OK 0
#define HEAT_ERR_INVALID 1     /* bad argument (reference raises ValueError) */
#define HEAT_ERR_CUDA 2        /* CUDA runtime error (reference: RuntimeError) */
#define HEAT_ERR_UNSUPPORTED 3 /* option outside the built path (ValueError) */

/* Execution modes of heat_train_range. */
#define HEAT_MODE_EXACT 0   /* pairs strictly in order; bit-identical to the
                               reference with num_threads=1 */
#define HEAT_MODE_HOGWILD 1 /* up to `window` pairs in flight, lock-free
                               atomic row updates (reference num_threads>1) */
#define HEAT_MODE_DELTA 2   /* hogwild reads, but item-row updates are logged
                               to a delta buffer instead of applied (the
                               multi-GPU step; users still updated in place) */

typedef struct heat_sgd_params {
    int32_t dim;          /* K: columns of S and T                          */
    int32_t n_neg;        /* N: negatives per pair                          */
    int32_t use_cosine;   /* 1: cosine similarity, 0: dot                   */
    int32_t mode;         /* HEAT_MODE_*                                    */
    double lr;            /* learning_rate                                  */
    double l2;            /* l2_reg                                         */
    double mu;            /* loss.mu (negative weight)                      */
    double theta;         /* loss.theta (margin)                            */
    uint64_t stream_base; /* s0 = derive_stream(seed, 0x45504F43, epoch, 0);
                             negative j of the pair at epoch position p is
                             draw p*N+j of this stream                      */
    int32_t window;       /* HOGWILD/DELTA: max pairs in flight (step size B);
                             <=0 means "as many as the GPU holds"           */
    int32_t flags;        /* bit0: fp64 dot products in HOGWILD (default fp32
                             partials + fp64 combine when 0)               */
} heat_sgd_params;

/* SimpleX behaviour aggregation (aggregator.py:30-113; trainer.py:148-173,
 * 299-331): the query is h = gamma*S[u] + (1-gamma)*mean(history rows)*W.
 * Device pointers; `accu`/`counter` are the per-epoch accumulator state
 * (zero them at the start of every epoch, as trainer.py:348-349 does). */
typedef struct heat_agg_params {
    float *W;                  /* K x K float32, input-major W[k*K+j]; updated */
    const int64_t *tr_offsets; /* train CSR: a user's history is its first   */
    const int32_t *tr_items;   /* max_history items (trainer.py:151-155)      */
    double gamma;              /* aggregator.gamma                            */
    double lr;                 /* aggregator.learning_rate or the embedding lr */
    int64_t mini_batch;        /* accumulator flush period (pairs)            */
    int64_t max_history;
    int32_t history_grad;      /* propagate into the history item rows        */
    int32_t reserved;
    double *accu;              /* K x K binary64 weight-gradient accumulator  */
    int64_t *counter;          /* pairs since the last flush                  */
} heat_agg_params;

/* Device-resident accumulators (caller zeroes them; kernels add). */
typedef struct heat_counters {
    double loss;        /* running sum of per-pair losses (trainer.py:222)  */
    int64_t degenerate; /* zero-norm similarity hits (trainer.py:187,203)   */
    int64_t active;     /* negatives with nonzero loss gradient             */
    int64_t pairs;      /* pairs processed                                  */
} heat_counters;

/* Train pairs [start, stop) of an epoch's (ep_users, ep_items) order.
 * S: s_rows x dim float32 row-major; T: t_rows x dim; negatives are uniform
 * over [0, t_rows) exactly like trainer.py:136 (num_items = T.rows).
 * `counters` is a device pointer.  For HEAT_MODE_DELTA, `delta_ids`
 * (int32, capacity entries) and `delta_rows` (capacity x dim float32) receive
 * the item-row updates and `delta_count` (device int64) their number.
 * `pair_index` (optional, int64 per pair) is the pair's global epoch position,
 * the key of its negative draws (a user shard trains a subset of the epoch
 * and must draw the 1-GPU run's negatives); NULL means position p itself.
 * `agg` (optional) turns on behaviour aggregation.  HEAT_MODE_EXACT follows
 * the reference's single thread bit for bit (accu/counter carry the flush
 * state).  HEAT_MODE_HOGWILD runs steps of `window` pairs (4096 when <= 0)
 * with W frozen inside a step; every pair's (agg_lr/mini_batch) * pooled (x)
 * ugrad reaches W on the reference's flush schedule: when the pair's
 * mini-batch (epoch position / mini_batch) completes, the incomplete one
 * waiting in `accu` (counter unused; with accu NULL every pair goes straight
 * to W after its step); `scratch` is then
 * NULL or at least heat_agg_scratch_bytes(dim, window) bytes.  DELTA mode
 * returns HEAT_ERR_UNSUPPORTED.
 * Scratch (HEAT_MODE_EXACT): `scratch` may be NULL (internal allocation) or a
 * device buffer of at least heat_scratch_bytes(n_neg, dim, s_rows, t_rows)
 * bytes (active-row snapshots and the per-row commit stamps of the parallel
 * deterministic kernel). */
int heat_train_range(float *S, int64_t s_rows, float *T, int64_t t_rows,
                     const int32_t *ep_users, const int32_t *ep_items, int64_t start,
                     int64_t stop, const heat_sgd_params *params, heat_counters *counters,
                     int32_t *delta_ids, float *delta_rows, int64_t *delta_count,
                     int64_t delta_capacity, const int64_t *pair_index,
                     const heat_agg_params *agg, void *scratch, void *stream);

int64_t heat_scratch_bytes(int32_t n_neg, int32_t dim, int64_t s_rows, int64_t t_rows);

/* Scratch of HEAT_MODE_HOGWILD with aggregation (per-step pooled histories,
 * queries and user gradients). */
int64_t heat_agg_scratch_bytes(int32_t dim, int32_t window);

/* out[(p - first_pair) * n_neg + j] = negative j of pair p, for
 * p in [first_pair, first_pair + npairs): the id trainer.py:136 draws. */
int heat_sample_negatives(uint64_t stream_base, int64_t first_pair, int64_t npairs,
                          int32_t n_neg, int64_t num_items, int32_t *out, void *stream);

/* Recall/NDCG parts for a list of users (device arrays).
 * S holds the query rows, float32 (s_f64 = 0) or float64 (s_f64 = 1).
 * users[n_users]; train CSR (tr_offsets[tr_num_users+1], tr_items) masks
 * positives; test CSR (te_offsets, te_items; sorted slices) gives hits.
 * dcg_weights[k] = 1/log2(r+1), idcg[k] = prefix sums, both computed by the
 * caller in the reference's arithmetic (evaluator.py:144-148).
 * Outputs per user: recall (hits / n_test), ndcg (dcg / idcg[min(k,n)-1]);
 * topk (n_users x k, -1 padded) may be NULL.  similarity: 1 cosine, 0 dot. */
int heat_eval_users(const void *S, int32_t s_f64, const float *T, int64_t t_rows, int32_t dim,
                    const int32_t *users, int64_t n_users, const int64_t *tr_offsets,
                    const int32_t *tr_items, int64_t tr_num_users, const int64_t *te_offsets,
                    const int32_t *te_items, int32_t k, int32_t use_cosine,
                    const double *dcg_weights, const double *idcg, int32_t *topk,
                    double *recall, double *ndcg, void *stream);

/* out[u] = gamma*S[u] + (1-gamma) * mean(first max_history train items of u).W
 * for u < s_rows (binary64 rows, the aggregated evaluation query,
 * evaluator.py:91-110); users without history get gamma*S[u]. */
int heat_aggregate_users(const float *S, int64_t s_rows, const float *T, const float *W,
                         int32_t dim, const int64_t *tr_offsets, const int32_t *tr_items,
                         int64_t tr_num_users, double gamma, int64_t max_history, double *out,
                         void *stream);

/* T[ids[i]] += rows[i] for i < *count (device count), in index order per row
 * when `ordered` != 0 (deterministic replica update), atomically otherwise. */
int heat_apply_row_deltas(float *T, int64_t t_rows, int32_t dim, const int32_t *ids,
                          const float *rows, const int64_t *count, int64_t capacity,
                          int32_t ordered, void *stream);

/* Order-independent variant for the pipelined exchange: the all-gathered logs
 * of `world` ranks (rank r's entries at [r*stride, r*stride + counts[r]),
 * counts a device array) are summed per (row, column) in 2^-40 fixed point
 * with integer atomics, then each touched row gets T += float(sum) once; the
 * result does not depend on atomic ordering, so replicas stay bit-identical
 * without sorting.  acc (t_rows*dim int64) and flags (t_rows int32) are
 * caller-owned, zero before the first call, and left zero. */
int heat_apply_row_deltas_fixed(float *T, int64_t t_rows, int32_t dim, const int32_t *ids,
                                const float *rows, const int64_t *counts, int32_t world,
                                int64_t stride, int64_t *acc, int32_t *flags, void *stream);

/* ---- multi-GPU runtime --------------------------------
 * One rank per GPU.  For dim 128 (HEAT_SHARD_PERSIST=1, the default) an
 * epoch is ONE persistent kernel launch: steps are gated on the device (a
 * pair of global step g starts once this rank applied step g - lag and every
 * peer step g - lag - 1; lag 3, HEAT_SHARD_LAG 1..7), the workers add their
 * own item deltas into per-step fixed-point buffers and log them for the
 * peers, publish each finished step's entry count into every rank's mailbox
 * (IPC-mapped; st.release.sys), and between pairs pull the peers' logs and
 * convert the touched rows; each rank publishes its applied-step count the
 * same way.  Otherwise (dim 64, HEAT_SHARD_PERSIST=0, or the gather
 * exchange) the stream-ordered steps below run.
 * A heat_shard owns the rank's exchange state: rotating
 * log slots, the fixed-point accumulator, two compute streams, a
 * top-priority comm stream and (world > 1) an NCCL communicator created from
 * a unique id that rank 0 makes with heat_nccl_unique_id and the caller
 * broadcasts (e.g. torch.distributed).  heat_shard_epoch trains the rank's
 * pairs of one epoch: step s covers local pairs [step_bounds[s],
 * step_bounds[s+1]) (host array), DELTA-mode kernel on a compute stream;
 * then, on the comm stream, an NCCL all-gather of the step's 8-byte entry
 * counts (also the cross-rank fence) and the fused gather+apply kernels,
 * which read every rank's log straight from its memory over NVLink (CUDA IPC
 * mappings; HEAT_SHARD_EXCHANGE=gather selects an NCCL all-gather of the logs
 * instead) and add them in order-free fixed point.  Kernel(s) waits for the
 * apply of step s - lag (lag 3; HEAT_SHARD_LAG 1..3).  No host wait inside
 * the epoch; it returns once the epoch is done, with `stream` ordered after
 * it.  Every rank must pass the same nsteps; capacity is agreed (max). */
typedef struct heat_shard heat_shard;

typedef struct heat_shard_stats {
    int64_t steps;           /* exchanges performed                           */
    int64_t entries;         /* delta rows applied (sum over ranks and steps) */
    int64_t exchanged_bytes; /* bytes each rank read from its peers' logs     */
    int64_t max_entries;     /* largest per-rank log of a step                */
    int64_t launches;        /* kernel launches of the epoch (1: persistent)  */
} heat_shard_stats;

int heat_nccl_unique_id(unsigned char *out128);
int heat_shard_create(int32_t world, int32_t rank, const unsigned char *nccl_id, int32_t device,
                      heat_shard **out);
int heat_shard_epoch(heat_shard *h, float *S, int64_t s_rows, float *T, int64_t t_rows,
                     const int32_t *local_users, const int32_t *local_items,
                     const int64_t *pair_index, const int64_t *step_bounds, int64_t nsteps,
                     int64_t capacity, const heat_sgd_params *params, heat_counters *counters,
                     heat_shard_stats *stats, void *stream);
const char *heat_shard_last_error(heat_shard *h);
int heat_shard_destroy(heat_shard *h);

/* Host transport: the per-process runtime with its collectives carried by a
 * caller-supplied host all-gather instead of NCCL, for `world` PROCESSES that
 * share one GPU (NCCL refuses two ranks on a device).  `allgather(user, in,
 * nbytes, out)` gathers nbytes from every rank into out (world * nbytes, rank
 * order) and returns 0; every rank calls it in the same order.  The entry-
 * count exchange of each step becomes that call between two synchronisations
 * of the comm stream (the same cross-rank fence, with the host in the loop);
 * the peers' logs are read through CUDA IPC mappings by the same fused
 * gather+apply kernels as over NVLink (or, with HEAT_SHARD_EXCHANGE=gather,
 * all-gathered through host memory).  Stream-ordered steps only: the
 * persistent epoch and captured graphs are off, so no kernel of one process
 * ever waits on a kernel of another.  A test and bring-up path (it covers
 * the IPC mapping, the fence ordering and replica identity of the
 * multi-process runtime on a one-GPU box), not a fast one. */
typedef int (*heat_host_allgather_fn)(void *user, const void *in, int64_t nbytes, void *out);
int heat_shard_create_host(int32_t world, int32_t rank, heat_host_allgather_fn allgather,
                           void *user, int32_t device, heat_shard **out);

/* Loopback group: `world` ranks in ONE process on one device, for testing
 * the runtime's multi-rank step logic where only one GPU exists (no NCCL,
 * no CUDA IPC).  The collectives become stream-ordered copies into a shared
 * count row plus event waits: a rank's count "collective" of step s completes
 * once every rank's comm stream has finished its apply of step s-1 and seen
 * its own step-s log — the ordering the NCCL all-gather gives between
 * processes.  Peers' logs are read through plain device pointers by the same
 * fused gather+apply kernels (or, with HEAT_SHARD_EXCHANGE=gather, copied
 * into the gathered buffer).  Nothing spins: every cross-rank dependency is
 * an event wait, so the ranks' kernels never wait on one another.
 * heat_shard_epoch_loopback runs one epoch of every rank (same nsteps; each
 * rank its own S/T replica, pairs, bounds and counters), interleaving their
 * steps; stats is an array of `world`.  Handles from heat_shard_create_loopback
 * are destroyed one by one with heat_shard_destroy. */
typedef struct heat_shard_rank {
    float *S;
    int64_t s_rows;
    float *T;
    int64_t t_rows;
    const int32_t *local_users;
    const int32_t *local_items;
    const int64_t *pair_index;
    const int64_t *step_bounds; /* host, nsteps + 1 */
    int64_t capacity;
    heat_counters *counters;
} heat_shard_rank;

int heat_shard_create_loopback(int32_t world, int32_t device, heat_shard **out);
int heat_shard_epoch_loopback(heat_shard **ranks_h, int32_t world, const heat_shard_rank *ranks,
                              int64_t nsteps, const heat_sgd_params *params,
                              heat_shard_stats *stats, void *stream);

/* HOST function: one epoch's (user, positive) order, bit-identical to
 * numpy Generator(PCG64(seed)).permutation applied to the CSR pairs
 * (dataset.py:146-158).  offsets/items/out_* are host arrays; the PCG64 state
 * words are numpy's after its own seeding (bit_generator.state).  Returns 0,
 * or -1 on bad input. */
int heat_epoch_pairs(const int64_t *offsets, int64_t num_users, const int32_t *items, int64_t P,
                     uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int32_t has_uint32, uint32_t uinteger, int32_t *out_users,
                     int32_t *out_items);

/* Phase profile: the per-phase times of trainer.py's collect_phases
 * (trainer.py:120-331 cycle counters, timing.py:20-53; PHASE_NAMES order
 * read_emb, similarity, loss, gradient, update, aggregate).  While on
 * (heat_phase_collect(1)), heat_train_range runs phase-instrumented kernels
 * on the current device: EXACT the serial kernel (same bits; its phases are
 * the reference's, one pair at a time), HOGWILD at dim 64/128 (cosine,
 * fp32) the register-streamed kernel, whose fused phases are split by where
 * the time goes.  Other launches add nothing.
 * heat_phase_read returns seconds per phase averaged over the workers (one
 * worker = one warp / one CTA, as the reference averages its threads),
 * converted from clock64 with the workers' own clock/globaltimer ratio, plus
 * the worker and pair counts; reset != 0 zeroes the sums. */
int heat_phase_collect(int32_t on);
int heat_phase_read(double *seconds6, int64_t *workers, int64_t *pairs, int32_t reset);

/* Diagnostics of the parallel deterministic (EXACT) kernel: out[0..2] clock64
 * totals of speculate / commit-token wait / commit, out[3..5] partial
 * recomputes, full recomputes, pairs.  reset != 0 zeroes them. */
int heat_exact_stats(unsigned long long *out, int reset);

/* Diagnostic: streaming read of n floats (device buffer) `passes` times at
 * L2 on `stream`; bench.py times it to measure the L2 read ceiling that
 * bounds the L2-resident configurations (not a reference interface). */
int heat_probe_l2_read(const float *buf, int64_t n, int32_t passes, float *sink, void *stream);
/* Diagnostic: random-row gathers over a rows x dim table (dim 64 or 128) in
 * the training kernels' access pattern, no arithmetic; *rows_read = rows
 * gathered.  bench.py times it for the L2 roofline of gather-bound kernels. */
int heat_probe_l2_gather(const float *table, int64_t rows, int32_t dim, int32_t iters,
                         float *sink, int64_t *rows_read, void *stream);

const char *heat_last_error(void);
int heat_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HEAT_B200_H */
