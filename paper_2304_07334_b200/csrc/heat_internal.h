// heat_internal.h — launchers shared between the kernel TUs and heat_capi.cu.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/heat_b200.h"

namespace heat {

size_t exact_smem_bytes(int K, int N);

cudaError_t launch_exact(float *S, float *T, const int32_t *users, const int32_t *items,
                         int64_t start, int64_t stop, int K, int N, int cosine, double lr,
                         double l2, double mu, double theta, uint64_t s0, int64_t num_items,
                         heat_counters *ctr, float *snap, const int64_t *pair_index,
                         const heat_agg_params *agg, cudaStream_t stream,
                         unsigned long long *phase = nullptr);

struct HogwildArgs {
    float *S;
    float *T;
    const int32_t *users;
    const int32_t *items;
    int64_t start, stop;
    int K, N, cosine;
    float lr, l2;
    double mu, theta;
    uint64_t s0;
    int64_t num_items;
    heat_counters *ctr;
    int window;
    int fp64;
    int64_t s_rows = 0;  // user table rows (footprint heuristics)
    // delta mode (multi-GPU): item updates logged instead of applied
    int32_t *delta_ids;
    float *delta_rows;
    int64_t *delta_count;
    int64_t delta_capacity;
    // global epoch position of local pair p (RNG key); NULL = p itself
    const int64_t *pair_index;
    // device-side step descriptor (captured step graphs): when set, the kernel
    // trains pairs [range_dev[0], range_dev[1]) with stream base *s0_dev, and
    // start/stop above only size the grid (stop - start = the largest step)
    const int64_t *range_dev = nullptr;
    const uint64_t *s0_dev = nullptr;
    // phase profile (heat_phase_collect): device clock sums, kPhaseWords
    // words; non-NULL selects the phase-instrumented kernel
    unsigned long long *phase = nullptr;
    // behaviour aggregation (throughput mode): the query of local pair p is
    // query[(p - start) * K] instead of S[u]; the user gradient is written to
    // ugrad_out[(p - start) * K] and S[u] -= lr * (ugamma * ugrad + l2 * S[u])
    const float *query = nullptr;
    float *ugrad_out = nullptr;
    float ugamma = 1.f;
    // staged kernel: per-worker overflow area for written rows beyond its
    // shared-memory snapshot (set by the launcher)
    unsigned char *spill = nullptr;
    int64_t spill_stride = 0;  // bytes per worker
    int spill_cap = 0;         // rows per worker
    // register-streamed kernel: the L2 evict-last policy descriptor as a
    // launch parameter (made once on the device, stream_row_policy()), so it
    // lives in the constant bank / a uniform register instead of a vector
    // register pair re-moved to the uniform file before every load
    uint64_t l2_policy = 0;
};

// One rank of the persistent sharded epoch (heat_shard.cu drives it,
// heat_hogwild_stream.cu runs it): the whole epoch in one launch, steps gated
// on the device.  Everything a peer writes (mbox, rel) and reads (the log
// slots) lives in the owner's HBM; peers reach it through the *_tab tables
// (CUDA IPC mappings between processes, plain pointers in a loopback group).
constexpr int kPersistSlots = 8;  // log slots / accumulation buffers (lag <= 7)
constexpr int kPersistMaxWorld = 32;  // one lane per rank in the device checks
// per-step local state words (PersistRank::state, [kStepWords][nsteps])
// (kRows: rows the step touched = its accumulation buffer's slots in use)
// (kWritten: item rows this rank's pairs of the step wrote, owned or logged)
enum StepWord { kDone = 0, kAccClaim, kAccDone, kCvtClaim, kCvtDone, kFin, kRows, kWritten, kStepWords };
// entries (peer phase) / rows (convert phase) per claim of the apply work
constexpr int kApplyChunk = 16;
struct PersistRank {
    float *S, *T;
    const int32_t *users, *items;
    const int64_t *pidx;     // global epoch position of local pair p (RNG key); NULL = p
    const int64_t *bounds;   // [nsteps + 1] local pair bounds of each step
    int64_t nsteps;
    unsigned long long *claim;  // [2]: next local pair, finished warps
    unsigned long long *state;  // [kStepWords * nsteps], zeroed before the launch
    unsigned long long *cnt;    // [nsteps] entries this rank logged per step, zeroed
    int32_t *log_ids[kPersistSlots];  // own log slots (capacity `cap` entries each)
    float *log_rows[kPersistSlots];
    const int32_t *const *pids[kPersistSlots];  // per slot: device table [world] of every rank's ids
    const float *const *prows[kPersistSlots];
    float *const *t_tab;                  // [world]: every rank's T replica (the owner's convert writes them all)
    unsigned long long *const *mbox_tab;  // [world]: every rank's mailbox
    unsigned long long *const *rel_tab;   // [world]: every rank's released words
    // own mailbox [2][mbox_steps][world]: word (tag & 0xffff) << 48 | written
    // << 24 | logged of rank q's step s (24-bit counts)
    const unsigned long long *mbox;
    const unsigned long long *rel;        // own released words [world]
    // per accumulation buffer b = global step % lag (steps in flight never
    // share one): 2^-40 fixed-point sums [t_rows * K], each row's touched flag
    // [t_rows] (`map`), and the list of the step's touched rows [t_rows] (its
    // length is the step's kRows word)
    long long *acc[kPersistSlots];
    int32_t *map[kPersistSlots];
    int32_t *touched[kPersistSlots];
    heat_counters *ctr;
    int64_t *step_counts;  // [nsteps * world]: every rank's count per step (statistics)
    int64_t cap, mbox_steps;
    unsigned long long gbase;  // global step number of this epoch's step 0
    unsigned tag;              // epoch tag (>= 1) of the mailbox words
    int rank, world, lag, nslots, nblocks;  // nblocks: CTAs serving this rank
    int gmod_lag, gmod_slots;               // gbase % lag, gbase % nslots
    int acc_ef;                             // accumulator traffic evict-first (else evict-normal)
};

// Phase profile (trainer.py:120-331 collect_phases; timing.py): words
// [0, 6) clocks per phase in PHASE_NAMES order (read_emb, similarity, loss,
// gradient, update, aggregate), [6] clocks the workers spanned, [7] the
// same spans in globaltimer ns (clock calibration), [8] workers, [9] pairs.
constexpr int kPhaseWords = 10;
unsigned long long *phase_buffer();  // NULL unless heat_phase_collect(1)

cudaError_t launch_hogwild(const HogwildArgs &a, cudaStream_t stream, int *workers_out);
cudaError_t launch_hogwild_resident(const HogwildArgs &a, cudaStream_t stream, int *workers_out);
cudaError_t launch_hogwild_multi(const HogwildArgs &a, cudaStream_t stream, int *workers_out);
cudaError_t launch_hogwild_staged(const HogwildArgs &a, cudaStream_t stream, int *workers_out,
                                  bool bulk);
cudaError_t launch_hogwild_stream(const HogwildArgs &a, cudaStream_t stream, int *workers_out);
bool hogwild_stream_supported(const HogwildArgs &a);
// the persistent sharded epoch: `nctx` ranks in one launch (1 = this process's
// rank; > 1 = a loopback group, launched cooperatively so every rank's CTAs
// are co-resident).  a carries the shared SGD parameters; the per-rank
// pointers come from ctx_dev (device copy of ctx_host).
cudaError_t launch_shard_persist(const HogwildArgs &a, const PersistRank *ctx_host,
                                 PersistRank *ctx_dev, int nctx, cudaStream_t st);
void persist_prof_report();  // HEAT_PERSIST_PROF=1 diagnostics (stderr)
void persist_watchdog_report();  // after a failed persistent epoch (stderr)

size_t agg_hogwild_scratch_bytes(int K, int window);
cudaError_t launch_agg_hogwild(const HogwildArgs &base, const heat_agg_params &agg,
                               void *scratch, cudaStream_t stream);

cudaError_t launch_sample(uint64_t s0, int64_t first_pair, int64_t npairs, int N,
                          int64_t num_items, int32_t *out, cudaStream_t stream);

cudaError_t launch_eval(const void *S, int s_f64, const float *T, int64_t t_rows, int K,
                        const int32_t *users, int64_t n_users, const int64_t *tr_offsets,
                        const int32_t *tr_items, int64_t tr_num_users, const int64_t *te_offsets,
                        const int32_t *te_items, int k, int cosine, const double *dcg_w,
                        const double *idcg, int32_t *topk, double *recall, double *ndcg,
                        cudaStream_t stream);

cudaError_t launch_apply_deltas(float *T, int64_t t_rows, int K, const int32_t *ids,
                                const float *rows, const int64_t *count, int64_t capacity,
                                int ordered, cudaStream_t stream);

cudaError_t launch_apply_deltas_fixed(float *T, int K, const int32_t *ids, const float *rows,
                                      const int64_t *counts, int world, int64_t stride,
                                      long long *acc, int32_t *flags, cudaStream_t st);

cudaError_t launch_aggregate_users(const float *S, const float *T, const float *W,
                                   const int64_t *tr_off, const int32_t *tr_items,
                                   int64_t n_users, int64_t tr_num_users, int K, double gamma,
                                   int64_t max_history, double *out, cudaStream_t st);

bool exact_spec_supported(int K, int N);
void exact_spec_stats(unsigned long long *out, bool reset);
size_t exact_spec_scratch_bytes(int K, int N, int64_t s_rows, int64_t t_rows);
cudaError_t launch_exact_spec(float *S, int64_t s_rows, float *T, int64_t t_rows,
                              const int32_t *users, const int32_t *items, int64_t start,
                              int64_t stop, int K, int N, int cosine, double lr, double l2,
                              double mu, double theta, uint64_t s0, heat_counters *ctr,
                              void *scratch, const int64_t *pair_index, cudaStream_t stream);

// one DELTA step whose pair range / stream base live in device memory (the
// shard runtime's captured step graphs); device_step_supported says whether a
// kernel family with that mode serves these parameters
int train_range_device_step(float *S, int64_t s_rows, float *T, int64_t t_rows,
                            const int32_t *users, const int32_t *items,
                            const heat_sgd_params *p, heat_counters *counters, int32_t *delta_ids,
                            float *delta_rows, int64_t *delta_count, int64_t delta_capacity,
                            const int64_t *pair_index, const int64_t *range_dev,
                            const uint64_t *s0_dev, void *stream);
bool device_step_supported(const heat_sgd_params *p, const float *S, const float *T);

int sm_count();
// CTAs per SM of a kernel (dynamic smem opt-in applied), cached per device
int kernel_occupancy(const void *kern, int threads, size_t smem, cudaError_t *err);
// library-owned scratch per (purpose, device, stream); nullptr if out of memory
void *stream_scratch(int purpose, size_t bytes, cudaStream_t stream);
size_t eval_max_k_supported(int K);

}  // namespace heat
