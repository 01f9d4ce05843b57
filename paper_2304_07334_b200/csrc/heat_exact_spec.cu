// heat_exact_spec.cu — deterministic SGD with speculative parallelism.
//
// Same result, bit for bit, as heat_exact.cu and as the reference with
// num_threads=1 (trainer.py:114-293): pairs are COMMITTED strictly in epoch
// order, and every committed pair is computed from exactly the tables the
// sequential run would show it.  The parallelism comes from speculation:
//
//   * one CTA of NW warps; warp w owns pairs start+w, start+w+NW, ...;
//   * SPECULATE (no ordering): the warp reads the committed-prefix counter c,
//     the user row, the positive and its N negative rows, and computes ss,
//     tt_j, st_j, sim_j, the ordered active list, the hinge and the pair loss
//     in the reference's binary64 order (lane-per-row, sequential k).  It
//     then builds the pair's write list (T[pos], active T[neg_j] in j order,
//     S[u]), reads the snapshot of each written row, and evaluates the whole
//     update phase of trainer.py:229-293 lane-per-column into shared memory —
//     a row that appears twice in the write list takes its second update on
//     top of its first, as the reference's in-place writes do;
//   * COMMIT (in order, token in shared memory): the warp checks the
//     last-writer stamps of every row it read.  A stamp >= c means a pair
//     committed after the warp started reading wrote that row -> speculate
//     again (every earlier pair is committed, so the result is final).  Then
//     the precomputed rows are stored, stamped, the running loss is added in
//     pair order and the token passes — no global load on the commit path.
// Stamps: int16 relative pair indices in shared memory when the tables are
// small enough (launches are split so a launch never exceeds 32767 pairs),
// otherwise int32 in a global array reset per launch.  Writes that do not fit
// the precompute buffers (many active negatives, or l2 != 0 which rewrites
// every sampled row) take a commit-time path that reads the rows after the
// token arrives.  Ordering: committers store rows and stamps,
// __threadfence_block(), publish the token; speculators read the token,
// fence, then read rows, so a concurrently written row is always caught.
#include <cstdint>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

#define DMUL __dmul_rn
#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DDIV __ddiv_rn
#define DSQRT __dsqrt_rn

constexpr int kSpecWarps = 16;     // most warps per CTA (fewer when the rows are wide)
constexpr int kSpecMaxRows = 1024; // N+1 <= 1024: a lane's row mask is one 32-bit word
constexpr int kSpecMaxK = 256;
constexpr int kSpecChunk = 32767;  // pairs per launch (int16 stamps never wrap)

struct SpecWarp {  // per-warp shared state between speculate and commit
    double ss, sim_p, tt_p, st_p, pair_loss;
    int64_t u, pos, c0;
    int n_act;  // negatives with d > 0 (ordered in act[])
    int n_w;    // T rows in the precomputed write list (pos + updates), -1 = commit-time path
    int degen;
};

struct SpecLayout {
    int wcap;  // precomputed T-row writes per warp
    int smem_stamps;
    int warps;
    size_t off_sw, off_ubuf, off_tts, off_sts, off_sims, off_nids, off_act, off_wid, off_new,
        off_stamps, total;
};

__host__ __device__ inline SpecLayout spec_layout(int K, int N, int64_t rows_total, int wcap,
                                                  bool smem_stamps, int warps = kSpecWarps) {
    SpecLayout L;
    L.wcap = wcap;
    L.smem_stamps = smem_stamps ? 1 : 0;
    L.warps = warps;
    size_t o = 32;  // token, running loss
    auto take = [&](size_t b) {
        size_t at = (o + 15) & ~size_t(15);
        o = at + b;
        return at;
    };
    const size_t W = (size_t)warps;
    L.off_sw = take(sizeof(SpecWarp) * W);
    L.off_ubuf = take(8 * W * K);
    L.off_tts = take(8 * W * N);
    L.off_sts = take(8 * W * N);
    L.off_sims = take(8 * W * N);
    L.off_nids = take(4 * W * N);
    L.off_act = take(4 * W * N);
    L.off_wid = take(4 * W * wcap);
    L.off_new = take(4 * W * (wcap + 1) * K);  // wcap T rows + the S row
    L.off_stamps = smem_stamps ? take(2 * (size_t)rows_total) : 0;
    L.total = (o + 127) & ~size_t(127);
    return L;
}

// diagnostics: clock64 totals over all warps of the last launches
// [0] speculate, [1] token wait, [2] commit, [3] partial recomputes,
// [4] full recomputes, [5] pairs
__device__ unsigned long long g_spec_stats[8];

__device__ __forceinline__ int64_t ld_volatile(const int64_t *p) {
    return *reinterpret_cast<const volatile int64_t *>(p);
}

__global__ void __launch_bounds__(32 * kSpecWarps, 1)
    exact_spec_kernel(float *__restrict__ S, float *__restrict__ T,
                      const int32_t *__restrict__ users, const int32_t *__restrict__ items,
                      int64_t start, int64_t stop, int K, int N, int cosine, double lr, double l2,
                      double mu, double theta, uint64_t s0, FastMod fm, heat_counters *ctr,
                      float *__restrict__ snap_all, int32_t *__restrict__ gstamps,
                      int64_t t_rows, int64_t s_rows, const int64_t *__restrict__ pair_index,
                      SpecLayout Lo) {
    extern __shared__ __align__(16) unsigned char smem[];
    int64_t *token = reinterpret_cast<int64_t *>(smem);     // next pair to commit
    double *loss_run = reinterpret_cast<double *>(smem + 8);
    int64_t *visible = reinterpret_cast<int64_t *>(smem + 16);  // pairs whose row stores
                                                                 // are fenced (prefix)
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    SpecWarp &sw = reinterpret_cast<SpecWarp *>(smem + Lo.off_sw)[w];
    double *ubuf = reinterpret_cast<double *>(smem + Lo.off_ubuf) + w * K;
    double *tts = reinterpret_cast<double *>(smem + Lo.off_tts) + w * N;
    double *sts = reinterpret_cast<double *>(smem + Lo.off_sts) + w * N;
    double *sims = reinterpret_cast<double *>(smem + Lo.off_sims) + w * N;
    int32_t *nids = reinterpret_cast<int32_t *>(smem + Lo.off_nids) + w * N;
    int32_t *act = reinterpret_cast<int32_t *>(smem + Lo.off_act) + w * N;
    const int wcap = Lo.wcap;
    int32_t *wid = reinterpret_cast<int32_t *>(smem + Lo.off_wid) + w * wcap;
    float *newv = reinterpret_cast<float *>(smem + Lo.off_new) + (size_t)w * (wcap + 1) * K;
    float *snew = newv + (size_t)wcap * K;  // the new S row
    int16_t *sstamps = reinterpret_cast<int16_t *>(smem + Lo.off_stamps);
    float *snap = snap_all + (size_t)w * N * K;  // commit-path snapshots (global scratch)

    // stamps: T rows then S rows, relative pair index of the last writer
    auto stamp_ld = [&](int64_t row) -> int {
        return Lo.smem_stamps ? (int)*reinterpret_cast<volatile int16_t *>(sstamps + row)
                              : *reinterpret_cast<volatile int32_t *>(gstamps + row);
    };
    auto stamp_st = [&](int64_t row, int v) {
        if (Lo.smem_stamps)
            *reinterpret_cast<volatile int16_t *>(sstamps + row) = (int16_t)v;
        else
            *reinterpret_cast<volatile int32_t *>(gstamps + row) = v;
    };

    if (threadIdx.x == 0) {
        *token = start;
        *visible = start;
        *loss_run = ctr->loss;
    }
    if (Lo.smem_stamps)
        for (int64_t i = threadIdx.x; i < t_rows + s_rows; i += blockDim.x) sstamps[i] = -1;
    __syncthreads();

    const double inv_n = DDIV(1.0, (double)N);
    const double dneg_w = DMUL(mu, inv_n);
    const double dpos = -1.0;
    long long degen_total = 0, active_total = 0;

    // ---- speculate pair p from the tables as they are now
    // full: read the pair from scratch.  Otherwise (at commit, user row still
    // valid) only the rows flagged in this lane's `smask` (bit i = row
    // lane + 32 i) are re-read; the dot products of the others are pure
    // functions of (user row, item row) and are kept.
    auto speculate = [&](int64_t p, unsigned smask, bool full) {
        const int64_t c0 = ld_volatile(visible);  // rows of pairs < c0 are visible
        __threadfence_block();
        int64_t u, pos;
        double ss = 0.0;
        if (full) {
            u = users[p];
            pos = items[p];
            const int64_t pg = pair_index ? pair_index[p] : p;
            for (int k = lane; k < K; k += 32) ubuf[k] = (double)S[u * K + k];
            for (int j = lane; j < N; j += 32) nids[j] = neg_id(s0, pg, N, j, fm);
            __syncwarp();
            // ss by the last lane (fewest rows) while the lanes score rows r = lane + 32 i
            if (lane == 31)
                for (int k = 0; k < K; ++k) ss = DADD(ss, DMUL(ubuf[k], ubuf[k]));
        } else {
            u = sw.u;
            pos = sw.pos;
            ss = sw.ss;
        }
        double tt_p = full ? 0.0 : sw.tt_p, st_p = full ? 0.0 : sw.st_p;
        for (int r = lane, i = 0; r <= N; r += 32, ++i) {
            if (!full && !((smask >> i) & 1u)) continue;
            const float *row = T + (r == 0 ? pos : (int64_t)nids[r - 1]) * K;
            double a, b;
            row_dots_any(row, ubuf, K, a, b);
            if (r == 0) {
                tt_p = a;
                st_p = b;
            } else {
                tts[r - 1] = a;
                sts[r - 1] = b;
            }
        }
        if (full) ss = __shfl_sync(0xffffffffu, ss, 31);
        tt_p = __shfl_sync(0xffffffffu, tt_p, 0);
        st_p = __shfl_sync(0xffffffffu, st_p, 0);
        __syncwarp();
        int degen = 0;
        double sim_p = st_p;
        if (cosine) {
            if (ss <= 0.0 || tt_p <= 0.0) {
                sim_p = 0.0;
                degen = lane == 0 ? 1 : 0;
            } else {
                sim_p = DDIV(st_p, DMUL(DSQRT(ss), DSQRT(tt_p)));
            }
        }
        // sims + ordered active list (j ascending)
        int n_act = 0;
        for (int j0 = 0; j0 < N; j0 += 32) {
            const int j = j0 + lane;
            bool a = false;
            if (j < N) {
                double sim = sts[j];
                if (cosine) {
                    if (ss <= 0.0 || tts[j] <= 0.0) {
                        sim = 0.0;
                        ++degen;
                    } else {
                        sim = DDIV(sts[j], DMUL(DSQRT(ss), DSQRT(tts[j])));
                    }
                }
                sims[j] = sim;
                a = DSUB(sim, theta) > 0.0;
            }
            const unsigned m = __ballot_sync(0xffffffffu, a);
            if (a) act[n_act + __popc(m & ((1u << lane) - 1u))] = j;
            n_act += __popc(m);
        }
        __syncwarp();
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) degen += __shfl_xor_sync(0xffffffffu, degen, o);
        const int n_upd = dneg_w != 0.0 ? n_act : 0;
        // ---- precompute the update phase (trainer.py:229-293) when it fits
        int n_w = -1;
        if (l2 == 0.0 && 1 + n_upd <= wcap) {
            n_w = 1 + n_upd;
            if (lane == 0) wid[0] = (int32_t)pos;
            for (int a = lane; a < n_upd; a += 32) wid[1 + a] = nids[act[a]];
            __syncwarp();
            const double rs = ss > 0.0 ? DSQRT(ss) : 0.0;
            for (int k = lane; k < K; k += 32) {
                const double ub = ubuf[k];
                const double pk = (double)T[pos * K + k];  // snapshot = speculated state
                double ug = 0.0;
                if (cosine) {
                    if (ss > 0.0 && tt_p > 0.0) {
                        const double denom = DMUL(DMUL(ss, rs), DSQRT(tt_p));
                        ug = DADD(ug, DDIV(DMUL(dpos, DSUB(DMUL(pk, ss), DMUL(st_p, ub))), denom));
                    }
                } else {
                    ug = DADD(ug, DMUL(dpos, pk));
                }
                {  // new T[pos] (l2 == 0 on this path)
                    double g = 0.0;
                    bool wr = true;
                    if (cosine) {
                        if (ss > 0.0 && tt_p > 0.0) {
                            const double denom = DMUL(DMUL(tt_p, DSQRT(tt_p)), rs);
                            g = DDIV(DMUL(dpos, DSUB(DMUL(ub, tt_p), DMUL(st_p, pk))), denom);
                        } else {
                            wr = false;
                        }
                    } else {
                        g = DMUL(dpos, ub);
                    }
                    newv[k] = wr ? __double2float_rn(DSUB(pk, DMUL(lr, DADD(g, DMUL(l2, pk)))))
                                 : (float)pk;
                }
                // active negatives in j order; a repeated id continues from the
                // newest value written for it earlier in this pair
                for (int a = 0; a < n_upd; ++a) {
                    const int j = act[a];
                    const int32_t id = wid[1 + a];
                    const float vsf = T[(int64_t)id * K + k];  // snapshot
                    const double vs = (double)vsf;
                    float cur = vsf;
                    for (int b = a; b >= 0; --b) {
                        if (wid[b] == id) {
                            cur = newv[(size_t)b * K + k];
                            break;
                        }
                    }
                    const double tj = tts[j];
                    double g = 0.0;
                    bool wr = true;
                    if (cosine) {
                        if (ss > 0.0 && tj > 0.0) {
                            const double denom = DMUL(DMUL(ss, rs), DSQRT(tj));
                            ug = DADD(ug, DDIV(DMUL(dneg_w, DSUB(DMUL(vs, ss), DMUL(sts[j], ub))),
                                               denom));
                            const double denom2 = DMUL(DMUL(tj, DSQRT(tj)), rs);
                            g = DDIV(DMUL(dneg_w, DSUB(DMUL(ub, tj), DMUL(sts[j], vs))), denom2);
                        } else {
                            wr = false;
                        }
                    } else {
                        ug = DADD(ug, DMUL(dneg_w, vs));
                        g = DMUL(dneg_w, ub);
                    }
                    const double t = (double)cur;
                    newv[(size_t)(1 + a) * K + k] =
                        wr ? __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t))))) : cur;
                }
                const double s = ubuf[k];  // S[u] snapshot
                snew[k] = __double2float_rn(DSUB(s, DMUL(lr, DADD(ug, DMUL(l2, s)))));
            }
        }
        if (lane == 0) {
            double hinge = 0.0;
            for (int a = 0; a < n_act; ++a) hinge = DADD(hinge, DSUB(sims[act[a]], theta));
            sw.pair_loss = DADD(DSUB(1.0, sim_p), DMUL(dneg_w, hinge));
            sw.ss = ss;
            sw.sim_p = sim_p;
            sw.tt_p = tt_p;
            sw.st_p = st_p;
            sw.u = u;
            sw.pos = pos;
            sw.c0 = c0;
            sw.n_act = n_act;
            sw.n_w = n_w;
            sw.degen = degen;
        }
        __syncwarp();
    };

    // ---- commit-time update phase (overflow / l2 != 0): reads the current rows
    auto update_in_place = [&]() {
        const int64_t u = sw.u, pos = sw.pos;
        const double ss = sw.ss, tt_p = sw.tt_p, st_p = sw.st_p;
        const double rs = ss > 0.0 ? DSQRT(ss) : 0.0;
        const int n_upd = dneg_w != 0.0 ? sw.n_act : 0;
        for (int k = lane; k < K; k += 32) {
            const double ub = ubuf[k];
            const double pk = (double)T[pos * K + k];
            double ug = 0.0;
            if (cosine) {
                if (ss > 0.0 && tt_p > 0.0) {
                    const double denom = DMUL(DMUL(ss, rs), DSQRT(tt_p));
                    ug = DADD(ug, DDIV(DMUL(dpos, DSUB(DMUL(pk, ss), DMUL(st_p, ub))), denom));
                }
                for (int a = 0; a < n_upd; ++a) {
                    const int j = act[a];
                    const float v = T[(int64_t)nids[j] * K + k];
                    snap[(size_t)a * K + k] = v;
                    const double tj = tts[j];
                    if (ss > 0.0 && tj > 0.0) {
                        const double denom = DMUL(DMUL(ss, rs), DSQRT(tj));
                        ug = DADD(ug, DDIV(DMUL(dneg_w, DSUB(DMUL((double)v, ss),
                                                             DMUL(sts[j], ub))), denom));
                    }
                }
            } else {
                ug = DADD(ug, DMUL(dpos, pk));
                for (int a = 0; a < n_upd; ++a) {
                    const float v = T[(int64_t)nids[act[a]] * K + k];
                    snap[(size_t)a * K + k] = v;
                    ug = DADD(ug, DMUL(dneg_w, (double)v));
                }
            }
            float *tp = T + pos * K + k;
            if (cosine) {
                if (ss > 0.0 && tt_p > 0.0) {
                    const double denom = DMUL(DMUL(tt_p, DSQRT(tt_p)), rs);
                    const double g = DDIV(DMUL(dpos, DSUB(DMUL(ub, tt_p), DMUL(st_p, pk))), denom);
                    const double t = (double)*tp;
                    *tp = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
                } else if (l2 != 0.0) {
                    const double t = (double)*tp;
                    *tp = __double2float_rn(DSUB(t, DMUL(DMUL(lr, l2), t)));
                }
            } else {
                const double g = DMUL(dpos, ub);
                const double t = (double)*tp;
                *tp = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
            }
            int a = 0;
            for (int j = 0; j < N; ++j) {
                const bool is_act = a < n_upd && act[a] == j;
                if (!is_act && l2 == 0.0) {
                    if (a >= n_upd) break;
                    continue;
                }
                float *tn = T + (int64_t)nids[j] * K + k;
                const double t = (double)*tn;
                if (is_act) {
                    const double vs = (double)snap[(size_t)a * K + k];
                    ++a;
                    double g;
                    if (cosine) {
                        const double tj = tts[j];
                        if (!(ss > 0.0 && tj > 0.0)) continue;
                        const double denom = DMUL(DMUL(tj, DSQRT(tj)), rs);
                        g = DDIV(DMUL(dneg_w, DSUB(DMUL(ub, tj), DMUL(sts[j], vs))), denom);
                    } else {
                        g = DMUL(dneg_w, ub);
                    }
                    *tn = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
                } else {
                    *tn = __double2float_rn(DSUB(t, DMUL(DMUL(lr, l2), t)));
                }
            }
            float *su = S + u * K + k;
            const double s = (double)*su;
            *su = __double2float_rn(DSUB(s, DMUL(lr, DADD(ug, DMUL(l2, s)))));
        }
    };

    unsigned long long t_spec = 0, t_wait = 0, t_commit = 0, n_part = 0, n_full = 0, n_pairs = 0;
    const int nwarps = Lo.warps;
    for (int64_t p = start + w; p < stop; p += nwarps) {
        long long c_a = clock64();
        speculate(p, 0u, true);
        long long c_b = clock64();
        for (int64_t t; (t = ld_volatile(token)) != p;)
            if (p - t > 1) __nanosleep(64);  // the next in line spins without sleeping
        __threadfence_block();
        long long c_c = clock64();
        // validate: has any row this pair read been written since c0?
        const int c0 = (int)(sw.c0 - start);
        unsigned smask = 0u;
        for (int r = lane, i = 0; r <= N; r += 32, ++i)
            if (stamp_ld(r == 0 ? sw.pos : (int64_t)nids[r - 1]) >= c0) smask |= 1u << i;
        const bool user_stale = __any_sync(0xffffffffu, lane == 0 && stamp_ld(t_rows + sw.u) >= c0);
        const bool part_stale = __any_sync(0xffffffffu, smask != 0u);
        auto wait_visible = [&]() {  // every earlier pair's row stores are visible
            while (ld_volatile(visible) != p) {
            }
            __threadfence_block();
        };
        // every earlier pair is committed: re-read values are final once visible
        if (user_stale) {
            wait_visible();
            speculate(p, 0u, true);
            ++n_full;
        } else if (part_stale) {
            wait_visible();
            speculate(p, smask, false);
            ++n_part;
        }
        const int me = (int)(p - start);
        const int n_w = sw.n_w;
        const int n_upd = dneg_w != 0.0 ? sw.n_act : 0;
        auto stamp_and_count = [&]() {
            if (lane == 0) {
                stamp_st(sw.pos, me);
                stamp_st(t_rows + sw.u, me);
            }
            if (l2 != 0.0) {
                for (int j = lane; j < N; j += 32) stamp_st(nids[j], me);
            } else {
                for (int a = lane; a < n_upd; a += 32) stamp_st(nids[act[a]], me);
            }
            if (lane == 0) {
                *loss_run = DADD(*loss_run, sw.pair_loss);
                degen_total += sw.degen;
                if (dneg_w != 0.0) active_total += sw.n_act;
            }
        };
        if (n_w >= 0) {
            // precomputed: stamps first, hand the token on, then store the rows
            stamp_and_count();
            __threadfence_block();
            __syncwarp();
            if (lane == 0) *reinterpret_cast<volatile int64_t *>(token) = p + 1;
            for (int i = 0; i < n_w; ++i) {
                float *dst = T + (int64_t)wid[i] * K;
                const float *src = newv + (size_t)i * K;
                for (int k = lane; k < K; k += 32) dst[k] = src[k];
            }
            float *su = S + sw.u * K;
            for (int k = lane; k < K; k += 32) su[k] = snew[k];
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                while (ld_volatile(visible) != p) {
                }
                *reinterpret_cast<volatile int64_t *>(visible) = p + 1;
            }
            __syncwarp();
        } else {
            // update in place: reads the current rows, so every earlier store first
            wait_visible();
            update_in_place();
            __syncwarp();
            stamp_and_count();
            __threadfence_block();
            __syncwarp();
            if (lane == 0) {
                *reinterpret_cast<volatile int64_t *>(visible) = p + 1;
                *reinterpret_cast<volatile int64_t *>(token) = p + 1;
            }
            __syncwarp();
        }
        long long c_d = clock64();
        t_spec += c_b - c_a;
        t_wait += c_c - c_b;
        t_commit += c_d - c_c;
        ++n_pairs;
    }
    if (lane == 0) {
        atomicAdd(&g_spec_stats[0], t_spec);
        atomicAdd(&g_spec_stats[1], t_wait);
        atomicAdd(&g_spec_stats[2], t_commit);
        atomicAdd(&g_spec_stats[3], n_part);
        atomicAdd(&g_spec_stats[4], n_full);
        atomicAdd(&g_spec_stats[5], n_pairs);
    }
    __syncthreads();
    if (threadIdx.x == 0) ctr->loss = *loss_run;
    if (lane == 0) {
        if (degen_total)
            atomicAdd((unsigned long long *)&ctr->degenerate, (unsigned long long)degen_total);
        if (active_total)
            atomicAdd((unsigned long long *)&ctr->active, (unsigned long long)active_total);
    }
    if (threadIdx.x == 0)
        atomicAdd((unsigned long long *)&ctr->pairs, (unsigned long long)(stop - start));
}

static SpecLayout pick_layout(int K, int N, int64_t rows_total) {
    // most speculating warps first (16 for c1/c2), then stamps in shared
    // memory, then the widest precompute buffer; wide pairs (c3/c4: N+1 up to
    // 1024) fall back to fewer warps with stamps in global memory
    const size_t cap = 220 * 1024;
    const int warp_opts[] = {16, 12, 8, 6, 4};
    for (int warps : warp_opts)
        for (int smem_stamps = 1; smem_stamps >= 0; --smem_stamps)
            for (int wcap = 16; wcap >= 2; wcap /= 2) {
                SpecLayout L = spec_layout(K, N, rows_total, wcap, smem_stamps != 0, warps);
                if (L.total <= cap) return L;
            }
    return spec_layout(K, N, rows_total, 2, false, 4);
}

void exact_spec_stats(unsigned long long *out, bool reset) {
    cudaMemcpyFromSymbol(out, g_spec_stats, sizeof(unsigned long long) * 8);
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(g_spec_stats, z, sizeof z);
    }
}

bool exact_spec_supported(int K, int N) {
    if (K > kSpecMaxK || N + 1 > kSpecMaxRows) return false;
    return spec_layout(K, N, 0, 2, false, 4).total <= 220 * 1024;
}

size_t exact_spec_scratch_bytes(int K, int N, int64_t s_rows, int64_t t_rows) {
    return (size_t)kSpecWarps * N * K * sizeof(float) + (size_t)(s_rows + t_rows) * 4 + 256;
}

cudaError_t launch_exact_spec(float *S, int64_t s_rows, float *T, int64_t t_rows,
                              const int32_t *users, const int32_t *items, int64_t start,
                              int64_t stop, int K, int N, int cosine, double lr, double l2,
                              double mu, double theta, uint64_t s0, heat_counters *ctr,
                              void *scratch, const int64_t *pair_index, cudaStream_t stream) {
    float *snap = reinterpret_cast<float *>(scratch);
    uintptr_t sp = reinterpret_cast<uintptr_t>(snap + (size_t)kSpecWarps * N * K);
    int32_t *gstamps = reinterpret_cast<int32_t *>((sp + 15) & ~uintptr_t(15));
    const SpecLayout L = pick_layout(K, N, s_rows + t_rows);
    cudaError_t e = cudaFuncSetAttribute(exact_spec_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.total);
    if (e != cudaSuccess) return e;
    const FastMod fm = FastMod::make((uint64_t)t_rows);
    for (int64_t a = start; a < stop; a += kSpecChunk) {  // stamps are per launch
        const int64_t b = a + kSpecChunk < stop ? a + kSpecChunk : stop;
        if (!L.smem_stamps) {
            e = cudaMemsetAsync(gstamps, 0xff, (size_t)(s_rows + t_rows) * 4, stream);
            if (e != cudaSuccess) return e;
        }
        exact_spec_kernel<<<1, 32 * L.warps, L.total, stream>>>(
            S, T, users, items, a, b, K, N, cosine, lr, l2, mu, theta, s0, fm, ctr, snap, gstamps,
            t_rows, s_rows, pair_index, L);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace heat
