// heat_exact.cu — deterministic ("exact") SGD over pairs in strict order.
//
// Bit-identical to the reference with num_threads=1: it restates the
// per-pair body of /root/reference/pkg/src/heatcf/trainer.py:114-297
// (tiled=False, agg_on=False) with every binary64 operation written as an
// explicit round-to-nearest intrinsic (__dmul_rn, __dadd_rn, __ddiv_rn,
// __dsqrt_rn), so nothing can be contracted into an FMA, and float32
// rounding on store (__double2float_rn).  This file is also compiled with
// --fmad=false as a second guard.
//
// Parallel decomposition of one pair (one CTA, pairs sequential):
//   read/similarity  thread r owns row r (r=0 the positive, r>=1 negative r-1):
//                    a strictly sequential k-loop for tt and st, exactly the
//                    reference's accumulation order (trainer.py:176-207);
//   loss             ordered active list built with warp ballots, the hinge
//                    summed in j order by one thread (trainer.py:214-222);
//   gradient/update  thread k owns column k of every row: ugrad[k] in j order
//                    (trainer.py:230-251), then T[pos], T[neg_j] in j order,
//                    S[u] (trainer.py:259-293).  A column is only ever
//                    touched by its own thread inside a pair, so repeated ids
//                    (pos == neg, duplicate negatives) see the same
//                    read-after-write order as the reference.  Snapshots of
//                    active negative rows (the reference's neg_buf) are taken
//                    column-wise before any write.
#include <cstdint>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

#define DMUL __dmul_rn
#define DADD __dadd_rn
#define DSUB __dsub_rn
#define DDIV __ddiv_rn
#define DSQRT __dsqrt_rn

constexpr int kExactThreads = 512;
constexpr int kExactWarps = kExactThreads / 32;

struct ExactSmem {
    double ss, tt_p, st_p, sim_p;
    int n_loss;  // negatives with d > 0, in j order in list[]
    int warp_cnt[kExactWarps];
};

// phase profile (PH, heat_phase_collect): [0, 6) clocks per phase, [6] the
// last mark, [7] the start clock, [8] the start globaltimer, [9] the clocks
// thread 0 spent on its column's gradient in the fused gradient/update loop
__shared__ long long s_xph[10];

// PH: the clocks of the pair's phases (trainer.py:120-331 collect_phases)
// into `phase`, the phases in the reference's order and extent; the fused
// gradient + update loop (one column per thread) is split by thread 0's own
// share of it
template <bool PH>
__global__ void __launch_bounds__(kExactThreads, 1)
    exact_kernel(float *__restrict__ S, float *__restrict__ T, const int32_t *__restrict__ users,
                 const int32_t *__restrict__ items, int64_t start, int64_t stop, int K, int N,
                 int cosine, double lr, double l2, double mu, double theta, uint64_t s0,
                 FastMod fm, heat_counters *ctr, float *__restrict__ snap,
                 const int64_t *__restrict__ pair_index, heat_agg_params ag, int agg_on,
                 unsigned long long *phase) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ExactSmem &sh = *reinterpret_cast<ExactSmem *>(smem_raw);
    double *ubuf = reinterpret_cast<double *>(smem_raw + sizeof(ExactSmem) + 16 -
                                              (sizeof(ExactSmem) % 16));
    double *tts = ubuf + K;
    double *sts = tts + N;
    double *sims = sts + N;
    float *pos_buf = reinterpret_cast<float *>(sims + N);
    int32_t *nids = reinterpret_cast<int32_t *>(pos_buf + K);
    int32_t *list = nids + N;
    // aggregation buffers (binary64): pooled history, h-gradient
    double *pooled = reinterpret_cast<double *>(
        (reinterpret_cast<uintptr_t>(list + N) + 15) & ~uintptr_t(15));
    double *ugs = pooled + K;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    auto gtimer = []() -> long long {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return (long long)t;
    };
    if constexpr (PH) {
        if (tid == 0) {
            for (int i = 0; i < 6; ++i) s_xph[i] = 0;
            s_xph[7] = clock64();
            s_xph[8] = gtimer();
        }
    }
    auto mark = [&](int i) {  // phase i ends here (every thread calls it)
        if constexpr (PH) {
            __syncthreads();
            if (tid == 0) {
                const long long t = clock64();
                s_xph[i] += t - s_xph[6];
                s_xph[6] = t;
            }
        }
    };
    const double inv_n = DDIV(1.0, (double)N);  // trainer.py:113
    const double dneg_w = DMUL(mu, inv_n);      // trainer.py:219
    const double dpos = -1.0;                   // trainer.py:223
    double loss_acc = 0.0;
    if (tid == 0) loss_acc = ctr->loss;
    long long degen = 0, active = 0;
    int64_t agg_ctr = agg_on ? *ag.counter : 0;  // uniform across the CTA
    const double gamma = ag.gamma;

    for (int64_t p = start; p < stop; ++p) {
        if constexpr (PH) {
            __syncthreads();
            if (tid == 0) s_xph[6] = clock64();
        }
        const int64_t u = users[p];
        const int64_t pos = items[p];
        // ---- read (trainer.py:121-142): S[u] -> f64, T[pos] snapshot, ids
        for (int k = tid; k < K; k += kExactThreads) {
            if (!agg_on) ubuf[k] = (double)S[u * K + k];
            pos_buf[k] = T[pos * K + k];
        }
        const int64_t pg = pair_index ? pair_index[p] : p;  // RNG key
        for (int j = tid; j < N; j += kExactThreads) nids[j] = neg_id(s0, pg, N, j, fm);
        mark(0);
        // ---- aggregate forward (trainer.py:150-169): pooled = mean of the
        // first max_history history rows, h = gamma*S[u] + (1-gamma)*pooled.W
        int64_t hb = 0, hist_len = 0;
        if (agg_on) {
            hb = ag.tr_offsets[u];
            int64_t he = ag.tr_offsets[u + 1];
            if (he - hb > ag.max_history) he = hb + ag.max_history;
            hist_len = he - hb;
            for (int k = tid; k < K; k += kExactThreads) {
                double acc = 0.0;
                for (int64_t idx = hb; idx < he; ++idx)
                    acc = DADD(acc, (double)T[(int64_t)ag.tr_items[idx] * K + k]);
                if (hist_len > 0) acc = DDIV(acc, (double)hist_len);
                pooled[k] = acc;
            }
            __syncthreads();
            for (int j = tid; j < K; j += kExactThreads) {
                double acc = 0.0;
                for (int k = 0; k < K; ++k) acc = DADD(acc, DMUL(pooled[k], (double)ag.W[k * K + j]));
                ubuf[j] = DADD(DMUL(gamma, (double)S[u * K + j]), DMUL(DSUB(1.0, gamma), acc));
            }
            mark(5);
        }
        __syncthreads();

        // ---- similarity (trainer.py:176-207)
        if (tid == kExactThreads - 1) {
            double ss = 0.0;
            for (int k = 0; k < K; ++k) ss = DADD(ss, DMUL(ubuf[k], ubuf[k]));
            sh.ss = ss;
        }
        for (int r = tid; r <= N; r += kExactThreads) {
            double tt, st;
            if (r == 0) {
                // pos row from the snapshot (trainer.py:181-183)
                double a = 0.0, b = 0.0;
                for (int k = 0; k < K; ++k) {
                    double x = (double)pos_buf[k];
                    a = DADD(a, DMUL(x, x));
                    b = DADD(b, DMUL(ubuf[k], x));
                }
                sh.tt_p = a;
                sh.st_p = b;
            } else {
                row_dots_any(T + (int64_t)nids[r - 1] * K, ubuf, K, tt, st);
                tts[r - 1] = tt;
                sts[r - 1] = st;
            }
        }
        __syncthreads();
        const double ss = sh.ss;
        for (int r = tid; r <= N; r += kExactThreads) {
            double tt = r == 0 ? sh.tt_p : tts[r - 1];
            double st = r == 0 ? sh.st_p : sts[r - 1];
            double sim;
            if (cosine) {
                if (ss <= 0.0 || tt <= 0.0) {
                    sim = 0.0;
                    ++degen;
                } else {
                    sim = DDIV(st, DMUL(DSQRT(ss), DSQRT(tt)));
                }
            } else {
                sim = st;
            }
            if (r == 0) sh.sim_p = sim; else sims[r - 1] = sim;
        }
        __syncthreads();
        mark(1);

        // ---- loss (trainer.py:214-222): ordered list of j with d > 0
        int base = 0;
        for (int j0 = 0; j0 < N; j0 += kExactThreads) {
            int j = j0 + tid;
            bool act = j < N && DSUB(sims[j], theta) > 0.0;
            unsigned m = __ballot_sync(0xffffffffu, act);
            if (lane == 0) sh.warp_cnt[warp] = __popc(m);
            __syncthreads();
            int off = base;
            int total = 0;
            for (int w = 0; w < kExactWarps; ++w) {
                int c = sh.warp_cnt[w];
                if (w < warp) off += c;
                total += c;
            }
            if (act) list[off + __popc(m & ((1u << lane) - 1u))] = j;
            base += total;
            __syncthreads();
        }
        const int n_loss = base;  // identical in every thread
        if (tid == 0) {
            double hinge = 0.0;
            for (int a = 0; a < n_loss; ++a) hinge = DADD(hinge, DSUB(sims[list[a]], theta));
            double pl = DADD(DSUB(1.0, sh.sim_p), DMUL(dneg_w, hinge));
            loss_acc = DADD(loss_acc, pl);
            if (dneg_w != 0.0) active += n_loss;
        }
        // negatives with dnegs[j] != 0 (trainer.py:219: dneg = mu*inv_n)
        const int n_upd = dneg_w != 0.0 ? n_loss : 0;
        mark(2);
        long long tg0 = 0;
        if constexpr (PH) {
            if (tid == 0) tg0 = clock64();
        }

        // ---- gradient + update, thread k owns column k
        const double tt_p = sh.tt_p, st_p = sh.st_p;
        const double rs = ss > 0.0 ? DSQRT(ss) : 0.0;
        for (int k = tid; k < K; k += kExactThreads) {
            const double ub = ubuf[k];
            const double pk = (double)pos_buf[k];
            double ug = 0.0;
            if (cosine) {
                if (ss > 0.0 && tt_p > 0.0) {
                    double denom = DMUL(DMUL(ss, rs), DSQRT(tt_p));
                    ug = DADD(ug, DDIV(DMUL(dpos, DSUB(DMUL(pk, ss), DMUL(st_p, ub))), denom));
                }
                for (int a = 0; a < n_upd; ++a) {
                    const int j = list[a];
                    const float v = T[(int64_t)nids[j] * K + k];
                    snap[(int64_t)a * K + k] = v;
                    const double tj = tts[j];
                    if (ss > 0.0 && tj > 0.0) {
                        double denom = DMUL(DMUL(ss, rs), DSQRT(tj));
                        ug = DADD(ug, DDIV(DMUL(dneg_w, DSUB(DMUL((double)v, ss),
                                                             DMUL(sts[j], ub))), denom));
                    }
                }
            } else {
                ug = DADD(ug, DMUL(dpos, pk));
                for (int a = 0; a < n_upd; ++a) {
                    const float v = T[(int64_t)nids[list[a]] * K + k];
                    snap[(int64_t)a * K + k] = v;
                    ug = DADD(ug, DMUL(dneg_w, (double)v));
                }
            }
            if constexpr (PH) {
                if (tid == 0) s_xph[9] = clock64() - tg0;
            }
            // T[pos] (trainer.py:259-271)
            float *tp = T + pos * K + k;
            if (cosine) {
                if (ss > 0.0 && tt_p > 0.0) {
                    double denom = DMUL(DMUL(tt_p, DSQRT(tt_p)), rs);
                    double g = DDIV(DMUL(dpos, DSUB(DMUL(ub, tt_p), DMUL(st_p, pk))), denom);
                    double t = (double)*tp;
                    *tp = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
                } else if (l2 != 0.0) {
                    double t = (double)*tp;
                    *tp = __double2float_rn(DSUB(t, DMUL(DMUL(lr, l2), t)));
                }
            } else {
                double g = DMUL(dpos, ub);
                double t = (double)*tp;
                *tp = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
            }
            // T[neg_j] in j order (trainer.py:272-290)
            if (l2 == 0.0) {
                for (int a = 0; a < n_upd; ++a) {
                    const int j = list[a];
                    float *tn = T + (int64_t)nids[j] * K + k;
                    const double vs = (double)snap[(int64_t)a * K + k];
                    double g;
                    if (cosine) {
                        const double tj = tts[j];
                        if (!(ss > 0.0 && tj > 0.0)) continue;
                        double denom = DMUL(DMUL(tj, DSQRT(tj)), rs);
                        g = DDIV(DMUL(dneg_w, DSUB(DMUL(ub, tj), DMUL(sts[j], vs))), denom);
                    } else {
                        g = DMUL(dneg_w, ub);
                    }
                    double t = (double)*tn;
                    *tn = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
                }
            } else {
                int a = 0;
                for (int j = 0; j < N; ++j) {
                    float *tn = T + (int64_t)nids[j] * K + k;
                    double t = (double)*tn;
                    if (a < n_upd && list[a] == j) {
                        const double vs = (double)snap[(int64_t)a * K + k];
                        ++a;
                        double g;
                        if (cosine) {
                            const double tj = tts[j];
                            if (!(ss > 0.0 && tj > 0.0)) continue;
                            double denom = DMUL(DMUL(tj, DSQRT(tj)), rs);
                            g = DDIV(DMUL(dneg_w, DSUB(DMUL(ub, tj), DMUL(sts[j], vs))), denom);
                        } else {
                            g = DMUL(dneg_w, ub);
                        }
                        *tn = __double2float_rn(DSUB(t, DMUL(lr, DADD(g, DMUL(l2, t)))));
                    } else {
                        *tn = __double2float_rn(DSUB(t, DMUL(DMUL(lr, l2), t)));
                    }
                }
            }
            // S[u] (trainer.py:291-293; with aggregation gamma*ugrad, 303)
            float *su = S + u * K + k;
            double s = (double)*su;
            if (!agg_on) {
                *su = __double2float_rn(DSUB(s, DMUL(lr, DADD(ug, DMUL(l2, s)))));
            } else {
                *su = __double2float_rn(DSUB(s, DMUL(lr, DADD(DMUL(gamma, ug), DMUL(l2, s)))));
                ugs[k] = ug;
            }
        }
        if constexpr (PH) {  // the loop: thread 0's gradient share, then the update
            __syncthreads();
            if (tid == 0) {
                const long long t = clock64();
                const long long gpart = K > 0 ? s_xph[9] : 0;
                s_xph[3] += gpart;
                s_xph[4] += t - s_xph[6] - gpart;
                s_xph[6] = t;
            }
        }
        if (agg_on) {
            // ---- aggregate backward (trainer.py:304-328)
            __syncthreads();
            const double omg = DSUB(1.0, gamma);
            for (int e = tid; e < K * K; e += kExactThreads) {
                const double pa = DMUL(omg, pooled[e / K]);
                if (pa != 0.0) ag.accu[e] = DADD(ag.accu[e], DMUL(pa, ugs[e % K]));
            }
            agg_ctr += 1;
            if (agg_ctr >= ag.mini_batch) {
                const double inv_m = DDIV(1.0, (double)ag.mini_batch);
                for (int e = tid; e < K * K; e += kExactThreads) {
                    ag.W[e] = __double2float_rn(
                        DSUB((double)ag.W[e], DMUL(DMUL(ag.lr, ag.accu[e]), inv_m)));
                    ag.accu[e] = 0.0;
                }
                agg_ctr = 0;
            }
            if (ag.history_grad && hist_len > 0) {
                __syncthreads();  // W after the flush
                const double scale = DDIV(omg, (double)hist_len);
                for (int k = tid; k < K; k += kExactThreads) {
                    double acc = 0.0;
                    for (int b = 0; b < K; ++b) acc = DADD(acc, DMUL((double)ag.W[k * K + b], ugs[b]));
                    const double wh = DMUL(scale, acc);
                    for (int64_t idx = hb; idx < hb + hist_len; ++idx) {
                        float *th = T + (int64_t)ag.tr_items[idx] * K + k;
                        const double t = (double)*th;
                        *th = __double2float_rn(DSUB(t, DMUL(lr, DADD(wh, DMUL(l2, t)))));
                    }
                }
            }
            mark(5);
        }
        __syncthreads();
    }
    if constexpr (PH) {
        if (tid == 0 && phase) {
            for (int i = 0; i < 6; ++i) atomicAdd(phase + i, (unsigned long long)s_xph[i]);
            atomicAdd(phase + 6, (unsigned long long)(clock64() - s_xph[7]));
            atomicAdd(phase + 7, (unsigned long long)(gtimer() - s_xph[8]));
            atomicAdd(phase + 8, 1ull);
            atomicAdd(phase + 9, (unsigned long long)(stop - start));
        }
    }
    if (agg_on && tid == 0) *ag.counter = agg_ctr;
    // telemetry (order-free integer sums)
    for (int o = 16; o > 0; o >>= 1) degen += __shfl_xor_sync(0xffffffffu, degen, o);
    if (lane == 0 && degen) atomicAdd((unsigned long long *)&ctr->degenerate, (unsigned long long)degen);
    if (tid == 0) {
        ctr->loss = loss_acc;
        atomicAdd((unsigned long long *)&ctr->active, (unsigned long long)active);
        atomicAdd((unsigned long long *)&ctr->pairs, (unsigned long long)(stop - start));
    }
}

size_t exact_smem_bytes(int K, int N) {
    size_t head = sizeof(ExactSmem) + 16 - (sizeof(ExactSmem) % 16);
    return head + (size_t)K * 8 + (size_t)N * 8 * 3 + (size_t)K * 4 + (size_t)N * 4 * 2 + 16 +
           (size_t)K * 8 * 3 + 16;
}

cudaError_t launch_exact(float *S, float *T, const int32_t *users, const int32_t *items,
                         int64_t start, int64_t stop, int K, int N, int cosine, double lr,
                         double l2, double mu, double theta, uint64_t s0, int64_t num_items,
                         heat_counters *ctr, float *snap, const int64_t *pair_index,
                         const heat_agg_params *agg, cudaStream_t stream,
                         unsigned long long *phase) {
    size_t smem = exact_smem_bytes(K, N);
    auto kern = phase ? exact_kernel<true> : exact_kernel<false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<1, kExactThreads, smem, stream>>>(S, T, users, items, start, stop, K, N, cosine, lr,
                                             l2, mu, theta, s0, FastMod::make((uint64_t)num_items),
                                             ctr, snap, pair_index,
                                             agg ? *agg : heat_agg_params{}, agg != nullptr, phase);
    return cudaGetLastError();
}

}  // namespace heat
