// heat_hogwild_resident.cu — throughput SGD for pairs whose rows fit in shared
// memory (N+1 <= 32*kMaxStages rows): one CTA per pair-worker, one warp per
// 32-row stage, the whole pair resident at once.
//
// Why: with a window of B pairs in flight only ~B/148 workers share an SM.
// One warp per worker leaves ~1.7 warps per scheduler and exposes every
// shared-memory and FMA latency (measured: 36 % issue efficiency).  Here the
// same B pairs are served by NB = ceil((N+1)/32) warps each, so an SM holds
// ~7 pairs but ~28 warps.
//
// Per pair (math = trainer.py:114-293, Hogwild across CTAs):
//   A  every warp draws its stage's negative ids (counter-form SplitMix64,
//      one draw per lane) and copies its rows with per-lane 16-byte
//      cp.async.cg (LDGSTS, L2 evict-last hint) into a padded ring
//      (rows padded by 16 bytes: conflict-free lane-per-row reads), plus its
//      own copy of the user row.  wait_group 0; the warp then arrives on the
//      pair's mbarrier (its reads are complete).
//   B  lane j of warp w scores row w*rw+j: tt = v.v, st = u.v (fp32 FFMA2),
//      fp32 similarity screen, exact binary64 only near the margin
//      (trainer.py:184-221).  Then the warp waits on the mbarrier: every row
//      of the pair has landed before anything is written (the reference
//      reads all rows first, trainer.py:118-146).
//   C  each warp applies the rows of its own stage that must be written:
//      item deltas with red.global.add from the resident snapshot rows
//      (pre-pair values even for repeated ids), and adds its user-gradient
//      partial to the user row (trainer.py:236-293).  Only the warp that
//      reads a stage ever reads it, so no other barrier is needed.
// Measured on c2: a CTA barrier before B: 333 M samples/s; after B (EARLY):
// 340 M; the split arrive/wait (SPLIT, default): 356 M.  HEAT_RESIDENT_EARLY
// = 0 / 1 / 2 selects them.
// The pair's loss (1 - sim_p) + mu/N * sum(hinge) is linear, so each warp
// accumulates its share (trainer.py:222).
#include <cstdint>
#include <cstdlib>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

constexpr int kMaxStages = 8;
#ifndef RS_SLEEP_WAIT
#define RS_SLEEP_WAIT 1
#endif
constexpr bool kSleepWait = RS_SLEEP_WAIT != 0;

template <int K>
struct RsGeom {
    static constexpr int ROWB = K * 4;
    static constexpr int CH = K / 4;  // 16-byte chunks per row
    static constexpr int VW = K >= 32 ? K / 32 : 1;
    static constexpr int ACT = K >= 32 ? 32 : K;
    // rows padded by 16 bytes: lane j reading row j at the same chunk hits
    // bank group (j * (K/4 + 1)) mod 8 — conflict-free LDS.128, constant
    // offsets (an XOR swizzle saves 1.6 KB but costs ~400 instructions/pair)
    static constexpr int SLOTF = K + 4;
};

template <int K>
__host__ __device__ inline size_t rs_smem_bytes(int rows, int nb, bool early) {
    size_t b = sizeof(float) * RsGeom<K>::SLOTF * rows;  // ring, one padded slot per row
    // user row: double-buffered by pair parity, or one copy per warp (EARLY)
    b += sizeof(float) * K * (early ? nb : 2);
    return (b + 127) & ~size_t(127);
}

template <int VW>
__device__ __forceinline__ void rs_red(float *p, const float (&d)[VW]) {
    if constexpr (VW == 1) {
        atomicAdd(p, d[0]);
    } else if constexpr (VW == 2) {
        red_add2(p, d[0], d[1]);
    } else {
#pragma unroll
        for (int i = 0; i < VW; i += 4) red_add4(p + i, d[i], d[i + 1], d[i + 2], d[i + 3]);
    }
}

// EARLY: every warp copies its own user row and scores its stage as soon as
// its own copies land; the CTA barrier moves to just before the writes (all
// of the pair's reads still precede any of its writes).  Otherwise warp 0
// copies one shared user row and every warp waits at the barrier first.
// SPLIT (with EARLY): the pre-write barrier is an mbarrier whose arrival each
// warp signals as soon as its own copies land, before it scores, so the wait
// before the writes rarely stalls.
// DR: the pair range and stream base come from HogwildArgs::range_dev/s0_dev
// PIPE (with SPLIT and IDPF, not at window 1): a warp whose stage has at most
// two rows to write computes their deltas into registers right after scoring,
// issues the NEXT pair's copies into its stage (now free), and only then waits
// for the pair's mbarrier and writes — the wait overlaps the next copies
// instead of spinning (round 1: ~470 of 2198 instructions per c2 pair were the
// wait loop).  A stage with more rows to write takes the unpipelined order.
// Measured on c2: 303.6 M samples/s against 346.2 M without it (the next
// pair's copies, issued ahead of the writes, delay them; the wait was not the
// binding cost), so HEAT_RESIDENT_PIPE=1 only.
template <int K, int NB, bool EARLY, bool SPLIT, bool IDPF, bool DR, bool PIPE>
// 7 resident CTAs per SM (the window allows ~7 pairs per SM), but never
// fewer than 64 registers per thread
__global__ void __launch_bounds__(32 * NB, (32 / NB < 7 ? (32 / NB > 0 ? 32 / NB : 1) : 7))
    hogwild_resident(HogwildArgs a, FastMod fm, int n_workers, int strict) {
    using G = RsGeom<K>;
    constexpr int VW = G::VW;
    extern __shared__ __align__(128) unsigned char sm[];
    float *ring = reinterpret_cast<float *>(sm);
    const int rw_all = (a.N + 1 + NB - 1) / NB;  // rows per warp (see below)
    float *ubuf = ring + (size_t)G::SLOTF * (rw_all * NB);

    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    __shared__ uint64_t reads_done;  // SPLIT: one arrival per warp per pair
    uint32_t phase = 0;
    if (SPLIT) {
        if (threadIdx.x == 0) mbar_init(&reads_done, NB);
        __syncthreads();
    }
    const int N = a.N;
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;
    const uint64_t pol = policy_evict_last();
    // rows spread evenly over the NB warps (c2: 26/25/25/25 instead of
    // 32/32/32/5), so no warp's loads gate the pair barrier for long
    const int rw = (N + 1 + NB - 1) / NB;      // rows per warp
    const int r = w * rw + lane;               // my row of every pair
    const bool valid = lane < rw && r <= N;
    const int nvalid = max(0, min(rw, N + 1 - w * rw));
    constexpr int RPI = 32 / G::CH > 0 ? 32 / G::CH : 1;  // rows per copy instruction
    constexpr int NI = 32 / RPI;
    const int my_ch = lane % G::CH, my_rsub = lane / G::CH;
    float *my_stage = ring + (size_t)w * rw * G::SLOTF;

    double loss = 0.0;
    long long degen = 0, active = 0, mine = 0;
    int parity = 0;
    // counter-form SplitMix64: draw (pg*N + r - 1) of the epoch stream has
    // state s0 + (pg*N + r) * GAMMA = s0 + pg*(N*GAMMA) + r*GAMMA
    const uint64_t lane_off = (uint64_t)r * kGamma;
    const uint64_t pair_step = (uint64_t)N * kGamma;
    // pair metadata one pair ahead, so no dependent global load sits at the
    // head of a pair
    int64_t k_start = a.start, k_stop = a.stop;
    uint64_t k_s0 = a.s0;
    if constexpr (DR) {
        k_start = a.range_dev[0];
        k_stop = a.range_dev[1];
        k_s0 = *a.s0_dev;
    }
    int64_t p = k_start + blockIdx.x;
    int32_t nx_pos = 0, nx_u = 0;
    int64_t nx_pg = 0;
    if (p < k_stop) {
        nx_pos = a.items[p];
        nx_u = a.users[p];
        nx_pg = a.pair_index ? a.pair_index[p] : p;
    }
    // IDPF: the next pair's row ids are drawn while this pair's copies are in
    // flight (the SplitMix64 + modulo chain then never sits at a pair's head)
    uint32_t nx_id = (uint32_t)nx_pos;
    if (IDPF && r > 0) nx_id = (uint32_t)fm.mod(mix64(k_s0 + (uint64_t)nx_pg * pair_step + lane_off));

    // this warp's stage copies (row ids: lane j holds row j's) and its user row
    auto issue_copies = [&](uint32_t ids, int64_t uid, float *udst) {
        const float *srcb = a.T + my_ch * 4;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int row = i * RPI + my_rsub;
            const uint32_t rid = __shfl_sync(0xffffffffu, ids, row & 31);
            if (row < nvalid)
                cp_async16_hint(my_stage + row * G::SLOTF + my_ch * 4, srcb + (size_t)rid * K, pol);
        }
        if (EARLY || w == 0)
            for (int ch = lane; ch < G::CH; ch += 32)
                cp_async16(udst + ch * 4, a.S + uid * K + ch * 4);
        cp_async_commit();
    };
    bool pre = false;  // PIPE: this pair's copies were issued by the previous one

    for (; p < k_stop; p += n_workers, parity ^= 1) {
        ++mine;
        float *urow = EARLY ? ubuf + w * K : ubuf + parity * K;
        // ---- A: ids, copies
        const int32_t pos = nx_pos;
        const int64_t u = nx_u;
        const int64_t pg = nx_pg;
        const bool has_next = p + n_workers < k_stop;
        if (has_next) {
            nx_pos = a.items[p + n_workers];
            nx_u = a.users[p + n_workers];
            nx_pg = a.pair_index ? a.pair_index[p + n_workers] : p + n_workers;
        }
        uint32_t id = (uint32_t)pos;
        if (IDPF)
            id = nx_id;
        else if (r > 0)
            id = (uint32_t)fm.mod(mix64(k_s0 + (uint64_t)pg * pair_step + lane_off));
        {
            if (!pre) issue_copies(id, u, urow);
            if (IDPF) {
                nx_id = (uint32_t)nx_pos;
                if (r > 0)
                    nx_id = (uint32_t)fm.mod(
                        mix64(k_s0 + (uint64_t)nx_pg * pair_step + lane_off));
            }
            cp_async_wait<0>();
        }
        if (EARLY) {
            __syncwarp();  // this warp's stage and user row have landed
            if (SPLIT && lane == 0) mbar_arrive(&reads_done);
        } else
            __syncthreads();  // every row of the pair (and the user row) has landed

        // ---- B: score my row
        float uu[VW];
        float sp = 0.f;
#pragma unroll
        for (int i = 0; i < VW; ++i) {
            uu[i] = lane < G::ACT ? urow[lane * VW + i] : 0.f;
            sp = fmaf(uu[i], uu[i], sp);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
        const double ss = (double)sp;
        const float rss = sp > 0.f ? rsqrtf(sp) : 0.f;
        const float *row = my_stage + lane * G::SLOTF;
        // packed fp32x2 FMA (FFMA2, sm_100): half the FMA instructions of the
        // scalar loop, four independent accumulator pairs
        float2 ta = make_float2(0.f, 0.f), tb = ta, sa = ta, sb = ta;
        if (valid) {
#pragma unroll
            for (int c = 0; c < G::CH; ++c) {
                const float4 v = *reinterpret_cast<const float4 *>(row + c * 4);
                const float4 w4 = *reinterpret_cast<const float4 *>(urow + c * 4);
                const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
                ta = __ffma2_rn(vlo, vlo, ta);
                tb = __ffma2_rn(vhi, vhi, tb);
                sa = __ffma2_rn(make_float2(w4.x, w4.y), vlo, sa);
                sb = __ffma2_rn(make_float2(w4.z, w4.w), vhi, sb);
            }
        }
        const float ttf = (ta.x + ta.y) + (tb.x + tb.y);
        const float stf = (sa.x + sa.y) + (sb.x + sb.y);
        // fp32 screen; rows that can reach the margin are decided from the
        // reference's binary64 sums over the resident row (heat_row_update.cuh)
        float sf = 0.f;
        const bool band = valid && margin_band(r, a.cosine, sp, ttf, stf, rss, theta_f, &sf);
        double ssx = ss, ttx = (double)ttf, stx = (double)stf;
        for (unsigned mb = __ballot_sync(0xffffffffu, band), first = 1; mb; first = 0) {
            const int src = __ffs(mb) - 1;
            mb &= mb - 1;
            double s_, t_, c_;
            warp_dots64<K>(urow, my_stage + src * G::SLOTF, ContiguousCols{}, first != 0, s_, t_,
                           c_);
            if (first) ssx = s_;  // every lane: the binary64 u.u of the pair
            if (lane == src) {
                ttx = t_;
                stx = c_;
            }
        }
        if (!band) ssx = ss;
        bool write = false;
        double wt = 0.0, hinge = 0.0, sim = 0.0;
        if (valid) {
            bool degenerate = false;
            sim = band ? stx : (double)sf;
            if (a.cosine) {
                if (band) {
                    degenerate = ssx <= 0.0 || ttx <= 0.0;
                    sim = degenerate ? 0.0 : stx / (sqrt(ssx) * sqrt(ttx));
                }
                if (degenerate) ++degen;
            }
            if (r == 0) {
                wt = -1.0;
                write = !(a.cosine && degenerate) || a.l2 != 0.f;
                loss += 1.0 - sim;
            } else {
                if (sim - a.theta > 0.0) {
                    hinge = sim - a.theta;
                    wt = wneg;
                    if (wt != 0.0) ++active;
                }
                write = (wt != 0.0 && !(a.cosine && degenerate)) || (wt == 0.0 && a.l2 != 0.f);
            }
        }
        loss += wneg * hinge;
        unsigned m = __ballot_sync(0xffffffffu, write);
        // PIPE: deltas of at most two written rows into registers, then the
        // next pair's copies, then the wait
        const bool pipe = PIPE && !strict && has_next && __popc(m) <= 2;
        pre = pipe;
        float dq[2][VW], ugp[VW];
        int32_t idq[2] = {0, 0};
        if (pipe) {
#pragma unroll
            for (int i = 0; i < VW; ++i) ugp[i] = 0.f;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int src = m ? __ffs(m) - 1 : 0;
                const bool live = m != 0;
                m &= m ? m - 1 : 0u;
                const double tt_s = __shfl_sync(0xffffffffu, ttx, src);
                const double st_s = __shfl_sync(0xffffffffu, stx, src);
                const double ss_s = __shfl_sync(0xffffffffu, ssx, src);
                const float w_s = (float)__shfl_sync(0xffffffffu, wt, src);
                idq[q] = live ? (int32_t)__shfl_sync(0xffffffffu, id, src) : -1;
                if (live) {
                    const WriteEntry we{tt_s, st_s, (double)w_s, idq[q], 0};
                    const RowCoef co = row_coef_f(we, ss_s, rss, a.lr, a.l2, a.cosine);
                    const float *srow = my_stage + src * G::SLOTF;
#pragma unroll
                    for (int i = 0; i < VW; ++i) {
                        const int col = lane * VW + i;
                        const float v = lane < G::ACT ? srow[col] : 0.f;
                        row_apply(co, uu[i], v, dq[q][i], ugp[i]);
                    }
                }
            }
            __syncwarp();  // every lane's reads of the stage are done
            issue_copies(nx_id, nx_u, urow);
        }
        if (SPLIT) {  // every read of the pair precedes every write
            if (kSleepWait)
                mbar_wait_sleep(&reads_done, phase);
            else
                mbar_wait(&reads_done, phase);
            phase ^= 1;
        } else if (EARLY) {
            __syncthreads();
        }

        if (pipe) {  // ---- C (pipelined): the registered deltas
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (idq[q] < 0) continue;
                if (!dmode) {
                    if (lane < G::ACT) rs_red<VW>(a.T + (int64_t)idq[q] * K + lane * VW, dq[q]);
                } else {
                    long long sl = 0;
                    if (lane == 0) sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                    sl = __shfl_sync(0xffffffffu, sl, 0);
                    if (sl < a.delta_capacity) {
                        if (lane == 0) a.delta_ids[sl] = idq[q];
                        if (lane < G::ACT) {
#pragma unroll
                            for (int i = 0; i < VW; ++i) a.delta_rows[sl * K + lane * VW + i] = dq[q][i];
                        }
                    }
                }
            }
            if (idq[0] >= 0 && lane < G::ACT) {
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) d[i] = -a.lr * ugp[i];
                rs_red<VW>(a.S + u * K + lane * VW, d);
            }
            m = 0;
        }

        // ---- C: apply my stage's written rows from their resident snapshots
        if (m) {
            float ug[VW];
#pragma unroll
            for (int i = 0; i < VW; ++i) ug[i] = 0.f;
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const double tt_s = __shfl_sync(0xffffffffu, ttx, src);
                const double st_s = __shfl_sync(0xffffffffu, stx, src);
                const double ss_s = __shfl_sync(0xffffffffu, ssx, src);
                const float w_s = (float)__shfl_sync(0xffffffffu, wt, src);
                const int32_t id_s = (int32_t)__shfl_sync(0xffffffffu, id, src);
                const WriteEntry we{tt_s, st_s, (double)w_s, id_s, 0};
                const RowCoef co = row_coef_f(we, ss_s, rss, a.lr, a.l2, a.cosine);
                const float *srow = my_stage + src * G::SLOTF;
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) {
                    const int col = lane * VW + i;
                    const float v = lane < G::ACT ? srow[col] : 0.f;
                    row_apply(co, uu[i], v, d[i], ug[i]);
                }
                if (!dmode) {
                    if (lane < G::ACT) rs_red<VW>(a.T + (int64_t)id_s * K + lane * VW, d);
                } else {
                    long long sl = 0;
                    if (lane == 0)
                        sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                    sl = __shfl_sync(0xffffffffu, sl, 0);
                    if (sl < a.delta_capacity) {
                        if (lane == 0) a.delta_ids[sl] = id_s;
                        if (lane < G::ACT) {
#pragma unroll
                            for (int i = 0; i < VW; ++i) a.delta_rows[sl * K + lane * VW + i] = d[i];
                        }
                    }
                }
            }
            // this warp's share of the user gradient (trainer.py:291-293)
            if (lane < G::ACT) {
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) d[i] = -a.lr * ug[i];
                rs_red<VW>(a.S + u * K + lane * VW, d);
            }
        }
        // decay of the user row itself (l2 != 0), once per pair
        if (w == 0 && a.l2 != 0.f && lane < G::ACT) {
            float d[VW];
#pragma unroll
            for (int i = 0; i < VW; ++i) d[i] = -a.lr * a.l2 * uu[i];
            rs_red<VW>(a.S + u * K + lane * VW, d);
        }
        __syncwarp();
        // strict (window 1): the next pair reads only after every warp's
        // writes of this one, so the worker runs the reference's sequence;
        // otherwise a warp may read pair t+1 while another still writes t
        if (strict) {
            __threadfence_block();
            __syncthreads();
        }
    }
    // telemetry
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(0xffffffffu, degen, o);
        active += __shfl_xor_sync(0xffffffffu, active, o);
        loss += __shfl_xor_sync(0xffffffffu, loss, o);
    }
    if (lane == 0) {
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
        atomicAdd(&a.ctr->loss, loss);
    }
    if (threadIdx.x == 0) atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine);
}

template <int K, int NB>
static cudaError_t launch_resident_kn(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    static const int early = [] {
        const char *e = getenv("HEAT_RESIDENT_EARLY");
        return e ? atoi(e) : 2;
    }();
    const size_t smem = rs_smem_bytes<K>(((a.N + 1 + NB - 1) / NB) * NB, NB, early != 0);
    if (smem > 96 * 1024) return cudaErrorNotSupported;
    static const bool idpf = [] {
        const char *e = getenv("HEAT_RESIDENT_IDPF");
        return e ? atoi(e) != 0 : true;  // measured c2: 357.7 M vs 355.9 M
    }();
    // PIPE measured slower on c2 (303.6 M vs 346.2 M samples/s): opt-in only
    static const bool pipe = [] {
        const char *e = getenv("HEAT_RESIDENT_PIPE");
        return e ? atoi(e) != 0 : false;
    }();
    auto kern = a.range_dev ? (pipe ? hogwild_resident<K, NB, true, true, true, true, true>
                                    : hogwild_resident<K, NB, true, true, true, true, false>)
                : early == 2 ? (idpf ? (pipe ? hogwild_resident<K, NB, true, true, true, false, true>
                                             : hogwild_resident<K, NB, true, true, true, false, false>)
                                     : hogwild_resident<K, NB, true, true, false, false, false>)
                : early == 1 ? hogwild_resident<K, NB, true, false, false, false, false>
                             : hogwild_resident<K, NB, false, false, false, false, false>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32 * NB, smem, &e);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (a.stop - a.start < nw) nw = a.stop - a.start;
    if (workers_out) *workers_out = (int)nw;
    kern<<<(unsigned)nw, 32 * NB, smem, st>>>(a, FastMod::make((uint64_t)a.num_items), (int)nw,
                                              a.window == 1 ? 1 : 0);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_resident_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    const int nb = (a.N + 1 + 31) / 32;
    // one stage per pair: the single-warp staged kernel covers it (as fast,
    // measured; the 1-warp instantiation also faulted on sm_100a — not used)
    if (nb > kMaxStages || nb < 2) return cudaErrorNotSupported;
    switch (nb) {
    case 2: return launch_resident_kn<K, 2>(a, st, workers_out);
    case 3: return launch_resident_kn<K, 3>(a, st, workers_out);
    case 4: return launch_resident_kn<K, 4>(a, st, workers_out);
    case 5: return launch_resident_kn<K, 5>(a, st, workers_out);
    case 6: return launch_resident_kn<K, 6>(a, st, workers_out);
    case 7: return launch_resident_kn<K, 7>(a, st, workers_out);
    default: return launch_resident_kn<K, 8>(a, st, workers_out);
    }
}

cudaError_t launch_hogwild_resident(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    if (a.fp64) return cudaErrorNotSupported;  // binary64 dots: staged kernel
    switch (a.K) {
    case 16: return launch_resident_k<16>(a, st, workers_out);
    case 32: return launch_resident_k<32>(a, st, workers_out);
    case 64: return launch_resident_k<64>(a, st, workers_out);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace heat
