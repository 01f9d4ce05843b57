// heat_hogwild_staged.cu — the throughput SGD kernel, shared-memory staged.
//
// Same math and semantics as heat_hogwild.cu (trainer.py:114-293 per pair,
// Hogwild across pairs), organised around the B200 memory system:
//
//  * one warp per CTA, one CTA per pair-worker, so the block scheduler
//    spreads the W workers evenly over all 148 SMs;
//  * every row a pair touches (user row, positive, N negatives) is copied
//    asynchronously into a per-warp ring of D shared-memory stages of 32 rows
//    (rows padded by 16 bytes so the compute reads are bank-conflict-free).
//    Mover (template BULK): per-lane 16-byte cp.async.cg (LDGSTS, 512 B per
//    warp instruction, completion by commit/wait groups) — the default — or
//    one cp.async.bulk per row (the TMA engine, UBLKCP, mbarrier complete_tx).
//    The producer runs D stages ahead, so a warp keeps up to D*32 rows in
//    flight without spending registers;
//  * lane j of the consumer owns row j of a stage and forms tt = v.v and
//    st = u.v with a k loop over LDS.128 (u broadcast) — no cross-lane
//    reduction; the similarity screen is fp32, the exact binary64 value is
//    recomputed for the few rows near the margin (trainer.py:184-221);
//  * rows to write (positive, negatives with sim > theta, decay rows when
//    l2 != 0) are copied from the ring into a per-warp snapshot buffer with
//    their cached scalars (HEAT's forward-value reuse, kernels.py:27-40); at
//    the end of the pair the warp applies them with red.global.add and then
//    updates the user row — every row of the pair is read before any write,
//    the reference's snapshot semantics (trainer.py:118-146, 257-293).
//
// Pairs in flight: with `cross` the producer prefetches the next pair's first
// stages while the current pair is finishing, so each worker holds up to
// 1 + ceil((D-1)/nb) pairs; the launcher divides `window` by that so the
// total never exceeds the window (the staleness bound of a B-pair step).
#include <cstdint>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

// LPR lanes score one row (LPR = 2: each lane takes half of the columns and
// a stage holds 16 rows).  The ring is shared memory's binding resource: at the
// same rows in flight per SM, LPR = 2 halves the rows per warp and doubles the
// warps that hide the LDS/FMA latency.  A slot stores each lane's segment of
// HALF columns followed by 16 bytes of padding, so the lanes of a quarter-warp
// read distinct bank groups.
template <int K, int LPR = 1>
struct StGeom {
    static constexpr int ROWB = K * 4;               // bytes per row
    static constexpr int HALF = K / LPR;             // columns per lane segment
    static constexpr int SEGF = HALF + 4;            // floats per padded segment
    static constexpr int SLOTF = LPR * SEGF;         // floats per padded slot
    static constexpr int CH = K / 4;                 // 16-byte chunks per row
    static constexpr int SR = 32 / LPR;              // rows per stage
    static constexpr int VW = K >= 32 ? K / 32 : 1;  // floats per lane in row-wide ops
    static constexpr int ACT = K >= 32 ? 32 : K;     // lanes active in row-wide ops
    // slot offset of column c
    __host__ __device__ static constexpr int pcol(int c) { return c + (c / HALF) * 4; }
};

struct StLayout {
    int ucap, snap_cap;
    size_t off_bars, off_ubars, off_ids, off_ring, off_urow, off_snap, off_ents, total;
};

template <int K, int D, int LPR = 1>
__host__ __device__ inline StLayout st_layout(int snap_cap) {
    using G = StGeom<K, LPR>;
    StLayout L;
    L.ucap = D + 1;
    L.snap_cap = snap_cap;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = (o + 127) & ~size_t(127);
        o = at + bytes;
        return at;
    };
    L.off_bars = take(sizeof(uint64_t) * D);
    L.off_ubars = take(sizeof(uint64_t) * L.ucap);
    L.off_ids = take(sizeof(int32_t) * G::SR * D);
    L.off_ring = take(sizeof(float) * G::SLOTF * G::SR * D);
    L.off_urow = take(sizeof(float) * G::SLOTF * L.ucap);
    L.off_snap = take(sizeof(float) * K * snap_cap);
    L.off_ents = take(sizeof(WriteEntry) * snap_cap);
    L.total = (o + 127) & ~size_t(127);
    return L;
}

template <int VW>
__device__ __forceinline__ void red_add_vec(float *p, const float (&d)[VW]) {
    if constexpr (VW == 1) {
        atomicAdd(p, d[0]);
    } else if constexpr (VW == 2) {
        red_add2(p, d[0], d[1]);
    } else {
#pragma unroll
        for (int i = 0; i < VW; i += 4) red_add4(p + i, d[i], d[i + 1], d[i + 2], d[i + 3]);
    }
}

#ifndef UREG_MAX
#define UREG_MAX 128
#endif

// DR: the pair range and stream base come from HogwildArgs::range_dev/s0_dev
template <int K, int D, bool F64, bool BULK, int LPR, bool DR>
__global__ void __launch_bounds__(32)
    hogwild_staged(HogwildArgs a, FastMod fm, int n_workers, int snap_cap, int cross) {
    using G = StGeom<K, LPR>;
    constexpr int VW = G::VW;
    constexpr int SR = G::SR;
    // user-row segment held in registers when it is small enough (the ring,
    // not registers, bounds residency)
    constexpr bool UREG = !F64 && G::HALF <= UREG_MAX;
    float2 ureg[UREG ? G::HALF / 2 : 1];
    extern __shared__ __align__(128) unsigned char sm[];
    const StLayout Lo = st_layout<K, D, LPR>(snap_cap);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + Lo.off_bars);
    uint64_t *ubars = reinterpret_cast<uint64_t *>(sm + Lo.off_ubars);
    int32_t *ids = reinterpret_cast<int32_t *>(sm + Lo.off_ids);
    float *ring = reinterpret_cast<float *>(sm + Lo.off_ring);
    float *urow = reinterpret_cast<float *>(sm + Lo.off_urow);
    float *snap = reinterpret_cast<float *>(sm + Lo.off_snap);
    WriteEntry *ents = reinterpret_cast<WriteEntry *>(sm + Lo.off_ents);

    const int lane = threadIdx.x;
    const int rr = lane / LPR;       // this lane's row within a stage
    const int hs = lane % LPR;       // and its column segment
    const bool lead = hs == 0;       // the lane that accounts for the row
    const int gw = blockIdx.x;
    int64_t k_start = a.start, k_stop = a.stop;
    uint64_t k_s0 = a.s0;
    if constexpr (DR) {
        k_start = a.range_dev[0];
        k_stop = a.range_dev[1];
        k_s0 = *a.s0_dev;
    }
    const int64_t npairs = k_stop - k_start;
    if (gw >= n_workers || gw >= npairs) return;
    const int64_t my_pairs = (npairs - gw + n_workers - 1) / n_workers;
    const int N = a.N;
    const int nb = (N + 1 + SR - 1) / SR;  // stages per pair
    const int64_t g_total = my_pairs * nb;
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;
    const uint64_t pol = policy_evict_last();
    float *sp_rows = a.spill ? reinterpret_cast<float *>(a.spill + (size_t)gw * a.spill_stride)
                             : nullptr;
    WriteEntry *sp_ents =
        a.spill ? reinterpret_cast<WriteEntry *>(a.spill + (size_t)gw * a.spill_stride +
                                                 (size_t)a.spill_cap * K * sizeof(float))
                : nullptr;

    if constexpr (BULK) {
        if (lane == 0) {
            for (int i = 0; i < D; ++i) mbar_init(&bars[i], 1);
            for (int i = 0; i < Lo.ucap; ++i) mbar_init(&ubars[i], 1);
        }
        fence_proxy_async();
    }
    __syncwarp();

    // ---- producer: next stage to issue (pair pt, stage ps, ring slot pslot)
    // and the prefetched (user, pos) of its pair; all counters incremental
    int64_t g_next = 0;
    int64_t pt = 0;
    int ps = 0, pslot = 0, pus = 0;
    int32_t pf_u = a.users[k_start + gw];
    int32_t pf_pos = a.items[k_start + gw];
    int64_t pf_p = k_start + gw;  // pair whose user row the producer loads next
    int32_t nx_u = 0, nx_pos = 0;
    if (my_pairs > 1) {
        nx_u = a.users[k_start + gw + n_workers];
        nx_pos = a.items[k_start + gw + n_workers];
    }
    // counter-form SplitMix64 state of this lane's next draw:
    // s0 + (p*N + j + 1) * GAMMA with j = 32*ps + lane - 1
    auto rng_key = [&](int64_t pp) -> uint64_t {
        return (uint64_t)(a.pair_index ? a.pair_index[pp] : pp);
    };
    uint64_t rng_state = k_s0 + (rng_key(k_start + gw) * (uint64_t)N + (uint64_t)rr) * kGamma;
    // this lane's fixed 16-byte chunk and row-within-instruction
    constexpr int RPI = 32 / G::CH > 0 ? 32 / G::CH : 1;  // rows per copy instruction
    constexpr int NI = SR / RPI > 0 ? SR / RPI : 1;       // copy instructions per stage
    const int my_ch = lane % G::CH;
    const int my_rsub = lane / G::CH;

    // Issue stage g_next if it is below `limit`; the cp.async mover commits
    // one (possibly empty) group per call so wait_group<D-1> always targets
    // the stage being consumed.
    // query row of a pair: S[u], or the aggregated query h (trainer.py:148-173)
    auto qrow = [&](int64_t pp, int32_t uu_) -> const float * {
        return a.query ? a.query + (pp - k_start) * K : a.S + (int64_t)uu_ * K;
    };
    auto issue = [&](int64_t limit) {
        if (g_next >= limit) {
            if constexpr (!BULK) cp_async_commit();
            return;
        }
        const int r = ps * SR + rr;
        const bool valid = r <= N;
        uint32_t id = (uint32_t)pf_pos;
        if (r > 0) id = (uint32_t)fm.mod(mix64(rng_state));
        if (!valid) id = 0;
        if (lead) ids[pslot * SR + rr] = (int32_t)id;
        const int nvalid = min(SR, N + 1 - ps * SR);
        float *dst0 = ring + (size_t)pslot * SR * G::SLOTF;
        if constexpr (BULK) {
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                if (ps == 0) {
                    mbar_arrive_expect_tx(&ubars[pus], G::ROWB);
                    for (int h = 0; h < LPR; ++h)
                        bulk_g2s(urow + pus * G::SLOTF + h * G::SEGF, qrow(pf_p, pf_u) + h * G::HALF,
                                 G::ROWB / LPR, &ubars[pus]);
                }
                mbar_arrive_expect_tx(&bars[pslot], (uint32_t)(nvalid * G::ROWB));
            }
            __syncwarp();
            if (valid)
                bulk_g2s_hint(dst0 + rr * G::SLOTF + hs * G::SEGF,
                              a.T + (int64_t)id * K + hs * G::HALF, G::ROWB / LPR, &bars[pslot],
                              pol);
        } else {
            __syncwarp();
            float *dst = dst0 + my_rsub * G::SLOTF + G::pcol(my_ch * 4);
            const float *srcb = a.T + my_ch * 4;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int row = i * RPI + my_rsub;
                const uint32_t rid = __shfl_sync(0xffffffffu, id, (row * LPR) & 31);
                if (row < nvalid)
                    cp_async16_hint(dst + i * RPI * G::SLOTF, srcb + (size_t)rid * K, pol);
            }
            if (ps == 0) {
                const float *q = qrow(pf_p, pf_u);
                for (int ch = lane; ch < G::CH; ch += 32)
                    cp_async16(urow + pus * G::SLOTF + G::pcol(ch * 4), q + ch * 4);
            }
            cp_async_commit();
        }
        ++g_next;
        rng_state += (uint64_t)SR * kGamma;
        if (++pslot == D) pslot = 0;
        if (++ps == nb) {  // next pair of this worker
            ps = 0;
            ++pt;
            if (++pus == Lo.ucap) pus = 0;
            pf_u = nx_u;
            pf_pos = nx_pos;
            const int64_t pn = k_start + gw + pt * n_workers;
            pf_p = pn;
            if (pt < my_pairs)
                rng_state = k_s0 + (rng_key(pn) * (uint64_t)N + (uint64_t)rr) * kGamma;
            if (pt + 1 < my_pairs) {
                nx_u = a.users[pn + n_workers];
                nx_pos = a.items[pn + n_workers];
            }
        }
    };

    if (cross)
        for (int i = 0; i < D; ++i) issue(g_total);

    double loss = 0.0;
    long long degen = 0, active = 0;

    int cslot = 0, cus = 0;  // consumer ring slot / user slot
    int64_t cgen = 0;        // consumer stage count (bulk mover parity)
    for (int64_t t = 0; t < my_pairs; ++t) {
        const int64_t p = k_start + gw + t * n_workers;
        const int64_t u = a.users[p];
        const int64_t limit = cross ? g_total : (t + 1) * nb;
        if (!cross)
            for (int i = 0; i < D; ++i) issue(limit);
        const int us = cus;
        if (++cus == Lo.ucap) cus = 0;
        const float *up = urow + us * G::SLOTF;
        float ug[VW];
#pragma unroll
        for (int i = 0; i < VW; ++i) ug[i] = 0.f;
        float uu[VW];
        double ss = 0.0, rs = 0.0;
        float rss = 0.f;
        double hinge = 0.0, sim_p = 0.0;
        int cnt = 0;

        int nsp = 0;  // rows of this pair parked in the global spill area
        // apply n written rows (values in rows_, scalars in ents_)
        auto apply = [&](const float *rows_, const WriteEntry *ents_, int n) {
            for (int e = 0; e < n; ++e) {
                const WriteEntry ent = ents_[e];
                const RowCoef co = row_coef(ent, ss, rs, a.lr, a.l2, a.cosine);
                float d[VW], vv[VW];
                if constexpr (VW == 4) {
                    const float4 v4 = *reinterpret_cast<const float4 *>(rows_ + e * K + lane * 4);
                    vv[0] = v4.x; vv[1] = v4.y; vv[2] = v4.z; vv[3] = v4.w;
                } else {
#pragma unroll
                    for (int i = 0; i < VW; ++i)
                        vv[i] = lane < G::ACT ? rows_[e * K + lane * VW + i] : 0.f;
                }
#pragma unroll
                for (int i = 0; i < VW; ++i) row_apply(co, uu[i], vv[i], d[i], ug[i]);
                if (!dmode) {
                    if (lane < G::ACT) red_add_vec<VW>(a.T + (int64_t)ent.id * K + lane * VW, d);
                } else {
                    long long sl = 0;
                    if (lane == 0)
                        sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                    sl = __shfl_sync(0xffffffffu, sl, 0);
                    if (sl < a.delta_capacity) {
                        if (lane == 0) a.delta_ids[sl] = ent.id;
                        if (lane < G::ACT) {
#pragma unroll
                            for (int i = 0; i < VW; ++i) a.delta_rows[sl * K + lane * VW + i] = d[i];
                        }
                    }
                }
            }
        };
        // end of the pair: every row has been read, so all writes go now
        auto flush = [&]() {
            __syncwarp();
            if (nsp) apply(sp_rows, sp_ents, nsp);
            apply(snap, ents, cnt);
            cnt = 0;
            nsp = 0;
            __syncwarp();
        };
        // the snapshot is full mid-pair: park it in global memory (writes must
        // wait until the pair's last row is read, trainer.py:118-146 — a later
        // stage can hold the same row again); without a spill area, apply
        auto spill = [&]() {
            __syncwarp();
            if (sp_rows && nsp + cnt <= a.spill_cap) {
                const float4 *src4 = reinterpret_cast<const float4 *>(snap);
                float4 *dst4 = reinterpret_cast<float4 *>(sp_rows + (size_t)nsp * K);
                for (int x = lane; x < cnt * (K / 4); x += 32) dst4[x] = src4[x];
                for (int e = lane; e < cnt; e += 32) sp_ents[nsp + e] = ents[e];
                nsp += cnt;
            } else {
                apply(snap, ents, cnt);
            }
            cnt = 0;
            __syncwarp();
        };

        for (int s = 0; s < nb; ++s) {
            const int slot = cslot;
            if (++cslot == D) cslot = 0;
            if constexpr (BULK) {
                if (s == 0) mbar_wait(&ubars[us], (uint32_t)((t / Lo.ucap) & 1));
                mbar_wait(&bars[slot], (uint32_t)((cgen / D) & 1));
                ++cgen;
            } else {
                cp_async_wait<D - 1>();
                __syncwarp();
            }
            if (s == 0) {
                // ss = u.u (trainer.py:176-178), once the user row has landed
                float sp = 0.f;
                double spd = 0.0;
#pragma unroll
                for (int i = 0; i < VW; ++i) {
                    uu[i] = lane < G::ACT ? up[G::pcol(lane * VW + i)] : 0.f;
                    sp = fmaf(uu[i], uu[i], sp);
                    spd += (double)uu[i] * (double)uu[i];
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) {
                    sp += __shfl_xor_sync(0xffffffffu, sp, o);
                    spd += __shfl_xor_sync(0xffffffffu, spd, o);
                }
                ss = F64 ? spd : (double)sp;
                rs = ss > 0.0 ? sqrt(ss) : 0.0;
                rss = ss > 0.0 ? rsqrtf((float)ss) : 0.f;
                if constexpr (UREG) {  // this lane's user-row segment, once per pair
                    const float *uph0 = up + hs * G::SEGF;
#pragma unroll
                    for (int k = 0; k < G::HALF; k += 4) {
                        const float4 w4 = *reinterpret_cast<const float4 *>(uph0 + k);
                        ureg[k / 2] = make_float2(w4.x, w4.y);
                        ureg[k / 2 + 1] = make_float2(w4.z, w4.w);
                    }
                }
            }
            const int r = s * SR + rr;
            const bool valid = r <= N;
            const float *row = ring + ((size_t)slot * SR + rr) * G::SLOTF + hs * G::SEGF;
            const float *uph = up + hs * G::SEGF;
            double tt = 0.0, st = 0.0;
            if (valid) {
                if constexpr (F64) {
                    double t0 = 0, t1 = 0, s0 = 0, s1 = 0;
#pragma unroll
                    for (int k = 0; k < G::HALF; k += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(row + k);
                        const float4 w4 = *reinterpret_cast<const float4 *>(uph + k);
                        t0 = fma((double)v.x, (double)v.x, t0);
                        t1 = fma((double)v.y, (double)v.y, t1);
                        t0 = fma((double)v.z, (double)v.z, t0);
                        t1 = fma((double)v.w, (double)v.w, t1);
                        s0 = fma((double)w4.x, (double)v.x, s0);
                        s1 = fma((double)w4.y, (double)v.y, s1);
                        s0 = fma((double)w4.z, (double)v.z, s0);
                        s1 = fma((double)w4.w, (double)v.w, s1);
                    }
                    tt = t0 + t1;
                    st = s0 + s1;
                } else {
                    // packed fp32x2 FMA (FFMA2, sm_100); with UREG the user
                    // segment is in registers and only the row is read from
                    // shared memory
                    float2 ta = make_float2(0.f, 0.f), tb = ta, sa = ta, sb = ta;
                    float2 tc = ta, td = ta, sc2 = ta, sd = ta;  // second chain set
#pragma unroll
                    for (int k = 0; k < G::HALF; k += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(row + k);
                        float2 wlo, whi;
                        if constexpr (UREG) {
                            wlo = ureg[k / 2];
                            whi = ureg[k / 2 + 1];
                        } else {
                            const float4 w4 = *reinterpret_cast<const float4 *>(uph + k);
                            wlo = make_float2(w4.x, w4.y);
                            whi = make_float2(w4.z, w4.w);
                        }
                        const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
                        if ((k / 4) & 1) {
                            tc = __ffma2_rn(vlo, vlo, tc);
                            td = __ffma2_rn(vhi, vhi, td);
                            sc2 = __ffma2_rn(wlo, vlo, sc2);
                            sd = __ffma2_rn(whi, vhi, sd);
                        } else {
                            ta = __ffma2_rn(vlo, vlo, ta);
                            tb = __ffma2_rn(vhi, vhi, tb);
                            sa = __ffma2_rn(wlo, vlo, sa);
                            sb = __ffma2_rn(whi, vhi, sb);
                        }
                    }
                    tt = (double)(((ta.x + ta.y) + (tb.x + tb.y)) + ((tc.x + tc.y) + (td.x + td.y)));
                    st = (double)(((sa.x + sa.y) + (sb.x + sb.y)) + ((sc2.x + sc2.y) + (sd.x + sd.y)));
                }
            }
            if constexpr (LPR == 2) {  // the row's two column segments
                if constexpr (F64) {
                    tt += __shfl_xor_sync(0xffffffffu, tt, 1);
                    st += __shfl_xor_sync(0xffffffffu, st, 1);
                } else {
                    float tf = (float)tt, sf2 = (float)st;
                    tf += __shfl_xor_sync(0xffffffffu, tf, 1);
                    sf2 += __shfl_xor_sync(0xffffffffu, sf2, 1);
                    tt = (double)tf;
                    st = (double)sf2;
                }
            }
            // similarity and loss weight (trainer.py:184-221).  fp32 screen; the
            // binary64 value only for rows that can cross the margin.
            // fp32 dots: screen, then the reference's binary64 sums for the
            // rows that can reach the margin (heat_row_update.cuh)
            bool band = false;
            float sf = 0.f;
            double ssx = ss;
            if constexpr (!F64) {
                band = valid && margin_band(r, a.cosine, (float)ss, (float)tt, (float)st, rss,
                                            theta_f, &sf);
                for (unsigned mb = __ballot_sync(0xffffffffu, band && lead), first = 1; mb;
                     first = 0) {
                    const int src = __ffs(mb) - 1;
                    mb &= mb - 1;
                    double s_, t_, c_;
                    warp_dots64<K>(up, ring + ((size_t)slot * SR + src / LPR) * G::SLOTF,
                                   [](int k) { return G::pcol(k); }, first != 0, s_, t_, c_);
                    if (first) ssx = s_;
                    if (lane / LPR == src / LPR) {
                        tt = t_;
                        st = c_;
                    }
                }
                if (!band) ssx = ss;
            }
            bool write = false;
            double w = 0.0;
            if (valid) {
                bool degenerate = false;
                double sim = st;
                if (a.cosine) {
                    if (F64 || band) {
                        if (ssx <= 0.0 || tt <= 0.0) {
                            degenerate = true;
                            sim = 0.0;
                        } else {
                            sim = st / (sqrt(ssx) * sqrt(tt));
                        }
                    } else {
                        sim = (double)sf;
                    }
                    if (degenerate && lead) ++degen;
                } else if (!F64 && !band) {
                    sim = (double)sf;
                }
                if (r == 0) {
                    sim_p = sim;
                    w = -1.0;
                    write = !(a.cosine && degenerate) || a.l2 != 0.f;
                } else {
                    if (sim - a.theta > 0.0) {
                        if (lead) hinge += sim - a.theta;
                        w = wneg;
                        if (w != 0.0 && lead) ++active;
                    }
                    write = (w != 0.0 && !(a.cosine && degenerate)) || (w == 0.0 && a.l2 != 0.f);
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, write && lead);
            while (m) {
                if (cnt == Lo.snap_cap) spill();
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const float *srow = ring + ((size_t)slot * SR + src / LPR) * G::SLOTF;
                if (lane < G::ACT) {
#pragma unroll
                    for (int i = 0; i < VW; ++i)
                        snap[cnt * K + lane * VW + i] = srow[G::pcol(lane * VW + i)];
                }
                if (lane == src) ents[cnt] = WriteEntry{tt, st, w, ids[slot * SR + src / LPR], 0};
                ++cnt;
            }
            __syncwarp();
            issue(limit);  // refill this slot with the stage D ahead
        }
        flush();
        // user row (trainer.py:291-293): S[u] -= lr * (ugrad + l2 * S[u]); with
        // aggregation the gamma-scaled chain (trainer.py:301-302) and the
        // gradient kept for the weight update
        if (lane < G::ACT) {
            float d[VW];
            if (a.query) {
                float sv[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) sv[i] = 0.f;
                if (a.l2 != 0.f) {
#pragma unroll
                    for (int i = 0; i < VW; ++i) sv[i] = a.S[u * K + lane * VW + i];
                }
                float *go = a.ugrad_out + (p - k_start) * K + lane * VW;
#pragma unroll
                for (int i = 0; i < VW; ++i) {
                    d[i] = -a.lr * (a.ugamma * ug[i] + a.l2 * sv[i]);
                    go[i] = ug[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < VW; ++i) d[i] = -a.lr * (ug[i] + a.l2 * uu[i]);
            }
            red_add_vec<VW>(a.S + u * K + lane * VW, d);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) hinge += __shfl_xor_sync(0xffffffffu, hinge, o);
        sim_p = __shfl_sync(0xffffffffu, sim_p, 0);
        if (lane == 0) loss += (1.0 - sim_p) + wneg * hinge;
    }
    if constexpr (!BULK) cp_async_wait<0>();
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(0xffffffffu, degen, o);
        active += __shfl_xor_sync(0xffffffffu, active, o);
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)my_pairs);
    }
}

template <int K, int D, bool F64, bool BULK, int LPR>
static cudaError_t launch_staged_k(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                   int cross) {
    int snap_cap = K <= 64 ? 16 : 8;
    if (const char *e = getenv("HEAT_SNAP")) snap_cap = atoi(e) > 0 ? atoi(e) : snap_cap;
    const StLayout L = st_layout<K, D, LPR>(snap_cap);
    if (L.total > 200 * 1024) return cudaErrorInvalidValue;
    auto kern = a.range_dev ? hogwild_staged<K, D, F64, BULK, LPR, true>
                            : hogwild_staged<K, D, F64, BULK, LPR, false>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32, L.total, &e);
    if (e != cudaSuccess) return e;
    const int nb = (a.N + 1 + StGeom<K, LPR>::SR - 1) / StGeom<K, LPR>::SR;
    const int pif = cross ? 1 + (D - 1 + nb - 1) / nb : 1;  // pairs in flight per worker
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0) nw = std::min<int64_t>(nw, std::max<int64_t>(1, a.window / pif));
    if (a.window > 0 && a.window < pif) cross = 0;  // a lone pair: never prefetch past it
    nw = std::min<int64_t>(nw, a.stop - a.start);
    if (workers_out) *workers_out = (int)nw;
    HogwildArgs b = a;
    // spill area: a pair writes at most N+1 rows (all of them when l2 != 0)
    if (a.N + 1 > snap_cap) {
        b.spill_cap = a.N + 1;
        b.spill_stride = ((int64_t)b.spill_cap * (K * sizeof(float) + sizeof(WriteEntry)) + 255) &
                         ~(int64_t)255;
        b.spill = static_cast<unsigned char *>(stream_scratch(1, (size_t)(b.spill_stride * nw), st));
        if (!b.spill) b.spill_cap = 0;  // no memory: mid-pair application (documented)
    }
    kern<<<(unsigned)nw, 32, L.total, st>>>(b, FastMod::make((uint64_t)a.num_items), (int)nw,
                                            snap_cap, cross);
    return cudaGetLastError();
}

template <int K, bool F64>
static cudaError_t launch_staged_d(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                   int D, int cross, bool bulk, int lpr) {
    if constexpr (K >= 64) {
        if (lpr == 2) {
            if (bulk) return launch_staged_k<K, 2, F64, true, 2>(a, st, workers_out, cross);
            switch (D) {
            case 1: return launch_staged_k<K, 1, F64, false, 2>(a, st, workers_out, cross);
            case 2: return launch_staged_k<K, 2, F64, false, 2>(a, st, workers_out, cross);
            case 4: return launch_staged_k<K, 4, F64, false, 2>(a, st, workers_out, cross);
            case 6: return launch_staged_k<K, 6, F64, false, 2>(a, st, workers_out, cross);
            default: return launch_staged_k<K, 3, F64, false, 2>(a, st, workers_out, cross);
            }
        }
    }
    if (bulk) return launch_staged_k<K, 2, F64, true, 1>(a, st, workers_out, cross);
    switch (D) {
    case 1: return launch_staged_k<K, 1, F64, false, 1>(a, st, workers_out, cross);
    case 2: return launch_staged_k<K, 2, F64, false, 1>(a, st, workers_out, cross);
    case 4: return launch_staged_k<K, 4, F64, false, 1>(a, st, workers_out, cross);
    case 6: return launch_staged_k<K, 6, F64, false, 1>(a, st, workers_out, cross);
    default: return launch_staged_k<K, 3, F64, false, 1>(a, st, workers_out, cross);
    }
}

cudaError_t launch_hogwild_staged(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                  bool bulk) {
    // stages in flight per warp: enough rows in flight to cover L2 latency,
    // few enough that the window's workers fit on the SMs
    // measured, K = 128 (two lanes per row): with L2-resident tables one stage
    // in flight per warp wins (15 warps per SM hide the latency; c4 +12 %);
    // when the tables live in HBM two stages win (full-size c5: 12.85 M vs
    // 10.90 M samples/s): the rows in flight, not the warps, bound it there
    const double footprint = (double)(a.num_items + a.s_rows) * a.K * sizeof(float);
    int D = a.K <= 32 ? 4 : (a.K >= 128 && footprint < 96e6 ? 1 : 2);
    if (const char *e = getenv("HEAT_STAGES")) D = atoi(e) > 0 ? atoi(e) : D;
    // cross-pair prefetch halves the workers a window allows; measured slower
    int cross = 0;
    if (const char *e = getenv("HEAT_CROSS")) cross = atoi(e);
    // lanes per row: 2 for K = 128 (more warps per SM at the same rows in
    // flight; measured c4 +5 %); at K = 64 the doubled per-stage overhead
    // outweighs it (c3 -30 %)
    int lpr = a.K >= 128 ? 2 : 1;
    if (const char *e = getenv("HEAT_LPR")) lpr = atoi(e) == 2 ? 2 : 1;
    switch (a.K) {
    case 16: return a.fp64 ? launch_staged_d<16, true>(a, st, workers_out, D, cross, bulk, lpr)
                           : launch_staged_d<16, false>(a, st, workers_out, D, cross, bulk, lpr);
    case 32: return a.fp64 ? launch_staged_d<32, true>(a, st, workers_out, D, cross, bulk, lpr)
                           : launch_staged_d<32, false>(a, st, workers_out, D, cross, bulk, lpr);
    case 64: return a.fp64 ? launch_staged_d<64, true>(a, st, workers_out, D, cross, bulk, lpr)
                           : launch_staged_d<64, false>(a, st, workers_out, D, cross, bulk, lpr);
    case 128: return a.fp64 ? launch_staged_d<128, true>(a, st, workers_out, D, cross, bulk, lpr)
                            : launch_staged_d<128, false>(a, st, workers_out, D, cross, bulk, lpr);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace heat
