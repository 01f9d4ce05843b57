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
#include <type_traits>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

template <int K>
struct StGeom {
    static constexpr int ROWB = K * 4;               // bytes per row
    static constexpr int SLOTF = K + 4;              // floats per padded slot
    static constexpr int CH = K / 4;                 // 16-byte chunks per row
    static constexpr int VW = K >= 32 ? K / 32 : 1;  // floats per lane in row-wide ops
    static constexpr int ACT = K >= 32 ? 32 : K;     // lanes active in row-wide ops
};

struct StLayout {
    int ucap, snap_cap;
    size_t off_bars, off_ubars, off_ids, off_ring, off_urow, off_snap, off_ents, total;
};

template <int K, int D>
__host__ __device__ inline StLayout st_layout(int snap_cap) {
    using G = StGeom<K>;
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
    L.off_ids = take(sizeof(int32_t) * 32 * D);
    L.off_ring = take(sizeof(float) * G::SLOTF * 32 * D);
    L.off_urow = take(sizeof(float) * K * L.ucap);
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

template <int K, int D, bool F64, bool BULK>
__global__ void __launch_bounds__(32)
    hogwild_staged(HogwildArgs a, FastMod fm, int n_workers, int snap_cap, int cross) {
    using G = StGeom<K>;
    constexpr int VW = G::VW;
    extern __shared__ __align__(128) unsigned char sm[];
    const StLayout Lo = st_layout<K, D>(snap_cap);
    uint64_t *bars = reinterpret_cast<uint64_t *>(sm + Lo.off_bars);
    uint64_t *ubars = reinterpret_cast<uint64_t *>(sm + Lo.off_ubars);
    int32_t *ids = reinterpret_cast<int32_t *>(sm + Lo.off_ids);
    float *ring = reinterpret_cast<float *>(sm + Lo.off_ring);
    float *urow = reinterpret_cast<float *>(sm + Lo.off_urow);
    float *snap = reinterpret_cast<float *>(sm + Lo.off_snap);
    WriteEntry *ents = reinterpret_cast<WriteEntry *>(sm + Lo.off_ents);

    const int lane = threadIdx.x;
    const int gw = blockIdx.x;
    const int64_t npairs = a.stop - a.start;
    if (gw >= n_workers || gw >= npairs) return;
    const int64_t my_pairs = (npairs - gw + n_workers - 1) / n_workers;
    const int N = a.N;
    const int nb = (N + 1 + 31) / 32;  // stages per pair
    const int64_t g_total = my_pairs * nb;
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;
    const uint64_t pol = policy_evict_last();

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
    int32_t pf_u = a.users[a.start + gw];
    int32_t pf_pos = a.items[a.start + gw];
    int64_t pf_p = a.start + gw;  // pair whose user row the producer loads next
    int32_t nx_u = 0, nx_pos = 0;
    if (my_pairs > 1) {
        nx_u = a.users[a.start + gw + n_workers];
        nx_pos = a.items[a.start + gw + n_workers];
    }
    // counter-form SplitMix64 state of this lane's next draw:
    // s0 + (p*N + j + 1) * GAMMA with j = 32*ps + lane - 1
    auto rng_key = [&](int64_t pp) -> uint64_t {
        return (uint64_t)(a.pair_index ? a.pair_index[pp] : pp);
    };
    uint64_t rng_state = a.s0 + (rng_key(a.start + gw) * (uint64_t)N + (uint64_t)lane) * kGamma;
    // this lane's fixed 16-byte chunk and row-within-instruction
    constexpr int RPI = 32 / G::CH > 0 ? 32 / G::CH : 1;  // rows per copy instruction
    constexpr int NI = 32 / RPI;                          // copy instructions per stage
    const int my_ch = lane % G::CH;
    const int my_rsub = lane / G::CH;

    // Issue stage g_next if it is below `limit`; the cp.async mover commits
    // one (possibly empty) group per call so wait_group<D-1> always targets
    // the stage being consumed.
    // query row of a pair: S[u], or the aggregated query h (trainer.py:148-173)
    auto qrow = [&](int64_t pp, int32_t uu_) -> const float * {
        return a.query ? a.query + (pp - a.start) * K : a.S + (int64_t)uu_ * K;
    };
    auto issue = [&](int64_t limit) {
        if (g_next >= limit) {
            if constexpr (!BULK) cp_async_commit();
            return;
        }
        const int r = ps * 32 + lane;
        const bool valid = r <= N;
        uint32_t id = (uint32_t)pf_pos;
        if (r > 0) id = (uint32_t)fm.mod(mix64(rng_state));
        if (!valid) id = 0;
        ids[pslot * 32 + lane] = (int32_t)id;
        const int nvalid = min(32, N + 1 - ps * 32);
        float *dst0 = ring + (size_t)pslot * 32 * G::SLOTF;
        if constexpr (BULK) {
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                if (ps == 0) {
                    mbar_arrive_expect_tx(&ubars[pus], G::ROWB);
                    bulk_g2s(urow + pus * K, qrow(pf_p, pf_u), G::ROWB, &ubars[pus]);
                }
                mbar_arrive_expect_tx(&bars[pslot], (uint32_t)(nvalid * G::ROWB));
            }
            __syncwarp();
            if (valid)
                bulk_g2s_hint(dst0 + lane * G::SLOTF, a.T + (int64_t)id * K, G::ROWB, &bars[pslot],
                              pol);
        } else {
            __syncwarp();
            float *dst = dst0 + my_rsub * G::SLOTF + my_ch * 4;
            const float *srcb = a.T + my_ch * 4;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int row = i * RPI + my_rsub;
                const uint32_t rid = __shfl_sync(0xffffffffu, id, row & 31);
                if (row < nvalid)
                    cp_async16_hint(dst + i * RPI * G::SLOTF, srcb + (size_t)rid * K, pol);
            }
            if (ps == 0) {
                const float *q = qrow(pf_p, pf_u);
                for (int ch = lane; ch < G::CH; ch += 32)
                    cp_async16(urow + pus * K + ch * 4, q + ch * 4);
            }
            cp_async_commit();
        }
        ++g_next;
        rng_state += 32ull * kGamma;
        if (++pslot == D) pslot = 0;
        if (++ps == nb) {  // next pair of this worker
            ps = 0;
            ++pt;
            if (++pus == Lo.ucap) pus = 0;
            pf_u = nx_u;
            pf_pos = nx_pos;
            const int64_t pn = a.start + gw + pt * n_workers;
            pf_p = pn;
            if (pt < my_pairs)
                rng_state = a.s0 + (rng_key(pn) * (uint64_t)N + (uint64_t)lane) * kGamma;
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
        const int64_t p = a.start + gw + t * n_workers;
        const int64_t u = a.users[p];
        const int64_t limit = cross ? g_total : (t + 1) * nb;
        if (!cross)
            for (int i = 0; i < D; ++i) issue(limit);
        const int us = cus;
        if (++cus == Lo.ucap) cus = 0;
        const float *up = urow + us * K;
        float ug[VW];
#pragma unroll
        for (int i = 0; i < VW; ++i) ug[i] = 0.f;
        float uu[VW];
        double ss = 0.0, rs = 0.0;
        float rss = 0.f;
        double hinge = 0.0, sim_p = 0.0;
        int cnt = 0;

        auto flush = [&]() {
            __syncwarp();
            for (int e = 0; e < cnt; ++e) {
                const WriteEntry ent = ents[e];
                const RowCoef co = row_coef(ent, ss, rs, a.lr, a.l2, a.cosine);
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) {
                    const float v = lane < G::ACT ? snap[e * K + lane * VW + i] : 0.f;
                    row_apply(co, uu[i], v, d[i], ug[i]);
                }
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
                    uu[i] = lane < G::ACT ? up[lane * VW + i] : 0.f;
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
            }
            const int r = s * 32 + lane;
            const bool valid = r <= N;
            const float *row = ring + ((size_t)slot * 32 + lane) * G::SLOTF;
            double tt = 0.0, st = 0.0;
            if (valid) {
                if constexpr (F64) {
                    double t0 = 0, t1 = 0, s0 = 0, s1 = 0;
#pragma unroll
                    for (int k = 0; k < K; k += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(row + k);
                        const float4 w4 = *reinterpret_cast<const float4 *>(up + k);
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
                    // packed fp32x2 FMA (FFMA2, sm_100)
                    float2 ta = make_float2(0.f, 0.f), tb = ta, sa = ta, sb = ta;
#pragma unroll
                    for (int k = 0; k < K; k += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(row + k);
                        const float4 w4 = *reinterpret_cast<const float4 *>(up + k);
                        const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
                        ta = __ffma2_rn(vlo, vlo, ta);
                        tb = __ffma2_rn(vhi, vhi, tb);
                        sa = __ffma2_rn(make_float2(w4.x, w4.y), vlo, sa);
                        sb = __ffma2_rn(make_float2(w4.z, w4.w), vhi, sb);
                    }
                    tt = (double)((ta.x + ta.y) + (tb.x + tb.y));
                    st = (double)((sa.x + sa.y) + (sb.x + sb.y));
                }
            }
            // similarity and loss weight (trainer.py:184-221).  fp32 screen; the
            // binary64 value only for rows that can cross the margin.
            bool write = false;
            double w = 0.0;
            if (valid) {
                bool degenerate = false;
                double sim = st;
                if (a.cosine) {
                    if (ss <= 0.0 || tt <= 0.0) {
                        degenerate = true;
                        sim = 0.0;
                        ++degen;
                    } else {
                        const float sf = (float)st * rss * rsqrtf((float)tt);
                        sim = (double)sf;
                        if (F64 || (r > 0 && sf > theta_f - 1e-5f)) sim = st / (sqrt(ss) * sqrt(tt));
                    }
                }
                if (r == 0) {
                    sim_p = sim;
                    w = -1.0;
                    write = !(a.cosine && degenerate) || a.l2 != 0.f;
                } else {
                    if (sim - a.theta > 0.0) {
                        hinge += sim - a.theta;
                        w = wneg;
                        if (w != 0.0) ++active;
                    }
                    write = (w != 0.0 && !(a.cosine && degenerate)) || (w == 0.0 && a.l2 != 0.f);
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, write);
            while (m) {
                if (cnt == Lo.snap_cap) flush();
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const float *srow = ring + ((size_t)slot * 32 + src) * G::SLOTF;
                if (lane < G::ACT) {
#pragma unroll
                    for (int i = 0; i < VW; ++i) snap[cnt * K + lane * VW + i] = srow[lane * VW + i];
                }
                if (lane == src) ents[cnt] = WriteEntry{tt, st, w, ids[slot * 32 + src], 0};
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
                float *go = a.ugrad_out + (p - a.start) * K + lane * VW;
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

template <int K, int D, bool F64, bool BULK>
static cudaError_t launch_staged_k(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                   int cross) {
    const int snap_cap = K <= 64 ? 16 : 8;
    const StLayout L = st_layout<K, D>(snap_cap);
    if (L.total > 200 * 1024) return cudaErrorInvalidValue;
    auto kern = hogwild_staged<K, D, F64, BULK>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.total);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, L.total);
    if (per_sm < 1) per_sm = 1;
    const int nb = (a.N + 1 + 31) / 32;
    const int pif = cross ? 1 + (D - 1 + nb - 1) / nb : 1;  // pairs in flight per worker
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0) nw = std::min<int64_t>(nw, std::max<int64_t>(1, a.window / pif));
    if (a.window > 0 && a.window < pif) cross = 0;  // a lone pair: never prefetch past it
    nw = std::min<int64_t>(nw, a.stop - a.start);
    if (workers_out) *workers_out = (int)nw;
    kern<<<(unsigned)nw, 32, L.total, st>>>(a, FastMod::make((uint64_t)a.num_items), (int)nw,
                                            snap_cap, cross);
    return cudaGetLastError();
}

template <int K, bool F64>
static cudaError_t launch_staged_d(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                   int D, int cross, bool bulk) {
    if (bulk) return launch_staged_k<K, 2, F64, true>(a, st, workers_out, cross);
    switch (D) {
    case 2: return launch_staged_k<K, 2, F64, false>(a, st, workers_out, cross);
    case 4: return launch_staged_k<K, 4, F64, false>(a, st, workers_out, cross);
    case 6: return launch_staged_k<K, 6, F64, false>(a, st, workers_out, cross);
    default: return launch_staged_k<K, 3, F64, false>(a, st, workers_out, cross);
    }
}

cudaError_t launch_hogwild_staged(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                  bool bulk) {
    // stages in flight per warp: enough rows in flight to cover L2 latency,
    // few enough that the window's workers fit on the SMs
    int D = a.K <= 32 ? 4 : 2;
    if (const char *e = getenv("HEAT_STAGES")) D = atoi(e) > 0 ? atoi(e) : D;
    // cross-pair prefetch halves the workers a window allows; measured slower
    int cross = 0;
    if (const char *e = getenv("HEAT_CROSS")) cross = atoi(e);
    switch (a.K) {
    case 16: return a.fp64 ? launch_staged_d<16, true>(a, st, workers_out, D, cross, bulk)
                           : launch_staged_d<16, false>(a, st, workers_out, D, cross, bulk);
    case 32: return a.fp64 ? launch_staged_d<32, true>(a, st, workers_out, D, cross, bulk)
                           : launch_staged_d<32, false>(a, st, workers_out, D, cross, bulk);
    case 64: return a.fp64 ? launch_staged_d<64, true>(a, st, workers_out, D, cross, bulk)
                           : launch_staged_d<64, false>(a, st, workers_out, D, cross, bulk);
    case 128: return a.fp64 ? launch_staged_d<128, true>(a, st, workers_out, D, cross, bulk)
                            : launch_staged_d<128, false>(a, st, workers_out, D, cross, bulk);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace heat
