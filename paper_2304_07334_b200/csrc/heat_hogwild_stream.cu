// heat_hogwild_stream.cu — the throughput SGD kernel for wide pairs
// (K = 64/128, hundreds of negatives: configs 3-5), register-streamed.
//
// Same math and semantics as the other throughput kernels (trainer.py:114-293
// per pair, Hogwild across pairs).  What differs is the data path.  A pair
// reads N+2 rows and writes ~1 + A of them, so the kernel is a gather of
// ~4K(N+2) bytes per pair from L2 (c3/c4: tables L2-resident) or HBM (c5).
// Staging those rows in shared memory (LDGSTS or TMA, then LDS) moves every
// byte through the SM's 128 B/clk shared-memory port twice, which caps a
// staged kernel at the same ~64 B/clk/SM the L2 can feed.  Here the rows go
// straight from L2 into registers:
//
//  * one warp per pair-worker; a row of K floats is read by 8 lanes
//    (K/8 columns each, LDG.128 of 128 contiguous bytes per 8 lanes), so one
//    warp instruction covers a GROUP of 4 rows and every L2 sector is used
//    whole;
//  * a register ring of P groups: group i+P's loads are issued as soon as
//    group i has been consumed, so each warp keeps 4P rows in flight with no
//    shared memory at all (c4: P = 4, 16 rows = 8 KB per warp);
//  * tt = v.v and st = u.v per lane with packed FFMA2, then a transposed
//    8-lane butterfly (4 shuffles per group of 4 rows): lanes 0-3 of a row
//    reduce tt while lanes 4-7 reduce st;
//  * the similarity screen is fp32 (error < 1e-6 for K <= 128; the band is
//    1e-5).  Rows that may be written — every candidate for sim > theta, the
//    positive, rows whose fp32 v.v underflows, decay rows when l2 != 0 — are
//    only RECORDED (id + flags) while streaming, so no row data is held past
//    its FFMA2s;
//  * after the pair's last round the recorded rows are re-read into a per-warp
//    shared-memory snapshot (a per-worker global spill area past its
//    capacity), and the band rows get tt and st in binary64 (warp-cooperative
//    sums; the user's u.u is the reference's sequential binary64 sum), so the
//    margin decisions are binary64 decisions (trainer.py:184-221), not fp32
//    ones.  Then every write is applied (red.global.add.v4, or logged in DELTA
//    mode) — all reads of a pair precede its writes, the reference's snapshot
//    semantics (trainer.py:118-146, 257-293);
//  * workers claim pairs from a per-launch atomic counter in epoch order, so
//    SMs that host fewer workers take more pairs (no tail from the uneven
//    window / 148 split).  Pairs in flight never exceed the worker count,
//    which the launcher caps at the window.
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 0, but the compiler cannot tell: ties a load's address to a value so the
// load is not hoisted above the arithmetic that frees its target registers
__device__ __forceinline__ int32_t opaque_zero(float v) {
    int32_t z;
    asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(__float_as_uint(v)));
    return z;
}

__device__ __forceinline__ float4 ld_row4(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// Per (device, stream) pair-claim counters: [0] next pair, [1] finished
// warps.  Zeroed once at allocation; the last warp of every launch re-arms
// them, so graph replays need no memset node.
unsigned long long *stream_claim(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t>, unsigned long long *> ctrs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto &p = ctrs[std::make_tuple(dev, st)];
    if (!p) {
        if (cudaMalloc(&p, 2 * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return nullptr;
        }
        cudaMemsetAsync(p, 0, 2 * sizeof(unsigned long long), st);
    }
    return p;
}

}  // namespace

// sum_k a[k]*b[k] over K floats widened to binary64, one k at a time, never
// contracted (trainer.py:177-178, 181-183, 195-197): the reference's value
template <int K>
__device__ __forceinline__ double seq_dot(const float *a, const float *b) {
    double acc = 0.0;
#pragma unroll 2
    for (int k = 0; k < K; k += 4) {
        const float4 x = *reinterpret_cast<const float4 *>(a + k);
        const float4 y = *reinterpret_cast<const float4 *>(b + k);
        acc = __dadd_rn(acc, __dmul_rn((double)x.x, (double)y.x));
        acc = __dadd_rn(acc, __dmul_rn((double)x.y, (double)y.y));
        acc = __dadd_rn(acc, __dmul_rn((double)x.z, (double)y.z));
        acc = __dadd_rn(acc, __dmul_rn((double)x.w, (double)y.w));
    }
    return acc;
}

template <int K, int MINB, bool DR>
__global__ void __launch_bounds__(32, MINB)
    hogwild_stream(HogwildArgs a, FastMod fm, int snap_cap, float band_lo,
                   unsigned long long *claim) {
    constexpr int V = K / 32;  // float4 per lane per row
    extern __shared__ __align__(16) unsigned char sm[];
    float *urow = reinterpret_cast<float *>(sm);  // K floats: the user row
    float *snap = urow + K;                       // snap_cap rows: the first written rows

    const int lane = threadIdx.x;
    const int g = lane >> 3;  // row slot of a group
    const int c = lane & 7;   // column chunk: columns 32j + 4c .. +3
    int64_t k_start = a.start, k_stop = a.stop;
    uint64_t k_s0 = a.s0;
    if constexpr (DR) {
        k_start = a.range_dev[0];
        k_stop = a.range_dev[1];
        k_s0 = *a.s0_dev;
    }
    const int64_t npairs = k_stop - k_start;
    const int N = a.N;
    const int niter = (N + 1 + 31) >> 5;  // 4 rounds of 8 rows per iteration
    const uint64_t pol = policy_evict_last();
    // per-worker global area: written-row entries, rows past the snapshot
    unsigned char *mine_area = a.spill + (size_t)blockIdx.x * a.spill_stride;
    float *sp_rows = reinterpret_cast<float *>(mine_area);
    WriteEntry *ents = reinterpret_cast<WriteEntry *>(mine_area + (size_t)a.spill_cap * K * 4);
    // (id, flags) of each recorded row, written while streaming (one 8-byte
    // store); the full entries are filled by the resolve
    int2 *recs = reinterpret_cast<int2 *>(ents + a.spill_cap);
    auto slot_row = [&](int e) -> float * {
        return e < snap_cap ? snap + (size_t)e * K : sp_rows + (size_t)(e - snap_cap) * K;
    };

    double loss = 0.0;
    int degen = 0, active = 0, npairs_mine = 0;

    auto claim_next = [&]() -> int64_t {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(claim, 1ull);
        return (int64_t)__shfl_sync(kFull, t, 0);
    };

    // the next pair is claimed and its (user, item, RNG key) fetched one pair
    // ahead, so a pair starts without a chain of dependent global reads
    // (atomic -> ids -> rows).  Only read-only inputs are prefetched: table
    // rows are read when the pair starts.
    struct Next { int64_t t; int32_t u, pos; uint64_t pg; };
    auto fetch = [&](int64_t tt) -> Next {
        Next n{tt, 0, 0, 0};
        if (tt < npairs) {
            const int64_t pp = k_start + tt;
            n.u = a.users[pp];
            n.pos = a.items[pp];
            n.pg = a.pair_index ? (uint64_t)a.pair_index[pp] : (uint64_t)pp;
        }
        return n;
    };
    Next nx = fetch(claim_next());
    while (nx.t < npairs) {
        const int32_t u = nx.u;
        const int32_t pos = nx.pos;
        const uint64_t pg = nx.pg;

        float4 uv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) uv[j] = ldcg4(a.S + (int64_t)u * K + 32 * j + 4 * c);

        // negative ids, 32 rows per draw block: lane l of block b holds the id
        // of row 32b + l; row r >= 1 is draw pg*N + r - 1 of the stream
        // (trainer.py:134-139): mix64(s0 + (pg*N + r) * GAMMA) mod rows.
        // Rows past N read row 0 (a harmless load) and are never recorded.
        uint64_t rstate = k_s0 + (pg * (uint64_t)N + (uint64_t)lane) * kGamma;
        auto draw = [&](int blk) -> int32_t {
            const int r = 32 * blk + lane;
            const int32_t id = (int32_t)fm.mod(mix64(rstate));
            return r == 0 ? pos : (r <= N ? id : 0);
        };
        int32_t idv = draw(0);

        // register ring: round rd (rows 8rd .. 8rd+7, two groups of 4) lives
        // in buffer rd & 1 and is loaded two rounds ahead
        float4 R[2][2][V];
        int32_t rid[2][2];
        // the row ids of round rd (rd & 3 selects them in idv) and the loads
        // of a round into buffer b, split so the id shuffles run ahead of the
        // arithmetic that frees the buffer
        auto round_ids = [&](int rd, int32_t (&ids)[2]) {
#pragma unroll
            for (int x = 0; x < 2; ++x)
                ids[x] = __shfl_sync(kFull, idv, ((rd & 3) << 3) + 4 * x + g);
        };
        auto load = [&](int b, const int32_t (&ids)[2], int32_t z) {
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                rid[b][x] = ids[x];
                const float *src = a.T + (int64_t)ids[x] * K + 4 * c + z;
#pragma unroll
                for (int j = 0; j < V; ++j) R[b][x][j] = ld_row4(src + 32 * j, pol);
            }
        };
        {
            int32_t ids[2];
            round_ids(0, ids);
            load(0, ids, 0);
            round_ids(1, ids);
            load(1, ids, 0);
        }
        nx = fetch(claim_next());

        // fp32 u.u for the screen; the exact binary64 ss (trainer.py:176-178)
        // is summed at the end of the pair, where the written rows are resolved
        float ssf;
        {
            float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                q0 = __ffma2_rn(make_float2(uv[j].x, uv[j].y), make_float2(uv[j].x, uv[j].y), q0);
                q1 = __ffma2_rn(make_float2(uv[j].z, uv[j].w), make_float2(uv[j].z, uv[j].w), q1);
            }
            ssf = (q0.x + q0.y) + (q1.x + q1.y);
            ssf += __shfl_xor_sync(kFull, ssf, 4);
            ssf += __shfl_xor_sync(kFull, ssf, 2);
            ssf += __shfl_xor_sync(kFull, ssf, 1);
        }
        // a query whose fp32 u.u is tiny or zero sends every row to the
        // binary64 resolve (the degenerate test of trainer.py:184, 203)
        const bool screen = ssf > 1e-30f;
        const float rss = screen ? rsqrt_approx(ssf) : 0.f;
        if (g == 0) {  // the user row: the rounds' u.v and the binary64 sums
#pragma unroll
            for (int j = 0; j < V; ++j) *reinterpret_cast<float4 *>(urow + 32 * j + 4 * c) = uv[j];
        }
        __syncwarp();
        // exact ss = u.u as trainer.py:176-178 sums it, while the first rows load
        const double ss = seq_dot<K>(urow, urow);
        const bool decay_all = a.l2 != 0.f;
        int cnt = 0;  // rows recorded for writing (same value in every lane)

        // one round: FFMA2 partials of its 8 rows, the buffer refilled two
        // rounds ahead as soon as they are consumed, then the reduction and
        // the fp32 screen.  Rows that may be written are only RECORDED here
        // (id + flags); the resolve below re-reads them, so no row data is
        // held past its FFMA2s.
        auto round = [&](int b, int rd, bool refill) {
            int32_t nids[2];
            if (refill) round_ids(rd + 2, nids);
            float2 tl[2], th[2], sl[2], sh[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) tl[x] = th[x] = sl[x] = sh[x] = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                // this lane's user columns, from shared memory (not held in
                // registers across the round: the ring needs them)
                const float4 w = *reinterpret_cast<const float4 *>(urow + 32 * j + 4 * c);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const float2 vlo = make_float2(R[b][x][j].x, R[b][x][j].y);
                    const float2 vhi = make_float2(R[b][x][j].z, R[b][x][j].w);
                    tl[x] = __ffma2_rn(vlo, vlo, tl[x]);
                    th[x] = __ffma2_rn(vhi, vhi, th[x]);
                    sl[x] = __ffma2_rn(make_float2(w.x, w.y), vlo, sl[x]);
                    sh[x] = __ffma2_rn(make_float2(w.z, w.w), vhi, sh[x]);
                }
            }
            const int32_t id0 = rid[b][0], id1 = rid[b][1];
            // refill only after every FFMA2 of the round consumed the buffer
            if (refill) load(b, nids, opaque_zero(th[1].x) + opaque_zero(sh[1].y));
            float q[4];  // tt(x=0), st(x=0), tt(x=1), st(x=1)
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                const float2 t2 = __fadd2_rn(tl[x], th[x]);
                const float2 s2 = __fadd2_rn(sl[x], sh[x]);
                q[2 * x] = t2.x + t2.y;
                q[2 * x + 1] = s2.x + s2.y;
            }
            // transposed butterfly over the row's 8 lanes: afterwards lane c
            // holds quantity (c >> 1) & 1 (tt, st) of group c >> 2
            const bool b2 = (c & 4) != 0, b1 = (c & 2) != 0;
            float k0 = b2 ? q[2] : q[0], k1 = b2 ? q[3] : q[1];
            const float s0 = b2 ? q[0] : q[2], s1 = b2 ? q[1] : q[3];
            k0 += __shfl_xor_sync(kFull, s0, 4);
            k1 += __shfl_xor_sync(kFull, s1, 4);
            float m = b1 ? k1 : k0;
            m += __shfl_xor_sync(kFull, b1 ? k0 : k1, 2);
            m += __shfl_xor_sync(kFull, m, 1);
            const float o = __shfl_xor_sync(kFull, m, 2);
            const float ttf = b1 ? o : m, stf = b1 ? m : o;
            // fp32 screen (lanes 0-3 decide for group 0, lanes 4-7 for group
            // 1).  Band rows — the positive, any row whose fp32 cosine is
            // within 1e-5 of theta or above (fp32 error < 1e-6 at K <= 128),
            // any row whose fp32 v.v underflows — are decided by the resolve
            // from binary64 sums; every other row cannot be active, so it is
            // written only as a decay row (l2 != 0).
            const int r = 8 * rd + (b2 ? 4 : 0) + g;
            const float sim32 = stf * rss * rsqrt_approx(ttf);
            const bool valid = r <= N;
            const bool band = valid & (!screen | (r == 0) | !(ttf > 1e-30f) | (sim32 > band_lo));
            const bool rec = band | (valid & decay_all);
            const unsigned mrec = __ballot_sync(kFull, rec & ((c & 3) == 0));
            if (rec & ((c & 3) == 0)) {
                const int idx = cnt + __popc(mrec & ((1u << lane) - 1u));
                recs[idx] = make_int2(b2 ? id1 : id0, band ? (r == 0 ? 3 : 1) : 0);
            }
            cnt += __popc(mrec);
        };

#pragma unroll 1
        for (int it = 0; it < niter; ++it) {
            const int rd = 4 * it;
            const bool more = it + 1 < niter;
            round(0, rd, true);
            round(1, rd + 1, true);
            rstate += 32ull * kGamma;  // rounds rd+4, rd+5 need the next block
            idv = draw(it + 1);
            round(0, rd + 2, more);
            round(1, rd + 3, more);
        }

        // resolve: re-read every recorded row into its snapshot slot (shared
        // memory, then the worker's spill rows; four rows per pass, one per
        // row slot g), then decide each band row from binary64 v.v and u.v
        // (warp-cooperative, heat_row_update.cuh) with the reference's
        // cosine, degenerate test, hinge and weight (trainer.py:184-227).  A
        // band row that is not written becomes a hole (id -1).  Every read
        // of the pair precedes every write.
        __syncwarp();
        const float irs = ss > 0.0 ? rsqrtf((float)ss) : 0.f;
        const double wneg = a.mu * (1.0 / (double)N);
        double hinge = 0.0, sim_p = 0.0;
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 4) {
            const int e = e0 + g;
            if (e < cnt) {
                float *dst = slot_row(e) + 4 * c;
                const float *src = a.T + (int64_t)recs[e].x * K + 4 * c;
#pragma unroll
                for (int j = 0; j < V; ++j)
                    *reinterpret_cast<float4 *>(dst + 32 * j) = ldcg4(src + 32 * j);
            }
        }
        __syncwarp();
#pragma unroll 1
        for (int e = 0; e < cnt; ++e) {
            const int2 rec = recs[e];
            if (!(rec.y & 1)) {  // a decay-only row: w = 0
                if (lane == 0) ents[e] = WriteEntry{0.0, 0.0, 0.0, rec.x, 0};
                continue;
            }
            double unused, tt, st;
            warp_dots64<K>(urow, slot_row(e), ContiguousCols{}, false, unused, tt, st);
            if (lane == 0) {
                const bool degenerate = ss <= 0.0 || tt <= 0.0;
                const double sim = degenerate ? 0.0 : st / (sqrt(ss) * sqrt(tt));
                if (degenerate) ++degen;
                double w = 0.0;
                bool write;
                if (rec.y & 2) {  // the positive
                    sim_p = sim;
                    w = -1.0;
                    write = !degenerate || a.l2 != 0.f;
                } else {
                    if (sim - a.theta > 0.0) {
                        hinge += sim - a.theta;
                        w = wneg;
                        if (w != 0.0) ++active;
                    }
                    write = (w != 0.0 && !degenerate) || (w == 0.0 && a.l2 != 0.f);
                }
                ents[e] = WriteEntry{tt, st, w, write ? rec.x : -1, 0};
            }
        }
        __syncwarp();

        float4 ug[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            ug[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            uv[j] = *reinterpret_cast<const float4 *>(urow + 32 * j + 4 * c);
        }
        // the writes, four rows at a time (trainer.py:236-251 user gradient,
        // 259-290 item update, cached scalars; fp32 coefficients)
        const bool dmode = a.delta_ids != nullptr;
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 4) {
            const int e = e0 + g;
            WriteEntry ent{};
            if (e < cnt) ent = ents[e];
            const bool ok = e < cnt && ent.id >= 0;
            float4 d[V];
            if (ok) {
                const RowCoef co = row_coef_f(ent, ss, irs, a.lr, a.l2, true);
                const float *row = slot_row(e);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const float4 v = *reinterpret_cast<const float4 *>(row + 32 * j + 4 * c);
                    row_apply(co, uv[j].x, v.x, d[j].x, ug[j].x);
                    row_apply(co, uv[j].y, v.y, d[j].y, ug[j].y);
                    row_apply(co, uv[j].z, v.z, d[j].z, ug[j].z);
                    row_apply(co, uv[j].w, v.w, d[j].w, ug[j].w);
                }
            }
            if (!dmode) {
                if (ok) {
                    float *dst = a.T + (int64_t)ent.id * K + 4 * c;
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        red_add4(dst + 32 * j, d[j].x, d[j].y, d[j].z, d[j].w);
                }
            } else {
                long long sl = 0;
                if (ok && c == 0) sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                sl = __shfl_sync(kFull, sl, g * 8);
                if (ok && sl < a.delta_capacity) {
                    if (c == 0) a.delta_ids[sl] = ent.id;
                    float *dst = a.delta_rows + sl * K + 4 * c;
#pragma unroll
                    for (int j = 0; j < V; ++j) *reinterpret_cast<float4 *>(dst + 32 * j) = d[j];
                }
            }
        }
        // user row (trainer.py:291-293): S[u] -= lr * (ugrad + l2 * S[u]),
        // the four row slots' partial gradients summed first
#pragma unroll
        for (int j = 0; j < V; ++j) {
#pragma unroll
            for (int o = 8; o <= 16; o <<= 1) {
                ug[j].x += __shfl_xor_sync(kFull, ug[j].x, o);
                ug[j].y += __shfl_xor_sync(kFull, ug[j].y, o);
                ug[j].z += __shfl_xor_sync(kFull, ug[j].z, o);
                ug[j].w += __shfl_xor_sync(kFull, ug[j].w, o);
            }
        }
        if (g == 0) {
#pragma unroll
            for (int j = 0; j < V; ++j)
                red_add4(a.S + (int64_t)u * K + 32 * j + 4 * c, -a.lr * (ug[j].x + a.l2 * uv[j].x),
                         -a.lr * (ug[j].y + a.l2 * uv[j].y), -a.lr * (ug[j].z + a.l2 * uv[j].z),
                         -a.lr * (ug[j].w + a.l2 * uv[j].w));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            hinge += __shfl_xor_sync(kFull, hinge, o);
            sim_p += __shfl_xor_sync(kFull, sim_p, o);  // one lane holds it
        }
        if (lane == 0) loss += (1.0 - sim_p) + wneg * hinge;
        ++npairs_mine;
        __syncwarp();
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(kFull, degen, o);
        active += __shfl_xor_sync(kFull, active, o);
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)npairs_mine);
        // re-arm the claim counter once every warp has made its last claim
        __threadfence();
        if (atomicAdd(claim + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
            claim[0] = 0;
            claim[1] = 0;
            __threadfence();
        }
    }
}

template <int K, int MINB>
static cudaError_t launch_stream_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    const int snap_cap = K <= 64 ? 16 : 8;
    const size_t smem = K * sizeof(float) + (size_t)snap_cap * K * sizeof(float);
    auto kern = a.range_dev ? hogwild_stream<K, MINB, true> : hogwild_stream<K, MINB, false>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32, smem, &e);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0) nw = std::min<int64_t>(nw, a.window);
    nw = std::min<int64_t>(nw, a.stop - a.start);
    if (nw < 1) return cudaSuccess;
    if (workers_out) *workers_out = (int)nw;
    HogwildArgs b = a;
    // spill area: a pair writes at most N+1 rows (all of them when l2 != 0)
    b.spill_cap = a.N + 1;
    b.spill_stride = ((int64_t)b.spill_cap * (K * sizeof(float) + sizeof(WriteEntry) + sizeof(int2)) + 255) &
                     ~(int64_t)255;
    b.spill = static_cast<unsigned char *>(stream_scratch(1, (size_t)(b.spill_stride * nw), st));
    unsigned long long *claim = stream_claim(st);
    if (!b.spill || !claim) return cudaErrorMemoryAllocation;
    kern<<<(unsigned)nw, 32, smem, st>>>(b, FastMod::make((uint64_t)a.num_items), snap_cap,
                                         (float)a.theta - 1e-5f, claim);
    return cudaGetLastError();
}

bool hogwild_stream_supported(const HogwildArgs &a) {
    return (a.K == 64 || a.K == 128) && !a.fp64 && a.cosine && !a.query &&
           ((uintptr_t)a.S % 16 == 0) && ((uintptr_t)a.T % 16 == 0);
}

cudaError_t launch_hogwild_stream(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    if (!hogwild_stream_supported(a)) return cudaErrorNotSupported;
    // resident warps per SM the register budget is compiled for
    int warps = 12;
    if (const char *e = getenv("HEAT_STREAM_WARPS")) warps = atoi(e) > 0 ? atoi(e) : warps;
    if (a.K == 128) {
        switch (warps) {
        case 8: return launch_stream_k<128, 8>(a, st, workers_out);
        case 16: return launch_stream_k<128, 16>(a, st, workers_out);
        default: return launch_stream_k<128, 12>(a, st, workers_out);
        }
    }
    switch (warps) {
    case 12: return launch_stream_k<64, 12>(a, st, workers_out);
    default: return launch_stream_k<64, 16>(a, st, workers_out);
    }
}

}  // namespace heat
