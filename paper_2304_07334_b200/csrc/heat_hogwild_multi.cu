// heat_hogwild_multi.cu — throughput SGD for large N with several warps per
// pair (config 3: K 64, N 500).
//
// With a window of B pairs in flight and one warp per pair (the staged
// kernel), an SM holds only B/148 warps: c3 at B = 1024 runs 7 warps per SM
// and stalls on fixed-latency dependencies (ncu: 10 % warps active, `wait`
// 42 %).  Here a CTA of NW warps serves one pair: warp w streams the pair's
// 32-row stages w, w+NW, ... through its own cp.async ring (lane per row,
// fp32 FFMA2 dots, fp32 similarity screen with the exact binary64 value near
// the margin), so the same B pairs keep NW times the warps busy.
//
// Semantics are the staged kernel's (trainer.py:114-293 per pair, Hogwild
// across pairs): written rows are snapshotted (spilled to global when the
// snapshot fills), a CTA barrier after the last stage of every warp orders
// all of the pair's reads before any of its writes, then each warp applies
// its own rows with red.global.add and adds its share of the user gradient.
#include <cstdint>
#include <cstdlib>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

// LPR lanes per row (2 for K = 128: 16-row stages, each lane half a row,
// half-row segments padded apart so a quarter-warp reads distinct banks)
template <int K, int LPR>
struct MwGeom {
    static constexpr int HALF = K / LPR;             // columns per lane segment
    static constexpr int SEGF = HALF + 4;            // padded segment (floats)
    static constexpr int SLOTF = LPR * SEGF;         // padded row slot (floats)
    static constexpr int SR = 32 / LPR;              // rows per stage
    static constexpr int CH = K / 4;                 // 16-byte chunks per row
    static constexpr int VW = K >= 32 ? K / 32 : 1;  // floats per lane in row-wide ops
    static constexpr int RPI = 32 / CH > 0 ? 32 / CH : 1;  // rows per copy instruction
    static constexpr int NI = SR / RPI > 0 ? SR / RPI : 1; // copy instructions per stage
    __host__ __device__ static constexpr int pcol(int c) { return c + (c / HALF) * 4; }
};

struct MwLayout {
    size_t ids, ring, urow, snap, ents, per_warp;
};

template <int K, int D, int LPR>
__host__ __device__ inline MwLayout mw_layout(int snap_cap) {
    using G = MwGeom<K, LPR>;
    MwLayout L;
    size_t o = 0;
    auto take = [&](size_t b) {
        size_t at = (o + 127) & ~size_t(127);
        o = at + b;
        return at;
    };
    L.ids = take(sizeof(int32_t) * G::SR * D);
    L.ring = take(sizeof(float) * G::SLOTF * G::SR * D);
    // (K floats when LPR = 1: the padding would cost c3 its fifth CTA per SM)
    L.urow = take(sizeof(float) * (LPR == 1 ? K : G::SLOTF));
    L.snap = take(sizeof(float) * K * snap_cap);
    L.ents = take(sizeof(WriteEntry) * snap_cap);
    L.per_warp = (o + 127) & ~size_t(127);
    return L;
}

#ifndef MULTI_UREG
#define MULTI_UREG 0  // measured: registers cost residency more than the LDS saved
#endif

#ifndef MULTI_MINB
#define MULTI_MINB 5  // measured: 5 CTAs (20 warps) per SM, registers <= 102
#endif

// SPLIT (opt-in, HEAT_MULTI_SPLIT=1): the "all reads before any write" point
// of a pair is an mbarrier that each warp arrives on as soon as its last
// stage has landed, instead of a CTA barrier after every warp's scoring.
// Unlike the resident kernel (+7 %), it measured slower here (c3 72.7 M vs
// 77.7 M samples/s): the warps' stage loops are equally long, so there is
// little barrier wait to hide, and the waiting warps poll.
// DR: the pair range and stream base come from HogwildArgs::range_dev/s0_dev
template <int K, int NW, int D, int LPR, bool SPLIT, bool DR>
__global__ void __launch_bounds__(32 * NW, MULTI_MINB)
    hogwild_multi(HogwildArgs a, FastMod fm, int n_workers, int snap_cap) {
    using G = MwGeom<K, LPR>;
    constexpr int VW = G::VW;
    constexpr int SR = G::SR;
    extern __shared__ __align__(128) unsigned char sm[];
    const MwLayout Lo = mw_layout<K, D, LPR>(snap_cap);
    const int lane = threadIdx.x & 31;
    const int rr = lane / LPR, hs = lane % LPR;  // my row in a stage, my column segment
    const bool lead = hs == 0;                   // the lane that accounts for the row
    const int w = threadIdx.x >> 5;
    unsigned char *mine = sm + (size_t)w * Lo.per_warp;
    int32_t *ids = reinterpret_cast<int32_t *>(mine + Lo.ids);
    float *ring = reinterpret_cast<float *>(mine + Lo.ring);
    float *urow = reinterpret_cast<float *>(mine + Lo.urow);
    float *snap = reinterpret_cast<float *>(mine + Lo.snap);
    WriteEntry *ents = reinterpret_cast<WriteEntry *>(mine + Lo.ents);

    const int gw = blockIdx.x;
    int64_t k_start = a.start, k_stop = a.stop;
    uint64_t k_s0 = a.s0;
    if constexpr (DR) {
        k_start = a.range_dev[0];
        k_stop = a.range_dev[1];
        k_s0 = *a.s0_dev;
    }
    const int64_t npairs = k_stop - k_start;
    if (gw >= n_workers || gw >= npairs) return;  // uniform per CTA
    __shared__ uint64_t reads_done;
    uint32_t phase = 0;
    if (SPLIT) {
        if (threadIdx.x == 0) mbar_init(&reads_done, NW);
        __syncthreads();
    }
    const int N = a.N;
    const int nb = (N + 1 + SR - 1) / SR;          // stages per pair
    const int nbw = nb > w ? (nb - w + NW - 1) / NW : 0;  // this warp's stages
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;
    const uint64_t pol = policy_evict_last();
    const int my_ch = lane % G::CH, my_rsub = lane / G::CH;
    const size_t spill_id = (size_t)gw * NW + w;
    float *sp_rows = a.spill ? reinterpret_cast<float *>(a.spill + spill_id * a.spill_stride)
                             : nullptr;
    WriteEntry *sp_ents =
        a.spill ? reinterpret_cast<WriteEntry *>(a.spill + spill_id * a.spill_stride +
                                                 (size_t)a.spill_cap * K * sizeof(float))
                : nullptr;

    double loss = 0.0;
    long long degen = 0, active = 0;
    for (int64_t p = k_start + gw; p < k_stop; p += n_workers) {
        const int64_t u = a.users[p];
        const int32_t pos = a.items[p];
        const uint64_t key = (uint64_t)(a.pair_index ? a.pair_index[p] : p);
        // ---- producer: stage i of this warp is the pair's stage w + NW*i
        int issued = 0;
        auto issue = [&]() {
            if (issued >= nbw) {
                cp_async_commit();  // keep one group per call
                return;
            }
            const int s = w + NW * issued;
            const int slot = issued % D;
            const int r = s * SR + rr;
            uint32_t id = (uint32_t)pos;
            if (r > 0 && r <= N)
                id = (uint32_t)fm.mod(mix64(k_s0 + (key * (uint64_t)N + (uint64_t)r) * kGamma));
            if (r > N) id = 0;
            if (lead) ids[slot * SR + rr] = (int32_t)id;
            const int nvalid = min(SR, N + 1 - s * SR);
            float *dst = ring + (size_t)slot * SR * G::SLOTF + my_rsub * G::SLOTF +
                         G::pcol(my_ch * 4);
            const float *srcb = a.T + my_ch * 4;
#pragma unroll
            for (int i = 0; i < G::NI; ++i) {
                const int row = i * G::RPI + my_rsub;
                const uint32_t rid = __shfl_sync(0xffffffffu, id, (row * LPR) & 31);
                if (row < nvalid)
                    cp_async16_hint(dst + i * G::RPI * G::SLOTF, srcb + (size_t)rid * K, pol);
            }
            if (issued == 0)  // the user row rides with the warp's first stage
                for (int ch = lane; ch < G::CH; ch += 32)
                    cp_async16(urow + G::pcol(ch * 4), a.S + u * K + ch * 4);
            cp_async_commit();
            ++issued;
        };
        for (int i = 0; i < D; ++i) issue();
        if (SPLIT && nbw == 0 && lane == 0) mbar_arrive(&reads_done);

        float ug[VW], uu[VW];
#pragma unroll
        for (int i = 0; i < VW; ++i) ug[i] = uu[i] = 0.f;
        constexpr bool UREG = MULTI_UREG != 0;  // user row in registers (else broadcast LDS)
        float2 ureg[UREG ? G::HALF / 2 : 1];
        double ss = 0.0, rs = 0.0;
        float rss = 0.f;
        double hinge = 0.0, sim_p = 0.0;
        int cnt = 0, nsp = 0;

        auto apply = [&](const float *rows_, const WriteEntry *ents_, int n) {
            for (int e = 0; e < n; ++e) {
                const WriteEntry ent = ents_[e];
                const RowCoef co = row_coef(ent, ss, rs, a.lr, a.l2, a.cosine);
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i)
                    row_apply(co, uu[i], rows_[e * K + lane * VW + i], d[i], ug[i]);
                if (!dmode) {
                    if constexpr (VW == 2) {
                        red_add2(a.T + (int64_t)ent.id * K + lane * 2, d[0], d[1]);
                    } else if constexpr (VW == 4) {
                        red_add4(a.T + (int64_t)ent.id * K + lane * 4, d[0], d[1], d[2], d[3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < VW; ++i)
                            atomicAdd(a.T + (int64_t)ent.id * K + lane * VW + i, d[i]);
                    }
                } else {
                    long long sl = 0;
                    if (lane == 0)
                        sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                    sl = __shfl_sync(0xffffffffu, sl, 0);
                    if (sl < a.delta_capacity) {
                        if (lane == 0) a.delta_ids[sl] = ent.id;
#pragma unroll
                        for (int i = 0; i < VW; ++i) a.delta_rows[sl * K + lane * VW + i] = d[i];
                    }
                }
            }
        };
        auto spill = [&]() {  // snapshot full mid-pair: park it until the pair's last read
            __syncwarp();
            if (sp_rows && nsp + cnt <= a.spill_cap) {
                const float4 *s4 = reinterpret_cast<const float4 *>(snap);
                float4 *d4 = reinterpret_cast<float4 *>(sp_rows + (size_t)nsp * K);
                for (int x = lane; x < cnt * (K / 4); x += 32) d4[x] = s4[x];
                for (int e = lane; e < cnt; e += 32) sp_ents[nsp + e] = ents[e];
                nsp += cnt;
            } else {
                apply(snap, ents, cnt);
            }
            cnt = 0;
            __syncwarp();
        };

        for (int i = 0; i < nbw; ++i) {
            cp_async_wait<D - 1>();
            __syncwarp();
            // the last stage has landed (the groups after it are empty): this
            // warp's reads of the pair are complete
            if (SPLIT && i == nbw - 1 && lane == 0) mbar_arrive(&reads_done);
            const int s = w + NW * i;
            const int slot = i % D;
            if (i == 0) {  // ss = u.u (trainer.py:176-178) once the user row landed
                float sp = 0.f;
#pragma unroll
                for (int v = 0; v < VW; ++v) {
                    uu[v] = urow[G::pcol(lane * VW + v)];
                    sp = fmaf(uu[v], uu[v], sp);
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
                ss = (double)sp;
                rs = ss > 0.0 ? sqrt(ss) : 0.0;
                rss = ss > 0.0 ? rsqrtf(sp) : 0.f;
                if constexpr (UREG) {
#pragma unroll
                    for (int k = 0; k < G::HALF; k += 4) {
                        const float4 w4 = *reinterpret_cast<const float4 *>(urow + hs * G::SEGF + k);
                        ureg[k / 2] = make_float2(w4.x, w4.y);
                        ureg[k / 2 + 1] = make_float2(w4.z, w4.w);
                    }
                }
            }
            const int r = s * SR + rr;
            const bool valid = r <= N;
            const float *row = ring + ((size_t)slot * SR + rr) * G::SLOTF + hs * G::SEGF;
            const float *uph = urow + hs * G::SEGF;
            float2 ta = make_float2(0.f, 0.f), tb = ta, sa = ta, sb = ta;
            float2 tc = ta, td = ta, sc = ta, sd = ta;
            if (valid) {
#pragma unroll
                for (int k = 0; k < G::HALF; k += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(row + k);
                    const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
                    float2 wlo, whi;
                    if constexpr (UREG) {
                        wlo = ureg[k / 2];
                        whi = ureg[k / 2 + 1];
                    } else {
                        const float4 w4 = *reinterpret_cast<const float4 *>(uph + k);
                        wlo = make_float2(w4.x, w4.y);
                        whi = make_float2(w4.z, w4.w);
                    }
                    if ((k / 4) & 1) {
                        tc = __ffma2_rn(vlo, vlo, tc);
                        td = __ffma2_rn(vhi, vhi, td);
                        sc = __ffma2_rn(wlo, vlo, sc);
                        sd = __ffma2_rn(whi, vhi, sd);
                    } else {
                        ta = __ffma2_rn(vlo, vlo, ta);
                        tb = __ffma2_rn(vhi, vhi, tb);
                        sa = __ffma2_rn(wlo, vlo, sa);
                        sb = __ffma2_rn(whi, vhi, sb);
                    }
                }
            }
            float ttf = ((ta.x + ta.y) + (tb.x + tb.y)) + ((tc.x + tc.y) + (td.x + td.y));
            float stf = ((sa.x + sa.y) + (sb.x + sb.y)) + ((sc.x + sc.y) + (sd.x + sd.y));
            if constexpr (LPR == 2) {  // the row's two column segments
                ttf += __shfl_xor_sync(0xffffffffu, ttf, 1);
                stf += __shfl_xor_sync(0xffffffffu, stf, 1);
            }
            // similarity and loss weight (trainer.py:184-221): fp32 screen;
            // rows that can reach the margin are decided from the reference's
            // binary64 sums over the staged row (heat_row_update.cuh)
            float sf = 0.f;
            const bool band =
                valid && margin_band(r, a.cosine, (float)ss, ttf, stf, rss, theta_f, &sf);
            double ssx = ss, ttx = (double)ttf, stx = (double)stf;
            for (unsigned mb = __ballot_sync(0xffffffffu, band && lead), first = 1; mb; first = 0) {
                const int src = __ffs(mb) - 1;
                mb &= mb - 1;
                double s_, t_, c_;
                warp_dots64<K>(urow, ring + ((size_t)slot * SR + src / LPR) * G::SLOTF,
                               [](int k) { return G::pcol(k); }, first != 0, s_, t_, c_);
                if (first) ssx = s_;
                if (lane / LPR == src / LPR) {
                    ttx = t_;
                    stx = c_;
                }
            }
            if (!band) ssx = ss;
            bool write = false;
            double wt = 0.0;
            if (valid) {
                bool degenerate = false;
                double sim = band ? stx : (double)sf;
                if (a.cosine) {
                    if (band) {
                        degenerate = ssx <= 0.0 || ttx <= 0.0;
                        sim = degenerate ? 0.0 : stx / (sqrt(ssx) * sqrt(ttx));
                    }
                    if (degenerate && lead) ++degen;
                }
                if (r == 0) {
                    sim_p = sim;
                    wt = -1.0;
                    write = !(a.cosine && degenerate) || a.l2 != 0.f;
                } else {
                    if (sim - a.theta > 0.0) {
                        if (lead) hinge += sim - a.theta;
                        wt = wneg;
                        if (wt != 0.0 && lead) ++active;
                    }
                    write = (wt != 0.0 && !(a.cosine && degenerate)) || (wt == 0.0 && a.l2 != 0.f);
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, write && lead);
            while (m) {
                if (cnt == snap_cap) spill();
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const float *srow = ring + ((size_t)slot * SR + src / LPR) * G::SLOTF;
#pragma unroll
                for (int v = 0; v < VW; ++v)
                    snap[cnt * K + lane * VW + v] = srow[G::pcol(lane * VW + v)];
                if (lane == src)
                    ents[cnt] = WriteEntry{ttx, stx, wt, ids[slot * SR + src / LPR], 0};
                ++cnt;
            }
            __syncwarp();
            issue();  // refill this slot with the warp's stage i + D
        }
        cp_async_wait<0>();
        // every warp has read all of its rows: the pair's writes may start
        if (SPLIT) {
            mbar_wait(&reads_done, phase);
            phase ^= 1;
        } else {
            __syncthreads();
        }
        if (nbw > 0) {  // ss (hence the coefficients) is known to warps with stages
            __syncwarp();
            if (nsp) apply(sp_rows, sp_ents, nsp);
            apply(snap, ents, cnt);
            // this warp's share of the user gradient; the decay once (warp 0)
            float d[VW];
#pragma unroll
            for (int v = 0; v < VW; ++v) d[v] = -a.lr * (ug[v] + (w == 0 ? a.l2 * uu[v] : 0.f));
            if constexpr (VW == 2) {
                red_add2(a.S + u * K + lane * 2, d[0], d[1]);
            } else if constexpr (VW == 4) {
                red_add4(a.S + u * K + lane * 4, d[0], d[1], d[2], d[3]);
            } else {
#pragma unroll
                for (int v = 0; v < VW; ++v) atomicAdd(a.S + u * K + lane * VW + v, d[v]);
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) hinge += __shfl_xor_sync(0xffffffffu, hinge, o);
        if (lane == 0) loss += wneg * hinge + (w == 0 ? 1.0 - sim_p : 0.0);
        if (n_workers == 1) {  // a lone worker: the next pair reads after these writes
            __threadfence();
            __syncthreads();
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(0xffffffffu, degen, o);
        active += __shfl_xor_sync(0xffffffffu, active, o);
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
    }
    if (threadIdx.x == 0) {
        const int64_t mine_pairs = (npairs - gw + n_workers - 1) / n_workers;
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine_pairs);
    }
}

template <int K, int NW, int D, int LPR>
static cudaError_t launch_multi_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    int snap_cap = 8;  // measured on c3: 8 (77.6 M) > 16 (72 M) at 5 CTAs per SM
    if (const char *e = getenv("HEAT_SNAP")) snap_cap = atoi(e) > 0 ? atoi(e) : snap_cap;
    const MwLayout L = mw_layout<K, D, LPR>(snap_cap);
    const size_t smem = L.per_warp * NW;
    if (smem > 200 * 1024) return cudaErrorNotSupported;
    static const bool split = [] {
        const char *e = getenv("HEAT_MULTI_SPLIT");
        return e ? atoi(e) != 0 : false;  // measured on c3: 72.7 M split vs 77.7 M barrier
    }();
    auto kern = a.range_dev ? hogwild_multi<K, NW, D, LPR, false, true>
                : split     ? hogwild_multi<K, NW, D, LPR, true, false>
                            : hogwild_multi<K, NW, D, LPR, false, false>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32 * NW, smem, &e);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (a.stop - a.start < nw) nw = a.stop - a.start;
    if (workers_out) *workers_out = (int)nw;
    HogwildArgs b = a;
    if (a.N + 1 > snap_cap) {  // per-warp spill areas: a pair writes at most N+1 rows
        b.spill_cap = a.N + 1;
        b.spill_stride = ((int64_t)b.spill_cap * (K * sizeof(float) + sizeof(WriteEntry)) + 255) &
                         ~(int64_t)255;
        b.spill = static_cast<unsigned char *>(
            stream_scratch(3, (size_t)(b.spill_stride * nw * NW), st));
        if (!b.spill) b.spill_cap = 0;
    }
    kern<<<(unsigned)nw, 32 * NW, smem, st>>>(b, FastMod::make((uint64_t)a.num_items), (int)nw,
                                              snap_cap);
    return cudaGetLastError();
}

template <int K, int LPR>
static cudaError_t launch_multi_nw(const HogwildArgs &a, cudaStream_t st, int *workers_out,
                                   int nw, int d) {
    if (nw == 2) return d == 1 ? launch_multi_k<K, 2, 1, LPR>(a, st, workers_out)
                               : launch_multi_k<K, 2, 2, LPR>(a, st, workers_out);
    if (nw == 8) return d == 1 ? launch_multi_k<K, 8, 1, LPR>(a, st, workers_out)
                               : launch_multi_k<K, 8, 2, LPR>(a, st, workers_out);
    return d == 1 ? launch_multi_k<K, 4, 1, LPR>(a, st, workers_out)
                  : launch_multi_k<K, 4, 2, LPR>(a, st, workers_out);
}

cudaError_t launch_hogwild_multi(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    if (a.fp64 || a.query) return cudaErrorNotSupported;
    int nw = 4, d = 1;  // measured on c3: NW 4, D 1 (75 M) > NW 2 (74 M) > staged (64 M)
    if (const char *e = getenv("HEAT_MULTI_NW")) nw = atoi(e);
    if (const char *e = getenv("HEAT_MULTI_D")) d = atoi(e) == 2 ? 2 : 1;
    switch (a.K) {
    case 32: return launch_multi_nw<32, 1>(a, st, workers_out, nw, d);
    case 64: return launch_multi_nw<64, 1>(a, st, workers_out, nw, d);
    case 128: return launch_multi_nw<128, 2>(a, st, workers_out, nw, d);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace heat
