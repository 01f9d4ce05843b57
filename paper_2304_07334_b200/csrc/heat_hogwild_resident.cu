// heat_hogwild_resident.cu — throughput SGD for pairs whose rows fit in shared
// memory (N+1 <= 32*kMaxStages rows): one CTA per pair-worker, one warp per
// 32-row stage, the whole pair resident at once.
//
// Why: with a window of B pairs in flight only ~B/148 workers share an SM.
// One warp per worker leaves ~1.7 warps per scheduler and exposes every
// shared-memory and FMA latency (measured: 36 % issue efficiency).  Here the
// same B pairs are served by nb = ceil((N+1)/32) warps each, so an SM holds
// ~7 pairs but ~28 warps.
//
// Per pair (math = trainer.py:114-293, Hogwild across CTAs):
//   A  every warp draws its stage's negative ids (counter-form SplitMix64,
//      one draw per lane) and copies its 32 rows with per-lane 16-byte
//      cp.async.cg (LDGSTS, L2 evict-last hint); warp 0 also copies the user
//      row.  wait_group 0, barrier.
//   B  lane j of warp w scores row 32w+j: tt = v.v, st = u.v (LDS.128, rows
//      padded by 16 bytes: conflict-free), fp32 similarity screen, exact
//      binary64 only near the margin (trainer.py:184-221); rows to write are
//      appended to a CTA list by reference to their ring slot.  barrier.
//   C  the list is applied by all warps (entry e -> warp e % nb): item deltas
//      with red.global.add from the still-resident snapshot rows, user-gradient
//      partials per warp.  barrier.
//   D  warp 0 sums the partials in warp order and updates the user row;
//      the loss adds (1 - sim_p) + mu/N * sum of per-warp hinges.
// Every row of the pair is read before any write (trainer.py:118-146) and
// the written rows are the pre-pair snapshots, even for repeated ids.
#include <cstdint>
#include <cstdlib>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

constexpr int kMaxStages = 8;

template <int K>
struct RsGeom {
    static constexpr int ROWB = K * 4;
    static constexpr int SLOTF = K + 4;  // padded slot (floats)
    static constexpr int CH = K / 4;
    static constexpr int VW = K >= 32 ? K / 32 : 1;
    static constexpr int ACT = K >= 32 ? 32 : K;
};

struct RsEntry {
    float tt, st, w;  // cached forward scalars (v.v, u.v, loss weight)
    int32_t id;       // item row
    int32_t slot;     // ring slot (= row index within the pair) of the snapshot
};

template <int K>
__host__ __device__ inline size_t rs_smem_bytes(int nb, int rows, int cap) {
    using G = RsGeom<K>;
    size_t b = 8 * kMaxStages;                // hinge per warp (doubles first)
    b += sizeof(float) * G::SLOTF * rows;      // ring: one padded slot per row
    b += sizeof(float) * K;                   // user row
    b += sizeof(int32_t) * 32 * nb;           // ids
    b += sizeof(RsEntry) * cap;               // write list
    b += sizeof(float) * K * nb;              // user-gradient partials
    b += 16;                                  // counter
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

template <int K>
__global__ void __launch_bounds__(32 * kMaxStages)
    hogwild_resident(HogwildArgs a, FastMod fm, int n_workers, int cap) {
    using G = RsGeom<K>;
    constexpr int VW = G::VW;
    const int nb = blockDim.x >> 5;  // warps = stages
    extern __shared__ __align__(128) unsigned char sm[];
    // carve-out by alignment: doubles, then 16-byte cp.async targets, then the rest
    double *hinge_w = reinterpret_cast<double *>(sm);                      // [kMaxStages]
    float *ring = reinterpret_cast<float *>(sm + 8 * kMaxStages);          // 16-aligned
    float *urow = ring + (size_t)G::SLOTF * (a.N + 1);                     // 16-aligned
    float *part = urow + K;                                                // [nb][K]
    int32_t *ids = reinterpret_cast<int32_t *>(part + K * nb);             // [32*nb]
    int *cnt_p = ids + 32 * nb;
    RsEntry *list = reinterpret_cast<RsEntry *>(cnt_p + 4);

    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int64_t npairs = a.stop - a.start;
    const int N = a.N;
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;
    const uint64_t pol = policy_evict_last();
    const int r = w * 32 + lane;  // my row of every pair
    const bool valid = r <= N;
    const int nvalid = min(32, N + 1 - w * 32);
    constexpr int RPI = 32 / G::CH > 0 ? 32 / G::CH : 1;
    constexpr int NI = 32 / RPI;
    const int my_ch = lane % G::CH, my_rsub = lane / G::CH;
    float *my_stage = ring + (size_t)w * 32 * G::SLOTF;

    double loss = 0.0;
    long long degen = 0, active = 0, mine = 0;

    for (int64_t p = a.start + blockIdx.x; p < a.stop; p += n_workers) {
        ++mine;
        // ---- A: ids, copies
        const int64_t pg = a.pair_index ? a.pair_index[p] : p;
        const int32_t pos = a.items[p];
        const int64_t u = a.users[p];
        uint32_t id = (uint32_t)pos;
        if (r > 0) id = (uint32_t)fm.mod(mix64(a.s0 + ((uint64_t)pg * (uint64_t)N + (uint64_t)r) * kGamma));
        if (!valid) id = 0;
        ids[r] = (int32_t)id;
        if (threadIdx.x == 0) *cnt_p = 0;
        {
            float *dst = my_stage + my_rsub * G::SLOTF + my_ch * 4;
            const float *srcb = a.T + my_ch * 4;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int row = i * RPI + my_rsub;
                const uint32_t rid = __shfl_sync(0xffffffffu, id, row & 31);
                if (row < nvalid)
                    cp_async16_hint(dst + i * RPI * G::SLOTF, srcb + (size_t)rid * K, pol);
            }
            if (w == 0)
                for (int ch = lane; ch < G::CH; ch += 32)
                    cp_async16(urow + ch * 4, a.S + u * K + ch * 4);
            cp_async_commit();
            cp_async_wait<0>();
        }
        __syncthreads();  // B1: the pair's rows and the user row are resident

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
        const double rs = ss > 0.0 ? sqrt(ss) : 0.0;
        const float rss = ss > 0.0 ? rsqrtf(sp) : 0.f;
        double tt = 0.0, st = 0.0;
        if (valid) {
            const float *row = my_stage + lane * G::SLOTF;
            float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int k = 0; k < K; k += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(row + k);
                const float4 w4 = *reinterpret_cast<const float4 *>(urow + k);
                t0 = fmaf(v.x, v.x, t0); t1 = fmaf(v.y, v.y, t1);
                t2 = fmaf(v.z, v.z, t2); t3 = fmaf(v.w, v.w, t3);
                s0 = fmaf(w4.x, v.x, s0); s1 = fmaf(w4.y, v.y, s1);
                s2 = fmaf(w4.z, v.z, s2); s3 = fmaf(w4.w, v.w, s3);
            }
            tt = (double)((t0 + t1) + (t2 + t3));
            st = (double)((s0 + s1) + (s2 + s3));
        }
        bool write = false;
        double wt = 0.0, hinge = 0.0, sim = 0.0;
        if (valid) {
            bool degenerate = false;
            sim = st;
            if (a.cosine) {
                if (ss <= 0.0 || tt <= 0.0) {
                    degenerate = true;
                    sim = 0.0;
                    ++degen;
                } else {
                    const float sf = (float)st * rss * rsqrtf((float)tt);
                    sim = (double)sf;
                    if (r > 0 && sf > theta_f - 1e-5f) sim = st / (sqrt(ss) * sqrt(tt));
                }
            }
            if (r == 0) {
                wt = -1.0;
                write = !(a.cosine && degenerate) || a.l2 != 0.f;
            } else {
                if (sim - a.theta > 0.0) {
                    hinge = sim - a.theta;
                    wt = wneg;
                    if (wt != 0.0) ++active;
                }
                write = (wt != 0.0 && !(a.cosine && degenerate)) || (wt == 0.0 && a.l2 != 0.f);
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, write);
        if (m) {
            int base = 0;
            if (lane == 0) base = atomicAdd(cnt_p, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            const int e = base + __popc(m & ((1u << lane) - 1u));
            if (write && e < cap) list[e] = RsEntry{(float)tt, (float)st, (float)wt, (int32_t)id, r};
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) hinge += __shfl_xor_sync(0xffffffffu, hinge, o);
        if (lane == 0) hinge_w[w] = hinge;
        const double sim_p = __shfl_sync(0xffffffffu, sim, 0);  // valid in warp 0
        __syncthreads();  // B2: every row of the pair has been read

        // ---- C: apply the writes from the resident snapshots
        const int n_ent = min(*cnt_p, cap);
        float ug[VW];
#pragma unroll
        for (int i = 0; i < VW; ++i) ug[i] = 0.f;
        for (int e = w; e < n_ent; e += nb) {
            const RsEntry ent = list[e];
            const WriteEntry we{ent.tt, ent.st, ent.w, ent.id, 0};
            const RowCoef co = row_coef(we, ss, rs, a.lr, a.l2, a.cosine);
            const float *srow = ring + (size_t)ent.slot * G::SLOTF;
            float d[VW];
#pragma unroll
            for (int i = 0; i < VW; ++i) {
                const float v = lane < G::ACT ? srow[lane * VW + i] : 0.f;
                row_apply(co, uu[i], v, d[i], ug[i]);
            }
            if (!dmode) {
                if (lane < G::ACT) rs_red<VW>(a.T + (int64_t)ent.id * K + lane * VW, d);
            } else {
                long long sl = 0;
                if (lane == 0) sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
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
        if (lane < G::ACT) {
#pragma unroll
            for (int i = 0; i < VW; ++i) part[w * K + lane * VW + i] = ug[i];
        }
        __syncthreads();  // B3: partial user gradients ready, ring reads done

        // ---- D: user row and loss (warp 0), fixed summation order
        if (w == 0) {
            if (lane < G::ACT) {
                float d[VW];
#pragma unroll
                for (int i = 0; i < VW; ++i) {
                    float g = 0.f;
                    for (int ww = 0; ww < nb; ++ww) g += part[ww * K + lane * VW + i];
                    d[i] = -a.lr * (g + a.l2 * uu[i]);
                }
                rs_red<VW>(a.S + u * K + lane * VW, d);
            }
            if (lane == 0) {
                double h = 0.0;
                for (int ww = 0; ww < nb; ++ww) h += hinge_w[ww];
                loss += (1.0 - sim_p) + wneg * h;
            }
        }
    }
    // telemetry
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(0xffffffffu, degen, o);
        active += __shfl_xor_sync(0xffffffffu, active, o);
    }
    if (lane == 0) {
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
    }
    if (threadIdx.x == 0) {
        atomicAdd(&a.ctr->loss, loss);
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine);
    }
    (void)npairs;
}

template <int K>
static cudaError_t launch_resident_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    const int nb = (a.N + 1 + 31) / 32;
    // one stage per pair: the single-warp staged kernel is as good (measured)
    if (nb > kMaxStages || (nb < 2 && !getenv("HEAT_HOGWILD_IMPL"))) return cudaErrorNotSupported;
    const int cap = a.N + 1;  // each row enters the list at most once: never overflows
    const size_t smem = rs_smem_bytes<K>(nb, a.N + 1, cap);
    if (smem > 96 * 1024) return cudaErrorNotSupported;
    auto kern = hogwild_resident<K>;
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * nb, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (a.stop - a.start < nw) nw = a.stop - a.start;
    if (workers_out) *workers_out = (int)nw;
    kern<<<(unsigned)nw, 32 * nb, smem, st>>>(a, FastMod::make((uint64_t)a.num_items), (int)nw,
                                              cap);
    return cudaGetLastError();
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
