// heat_hogwild.cu — throughput ("hogwild") SGD: many pairs in flight, lock-free
// atomic row updates.  The device counterpart of the reference's
// multi-threaded mode (trainer.py:12-17, 398-447: threads update shared S/T
// without locks); per-pair math is trainer.py:114-293 (cosine or dot,
// uniform negatives, l2), each pair's rows read ONCE and the forward
// reductions (ss, tt_j, st_j) reused by the backward pass (HEAT Eq. 3/4,
// PAPER.md:574-592).
//
// Scheduling: a persistent grid of W pair-workers (one warp each),
// W = min(window, resident warps, pairs); worker w takes pairs
// start + w, start + w + W, ...  So at most `window` (the step size B) pairs
// are in flight, the staleness bound of a batched step of B pairs, without a
// launch + tail per step.
//
// Row updates use red.global.add (T rows of the positive / active negatives,
// S row of the user).  Rows are read with ld.global.cg (L2, not L1) so a
// warp never sees an L1-stale copy of a row another SM updated.
#include <cstdint>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

constexpr int kHogThreads = 256;
constexpr int kHogWarps = kHogThreads / 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// Generic path: any K <= 32*kMaxC.  Warp per pair, one row at a time, lanes
// strided over columns, binary64 reductions.
// ---------------------------------------------------------------------------
constexpr int kMaxC = 16;

template <int C>
__global__ void __launch_bounds__(kHogThreads)
    hogwild_generic(HogwildArgs a, int n_workers) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kHogWarps + (threadIdx.x >> 5);
    if (gw >= n_workers) return;
    const int K = a.K, N = a.N;
    const FastMod fm = FastMod::make((uint64_t)a.num_items);
    const double inv_n = 1.0 / (double)N;
    const double wneg = a.mu * inv_n;
    const bool delta_mode = a.delta_ids != nullptr;
    double loss = 0.0;
    long long degen = 0, active = 0;

    for (int64_t p = a.start + gw; p < a.stop; p += n_workers) {
        const int64_t u = a.users[p];
        const int64_t pos = a.items[p];
        float ur[C], ug[C];
        double ssp = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            int k = lane + 32 * c;
            ur[c] = k < K ? __ldcg(a.S + u * K + k) : 0.f;
            ug[c] = 0.f;
            ssp += (double)ur[c] * (double)ur[c];
        }
        const double ss = warp_sum_d(ssp);
        const double rs = ss > 0.0 ? sqrt(ss) : 0.0;
        double hinge = 0.0, sim_p = 0.0;
        for (int r = 0; r <= N; ++r) {
            int64_t id = r == 0 ? pos : (int64_t)neg_id(a.s0, p, N, r - 1, fm);
            float v[C];
            double ttp = 0.0, stp = 0.0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                int k = lane + 32 * c;
                v[c] = k < K ? __ldcg(a.T + id * K + k) : 0.f;
                ttp += (double)v[c] * (double)v[c];
                stp += (double)ur[c] * (double)v[c];
            }
            const double tt = warp_sum_d(ttp);
            const double st = warp_sum_d(stp);
            double sim;
            bool degenerate = false;
            if (a.cosine) {
                if (ss <= 0.0 || tt <= 0.0) {
                    sim = 0.0;
                    degenerate = true;
                    ++degen;
                } else {
                    sim = st / (sqrt(ss) * sqrt(tt));
                }
            } else {
                sim = st;
            }
            double w;
            if (r == 0) {
                sim_p = sim;
                w = -1.0;
            } else {
                double d = sim - a.theta;
                if (d > 0.0) {
                    hinge += d;
                    w = wneg;
                } else {
                    w = 0.0;
                }
            }
            if (r > 0 && w != 0.0) ++active;
            float dv[C];
            bool write = false;
            if (w != 0.0 && !(a.cosine && degenerate)) {
                write = true;
                if (a.cosine) {
                    // item: w*(u*tt - st*v)/(tt*sqrt(tt)*rs); user: w*(v*ss - st*u)/(ss*rs*sqrt(tt))
                    const double ci = w / (tt * sqrt(tt) * rs);
                    const double cu = w / (ss * rs * sqrt(tt));
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        double g = ci * ((double)ur[c] * tt - st * (double)v[c]);
                        dv[c] = (float)(-(double)a.lr * (g + (double)a.l2 * (double)v[c]));
                        ug[c] += (float)(cu * ((double)v[c] * ss - st * (double)ur[c]));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        double g = w * (double)ur[c];
                        dv[c] = (float)(-(double)a.lr * (g + (double)a.l2 * (double)v[c]));
                        ug[c] += (float)(w * (double)v[c]);
                    }
                }
            } else if (a.l2 != 0.f && !(r > 0 && w != 0.0)) {
                // decay-only rows: pos when degenerate (trainer.py:265-267),
                // inactive negatives (trainer.py:287-290)
                write = true;
#pragma unroll
                for (int c = 0; c < C; ++c) dv[c] = -a.lr * a.l2 * v[c];
            }
            if (write) {
                if (!delta_mode) {
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        int k = lane + 32 * c;
                        if (k < K) atomicAdd(a.T + id * K + k, dv[c]);
                    }
                } else {
                    long long slot = 0;
                    if (lane == 0) slot = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                    slot = __shfl_sync(0xffffffffu, slot, 0);
                    if (slot < a.delta_capacity) {
                        if (lane == 0) a.delta_ids[slot] = (int32_t)id;
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            int k = lane + 32 * c;
                            if (k < K) a.delta_rows[slot * K + k] = dv[c];
                        }
                    }
                }
            }
        }
        loss += (1.0 - sim_p) + wneg * hinge;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            int k = lane + 32 * c;
            if (k < K) atomicAdd(a.S + u * K + k, -a.lr * (ug[c] + a.l2 * ur[c]));
        }
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
        int64_t mine = 0;
        for (int64_t p = a.start + gw; p < a.stop; p += n_workers) ++mine;
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine);
    }
}

template <int C>
static cudaError_t launch_generic_c(const HogwildArgs &a, int n_workers, cudaStream_t st) {
    int blocks = (n_workers + kHogWarps - 1) / kHogWarps;
    hogwild_generic<C><<<blocks, kHogThreads, 0, st>>>(a, n_workers);
    return cudaGetLastError();
}

static int resident_warps_generic() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hogwild_generic<4>, kHogThreads, 0);
    if (per_sm < 1) per_sm = 1;
    return per_sm * kHogWarps * sm_count();
}

cudaError_t launch_hogwild(const HogwildArgs &a, cudaStream_t stream, int *workers_out) {
    int64_t npairs = a.stop - a.start;
    if (npairs <= 0) {
        if (workers_out) *workers_out = 0;
        return cudaSuccess;
    }
    int64_t nw = resident_warps_generic();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (npairs < nw) nw = npairs;
    if (workers_out) *workers_out = (int)nw;
    const int C = (a.K + 31) / 32;
    if (C <= 1) return launch_generic_c<1>(a, (int)nw, stream);
    if (C <= 2) return launch_generic_c<2>(a, (int)nw, stream);
    if (C <= 4) return launch_generic_c<4>(a, (int)nw, stream);
    if (C <= 8) return launch_generic_c<8>(a, (int)nw, stream);
    return launch_generic_c<kMaxC>(a, (int)nw, stream);
}

}  // namespace heat
