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
#include <cstdlib>
#include <type_traits>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

constexpr int kHogThreads = 256;
constexpr int kHogWarps = kHogThreads / 32;
constexpr int kListCap = 32;  // deferred row writes per warp before a flush

template <typename T>
__device__ __forceinline__ T shfl_xor_t(T v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

// ---------------------------------------------------------------------------
// Generic path: any K <= 32*kMaxC.  Warp per pair, one row at a time, lanes
// strided over columns.  Pass 1 reads every row once and records the rows to
// write; pass 2 (flush) re-reads only those rows from L2 and applies them,
// so no row of the pair is read after the pair wrote it (the reference
// snapshots rows before updating, trainer.py:118-146).
// ---------------------------------------------------------------------------
constexpr int kMaxC = 16;

// PH: phase profile (heat_phase_collect) of the warp's pairs into a.phase:
// read_emb = the user row, similarity = each row's read and dots (one
// statement: the load latency lands here), loss = the margin decisions and
// hinge, gradient = the flush's row coefficients and deltas, update = its
// atomics and the user row's
template <int C, bool PH = false>
__global__ void __launch_bounds__(kHogThreads)
    hogwild_generic(HogwildArgs a, FastMod fm, int n_workers) {
    __shared__ WriteEntry lists[kHogWarps][kListCap];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * kHogWarps + wib;
    if (gw >= n_workers) return;
    WriteEntry *list = lists[wib];
    const int K = a.K, N = a.N;
    const double wneg = a.mu * (1.0 / (double)N);
    const bool dmode = a.delta_ids != nullptr;
    double loss = 0.0;
    long long degen = 0, active = 0, mine = 0;
    long long ph[6] = {0, 0, 0, 0, 0, 0}, tm = 0;
    long long c_start = 0, g_start = 0;
    auto gtimer = []() -> long long {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return (long long)t;
    };
    if constexpr (PH) {
        c_start = clock64();
        g_start = gtimer();
    }
    auto mark = [&](int i) {  // phase i ends here
        if constexpr (PH) {
            const long long t = clock64();
            ph[i] += t - tm;
            tm = t;
        }
    };

    for (int64_t p = a.start + gw; p < a.stop; p += n_workers) {
        if constexpr (PH) tm = clock64();
        ++mine;
        const int64_t u = a.users[p];
        const int64_t pos = a.items[p];
        const int64_t pg = a.pair_index ? a.pair_index[p] : p;  // RNG key
        float ur[C], ug[C];
        double ssp = 0.0;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int k = lane + 32 * c;
            ur[c] = k < K ? __ldcg(a.S + u * K + k) : 0.f;
            ug[c] = 0.f;
            ssp += (double)ur[c] * (double)ur[c];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssp += shfl_xor_t(ssp, o);
        const double ss = ssp;
        const double rs = ss > 0.0 ? sqrt(ss) : 0.0;
        int cnt = 0;
        mark(0);

        // rows of one flush round are all loaded before any update, so a row
        // written twice in a pair uses its pre-pair snapshot both times
        constexpr int E = 32 / C > 0 ? 32 / C : 1;
        auto flush = [&]() {
            __syncwarp();
            for (int e0 = 0; e0 < cnt; e0 += E) {
                float x[E][C];
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    const int32_t id = e0 + j < cnt ? list[e0 + j].id : 0;
#pragma unroll
                    for (int c = 0; c < C; ++c) {
                        const int k = lane + 32 * c;
                        x[j][c] = (e0 + j < cnt && k < K) ? __ldcg(a.T + (int64_t)id * K + k) : 0.f;
                    }
                }
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    if (e0 + j >= cnt) break;
                    const WriteEntry ent = list[e0 + j];
                    const RowCoef co = row_coef(ent, ss, rs, a.lr, a.l2, a.cosine);
                    float d[C];
#pragma unroll
                    for (int c = 0; c < C; ++c) row_apply(co, ur[c], x[j][c], d[c], ug[c]);
                    mark(3);
                    if (!dmode) {
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const int k = lane + 32 * c;
                            if (k < K) atomicAdd(a.T + (int64_t)ent.id * K + k, d[c]);
                        }
                    } else {
                        long long sl = 0;
                        if (lane == 0)
                            sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                        sl = __shfl_sync(0xffffffffu, sl, 0);
                        if (sl < a.delta_capacity) {
                            if (lane == 0) a.delta_ids[sl] = ent.id;
#pragma unroll
                            for (int c = 0; c < C; ++c) {
                                const int k = lane + 32 * c;
                                if (k < K) a.delta_rows[sl * K + k] = d[c];
                            }
                        }
                    }
                    mark(4);
                }
            }
            cnt = 0;
            __syncwarp();
        };

        double hinge = 0.0, sim_p = 0.0;
        for (int r = 0; r <= N; ++r) {
            const int32_t id = r == 0 ? (int32_t)pos : neg_id(a.s0, pg, N, r - 1, fm);
            double ttp = 0.0, stp = 0.0;
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int k = lane + 32 * c;
                const float v = k < K ? __ldcg(a.T + (int64_t)id * K + k) : 0.f;
                ttp += (double)v * (double)v;
                stp += (double)ur[c] * (double)v;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                ttp += shfl_xor_t(ttp, o);
                stp += shfl_xor_t(stp, o);
            }
            const double tt = ttp, st = stp;
            mark(1);
            bool degenerate = false;
            double sim = st;
            if (a.cosine) {
                if (ss <= 0.0 || tt <= 0.0) {
                    degenerate = true;
                    sim = 0.0;
                    ++degen;
                } else {
                    sim = st / (sqrt(ss) * sqrt(tt));
                }
            }
            double w = 0.0;
            bool write;
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
            if (write) {
                mark(2);
                if (cnt == kListCap) flush();
                if (lane == 0) list[cnt] = WriteEntry{tt, st, w, id, 0};
                ++cnt;
            }
            mark(2);
        }
        flush();
        loss += (1.0 - sim_p) + wneg * hinge;
        mark(2);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int k = lane + 32 * c;
            if (k < K) atomicAdd(a.S + u * K + k, -a.lr * (ug[c] + a.l2 * ur[c]));
        }
        mark(4);
    }
    if constexpr (PH) {
        if (lane == 0 && a.phase) {
            for (int i = 0; i < 6; ++i) atomicAdd(a.phase + i, (unsigned long long)ph[i]);
            atomicAdd(a.phase + 6, (unsigned long long)(clock64() - c_start));
            atomicAdd(a.phase + 7, (unsigned long long)(gtimer() - g_start));
            atomicAdd(a.phase + 8, 1ull);
            atomicAdd(a.phase + 9, (unsigned long long)mine);
        }
    }
    if (lane == 0) {
        atomicAdd(&a.ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&a.ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&a.ctr->active, (unsigned long long)active);
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine);
    }
}

template <int C>
static cudaError_t launch_generic_c(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    auto kern = a.phase ? hogwild_generic<C, true> : hogwild_generic<C, false>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHogThreads, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t nw = (int64_t)per_sm * kHogWarps * sm_count();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (a.stop - a.start < nw) nw = a.stop - a.start;
    if (workers_out) *workers_out = (int)nw;
    const int blocks = (int)((nw + kHogWarps - 1) / kHogWarps);
    kern<<<blocks, kHogThreads, 0, st>>>(a, FastMod::make((uint64_t)a.num_items), (int)nw);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fast path: K in {16, 32, 64, 128}.
//
// A row of K floats is read by a "row group" of L = K/4 lanes with one
// ld.global.cg.v4 each, so one warp instruction reads RPI = 32/L whole rows
// (fully coalesced 16-byte lanes).  A batch is U such instructions
// (RPB = U*RPI rows) held in registers; the next batch's loads are issued
// before the current batch is reduced (double buffering).  Each lane forms
// 4-term partial dot products (tt = v.v, st = u.v) for its U rows, and a
// transposed butterfly reduces all U rows of the group at once:
// U-1 + log2(L/U) shuffles per quantity instead of U*log2(L).  Afterwards
// lane c of group g holds the full (tt, st) of batch row (c/(L/U))*RPI + g.
//
// Rows to write (positive, active negatives, decay rows) are recorded with
// their cached scalars; at the end of the pair (or when the list fills) they
// are re-read from L2 — all rows of a flush round before any update, so
// duplicate ids inside a pair still use the pre-pair snapshot — and applied
// with red.global.add.v4.f32.  Negative ids of the pair are drawn once, one
// counter-form SplitMix64 draw per lane, into per-warp shared memory.
// ---------------------------------------------------------------------------
template <int U, int L, typename A>
__device__ __forceinline__ A transpose_reduce(A (&a)[U], int c) {
#pragma unroll
    for (int n = U, o = L / 2; n > 1; n >>= 1, o >>= 1) {
        const bool up = (c & o) != 0;
#pragma unroll
        for (int j = 0; j < n / 2; ++j) {
            A send = up ? a[j] : a[j + n / 2];
            A keep = up ? a[j + n / 2] : a[j];
            a[j] = keep + shfl_xor_t(send, o);
        }
    }
    A v = a[0];
#pragma unroll
    for (int o = L / (2 * U); o >= 1; o >>= 1) v += shfl_xor_t(v, o);
    return v;
}

template <int K, int U, bool F64>
__global__ void __launch_bounds__(kHogThreads)
    hogwild_fast(HogwildArgs a, FastMod fm, int n_workers, int ids_stride) {
    constexpr int L = K / 4;
    constexpr int RPI = 32 / L;
    constexpr int RPB = U * RPI;
    constexpr int SUB = L / U;  // lanes sharing one reduced row
    static_assert(L >= U && L <= 32, "row group must hold U partials");
    static_assert(RPB <= kListCap, "one batch of writes must fit the list");
    using A = typename std::conditional<F64, double, float>::type;

    __shared__ WriteEntry lists[kHogWarps][kListCap];
    extern __shared__ int32_t ids_all[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int gw = blockIdx.x * kHogWarps + wib;
    if (gw >= n_workers) return;
    int32_t *ids = ids_all + wib * ids_stride;
    WriteEntry *list = lists[wib];
    const int g = lane / L;    // row group
    const int c = lane % L;    // float4 column chunk
    const int slot = c / SUB;  // reduced row slot held after the reduction
    const bool owner = (c % SUB) == 0;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int N = a.N;
    const int nb = (N + 1 + RPB - 1) / RPB;
    const double wneg = a.mu * (1.0 / (double)N);
    const float theta_f = (float)a.theta;
    const bool dmode = a.delta_ids != nullptr;

    double loss = 0.0;
    long long degen = 0, active = 0, mine = 0;

    for (int64_t p = a.start + gw; p < a.stop; p += n_workers) {
        ++mine;
        const int64_t u = a.users[p];
        const int64_t pos = a.items[p];
        const int64_t pg = a.pair_index ? a.pair_index[p] : p;  // RNG key
        for (int r = lane; r < nb * RPB; r += 32)
            ids[r] = r == 0 ? (int32_t)pos : (r <= N ? neg_id(a.s0, pg, N, r - 1, fm) : 0);
        const float4 u4 = ldcg4(a.S + u * K + c * 4);
        A ssp = (A)u4.x * (A)u4.x + (A)u4.y * (A)u4.y + (A)u4.z * (A)u4.z + (A)u4.w * (A)u4.w;
#pragma unroll
        for (int o = L / 2; o >= 1; o >>= 1) ssp += shfl_xor_t(ssp, o);
        const double ss = (double)ssp;
        const double rs = ss > 0.0 ? sqrt(ss) : 0.0;
        const float rss = ss > 0.0 ? rsqrtf((float)ss) : 0.f;
        __syncwarp();

        float4 ug = make_float4(0.f, 0.f, 0.f, 0.f);
        double hinge = 0.0, sim_p = 0.0;
        int cnt = 0;

        auto flush = [&]() {
            __syncwarp();
            for (int e0 = 0; e0 < cnt; e0 += RPB) {
                float4 x[U];
#pragma unroll
                for (int i = 0; i < U; ++i) {
                    const int e = e0 + i * RPI + g;
                    x[i] = e < cnt ? ldcg4(a.T + (int64_t)list[e].id * K + c * 4)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int i = 0; i < U; ++i) {
                    const int e = e0 + i * RPI + g;
                    const bool ok = e < cnt;
                    WriteEntry ent;
                    if (ok) ent = list[e];
                    float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok) {
                        const RowCoef co = row_coef(ent, ss, rs, a.lr, a.l2, a.cosine);
                        row_apply(co, u4.x, x[i].x, d.x, ug.x);
                        row_apply(co, u4.y, x[i].y, d.y, ug.y);
                        row_apply(co, u4.z, x[i].z, d.z, ug.z);
                        row_apply(co, u4.w, x[i].w, d.w, ug.w);
                    }
                    if (!dmode) {
                        if (ok) red_add4(a.T + (int64_t)ent.id * K + c * 4, d.x, d.y, d.z, d.w);
                    } else {
                        long long sl = 0;
                        if (ok && c == 0)
                            sl = (long long)atomicAdd((unsigned long long *)a.delta_count, 1ull);
                        sl = __shfl_sync(0xffffffffu, sl, g * L);
                        if (ok && sl < a.delta_capacity) {
                            if (c == 0) a.delta_ids[sl] = ent.id;
                            *reinterpret_cast<float4 *>(a.delta_rows + sl * K + c * 4) = d;
                        }
                    }
                }
            }
            cnt = 0;
            __syncwarp();
        };

        float4 vA[U], vB[U];
        auto load = [&](float4 (&v)[U], int b) {
#pragma unroll
            for (int i = 0; i < U; ++i) {
                const int r = b * RPB + i * RPI + g;
                v[i] = r <= N ? ldcg4(a.T + (int64_t)ids[r] * K + c * 4)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };

        auto process = [&](float4 (&v)[U], int b) {
            A tt[U], st[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                tt[i] = (A)v[i].x * (A)v[i].x + (A)v[i].y * (A)v[i].y + (A)v[i].z * (A)v[i].z +
                        (A)v[i].w * (A)v[i].w;
                st[i] = (A)u4.x * (A)v[i].x + (A)u4.y * (A)v[i].y + (A)u4.z * (A)v[i].z +
                        (A)u4.w * (A)v[i].w;
            }
            const double ttr = (double)transpose_reduce<U, L>(tt, c);
            const double str = (double)transpose_reduce<U, L>(st, c);
            const int r = b * RPB + slot * RPI + g;
            const bool valid = owner && r <= N;
            // similarity and loss weight (trainer.py:184-221)
            bool write = false;
            double w = 0.0;
            if (valid) {
                bool degenerate = false;
                double sim = str;
                if (a.cosine) {
                    if (ss <= 0.0 || ttr <= 0.0) {
                        degenerate = true;
                        sim = 0.0;
                        ++degen;
                    } else if (F64 || r == 0) {
                        sim = str / (sqrt(ss) * sqrt(ttr));
                    } else {
                        // screen in fp32, exact value only for the few that pass
                        const float sf = (float)str * rss * rsqrtf((float)ttr);
                        sim = sf > theta_f - 1e-5f ? str / (sqrt(ss) * sqrt(ttr)) : (double)sf;
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
            const unsigned m = __ballot_sync(0xffffffffu, write);
            if (m) {
                const int nw = __popc(m);
                if (cnt + nw > kListCap) flush();
                if (write) list[cnt + __popc(m & lt_mask)] = WriteEntry{ttr, str, w, ids[r], 0};
                cnt += nw;
            }
        };

        load(vA, 0);
        for (int b = 0; b < nb; b += 2) {
            if (b + 1 < nb) load(vB, b + 1);
            process(vA, b);
            if (b + 1 < nb) {
                if (b + 2 < nb) load(vA, b + 2);
                process(vB, b + 1);
            }
        }
        flush();
        // user row: combine the row groups' partial gradients (same columns)
#pragma unroll
        for (int o = L; o < 32; o <<= 1) {
            ug.x += shfl_xor_t(ug.x, o); ug.y += shfl_xor_t(ug.y, o);
            ug.z += shfl_xor_t(ug.z, o); ug.w += shfl_xor_t(ug.w, o);
        }
        if (g == 0)
            red_add4(a.S + u * K + c * 4, -a.lr * (ug.x + a.l2 * u4.x), -a.lr * (ug.y + a.l2 * u4.y),
                     -a.lr * (ug.z + a.l2 * u4.z), -a.lr * (ug.w + a.l2 * u4.w));
        // hinge and sim_p live in owner lanes (sim_p in lane 0)
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) hinge += __shfl_xor_sync(0xffffffffu, hinge, o);
        if (lane == 0) loss += (1.0 - sim_p) + wneg * hinge;
        __syncwarp();
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
        atomicAdd((unsigned long long *)&a.ctr->pairs, (unsigned long long)mine);
    }
}

template <int K, int U, bool F64>
static cudaError_t launch_fast_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    constexpr int RPB = U * (32 / (K / 4));
    const int rows = a.N + 1;
    const int ids_stride = ((rows + RPB - 1) / RPB) * RPB;
    const size_t smem = (size_t)ids_stride * sizeof(int32_t) * kHogWarps;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    auto kern = hogwild_fast<K, U, F64>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, kHogThreads, smem, &e);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)per_sm * kHogWarps * sm_count();
    if (a.window > 0 && a.window < nw) nw = a.window;
    if (a.stop - a.start < nw) nw = a.stop - a.start;
    if (workers_out) *workers_out = (int)nw;
    int blocks = (int)((nw + kHogWarps - 1) / kHogWarps);
    kern<<<blocks, kHogThreads, smem, st>>>(a, FastMod::make((uint64_t)a.num_items), (int)nw,
                                             ids_stride);
    return cudaGetLastError();
}

template <int K>
static cudaError_t launch_fast(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    constexpr int U = (K / 4) >= 8 ? 8 : (K / 4);
    if (a.fp64) return launch_fast_k<K, U, true>(a, st, workers_out);
    return launch_fast_k<K, U, false>(a, st, workers_out);
}

cudaError_t launch_hogwild(const HogwildArgs &a, cudaStream_t stream, int *workers_out) {
    if (a.stop <= a.start) {
        if (workers_out) *workers_out = 0;
        return cudaSuccess;
    }
    // resident (default when the pair fits in smem) | staged (cp.async ring) |
    // tma (bulk-copy ring) | regs | generic
    const char *impl = getenv("HEAT_HOGWILD_IMPL");
    const bool aligned = ((uintptr_t)a.S % 16 == 0) && ((uintptr_t)a.T % 16 == 0);
    if (getenv("HEAT_FORCE_GENERIC")) impl = "generic";
    // phase profile: the instrumented kernels only (register-streamed at
    // dim 64/128, generic otherwise)
    if (a.phase && !a.delta_ids && !a.range_dev)
        impl = aligned && (a.K == 64 || a.K == 128) && hogwild_stream_supported(a) ? "wide" : "generic";
    if (aligned && (!impl || impl[0] == 'r' && impl[1] == 'e')) {
        cudaError_t e = launch_hogwild_resident(a, stream, workers_out);
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    // register-streamed rows (heat_hogwild_stream.cu): the default for
    // K = 128 (configs 4/5: c4 29.4 M vs 22.4 M samples/s staged, c5 14.5 M vs
    // 12.7 M); for K <= 64 the pair-per-CTA kernels keep more warps busy
    // under the config windows (c3: multi 77.6 M vs 40.4 M)
    const bool wide_default = (!impl || (impl[0] == 'r' && impl[1] == 'e')) && a.K == 128;
    if (aligned && ((impl && impl[0] == 'w') || wide_default)) {
        cudaError_t e = launch_hogwild_stream(a, stream, workers_out);
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue &&
            e != cudaErrorMemoryAllocation)
            return e;
    }
    // several warps per pair (large N, K <= 64: the pair does not fit the
    // resident kernel, and one warp per pair leaves the SMs underoccupied)
    const bool multi_forced = impl && impl[0] == 'm';
    const bool multi_default = (!impl || (impl[0] == 'r' && impl[1] == 'e')) &&
                               (a.K == 32 || a.K == 64) && a.N + 1 > 256;
    if (aligned && (multi_forced || multi_default)) {
        cudaError_t e = launch_hogwild_multi(a, stream, workers_out);
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    if (aligned && (!impl || impl[0] == 's' || impl[0] == 't' || impl[0] == 'm' ||
                    (impl[0] == 'r' && impl[1] == 'e'))) {
        cudaError_t e = launch_hogwild_staged(a, stream, workers_out, impl && impl[0] == 't');
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    if (a.range_dev) return cudaErrorNotSupported;  // the families below read start/stop only
    if (!impl || impl[0] != 'g') {  // regs
        cudaError_t e = cudaErrorNotSupported;
        switch (a.K) {
        case 16: e = launch_fast<16>(a, stream, workers_out); break;
        case 32: e = launch_fast<32>(a, stream, workers_out); break;
        case 64: e = launch_fast<64>(a, stream, workers_out); break;
        case 128: e = launch_fast<128>(a, stream, workers_out); break;
        default: break;
        }
        if (e != cudaErrorNotSupported && e != cudaErrorInvalidValue) return e;
    }
    const int C = (a.K + 31) / 32;
    if (C <= 1) return launch_generic_c<1>(a, stream, workers_out);
    if (C <= 2) return launch_generic_c<2>(a, stream, workers_out);
    if (C <= 4) return launch_generic_c<4>(a, stream, workers_out);
    if (C <= 8) return launch_generic_c<8>(a, stream, workers_out);
    return launch_generic_c<kMaxC>(a, stream, workers_out);
}

}  // namespace heat
