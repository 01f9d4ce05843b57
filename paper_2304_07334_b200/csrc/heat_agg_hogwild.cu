// heat_agg_hogwild.cu — SimpleX behaviour aggregation, throughput (Hogwild) mode.
//
// The reference's multi-thread aggregator (trainer.py:148-173, 299-331;
// aggregator.py:64-113) keeps a thread-local K x K accumulator of
// (1-gamma)*pooled (x) ugrad and flushes it into the shared W every
// mini_batch pairs, so W is stale by up to threads x mini_batch pairs.  On the
// GPU the epoch runs in steps of C = window pairs; within a step W is frozen
// and every per-pair quantity that touches W becomes a small dense product
// over the step's C pairs:
//
//   1. pool      P[m]  = (1-gamma) * mean(T[first max_history items of u_m])
//                 warp per pair, coalesced 128-bit row gathers (HBM/L2 bound)
//   2. query     Q     = gamma * S[u] + P . W        (C x K x K, tiled FMA GEMM)
//   3. CCL pair  the staged Hogwild kernel with Q as the query; writes the user
//                 gradient G[m], updates T and S[u] -= lr*(gamma*G + l2*S[u])
//   4. wgrad     W    -= (agg_lr / mini_batch) * P^T . G   (K x K, split over
//                 the step's pairs, red.global.add.v4)
//   5. history   (history_grad) WH = G . W^T, T[hist] -= lr*((1-gamma)/len * WH
//                 + l2*T[hist])  (trainer.py:316-326)
//
// Every pair contributes agg_lr/mini_batch * P (x) G to W exactly as in the
// reference, on the reference's flush schedule: a mini-batch's contributions
// reach W when its last pair is done (those of an incomplete batch wait in the
// fp64 accumulator, and the epoch's last incomplete batch is dropped, as the
// reference's per-epoch thread state drops it).  Only the staleness differs
// (one step instead of threads x mini_batch pairs).  The GEMMs are K x K x C with K <= 128: about 2*C*K^2
// flops per step (67 MFLOP for C = 2048, K = 128), a few percent of the
// step's gather traffic, so they stay on the FMA pipes (fp32 like the tables)
// instead of a tensor-core pipeline whose setup would dominate.
#include <cstdint>
#include <algorithm>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

// ---- 1. pooled history ------------------------------------------------------
// lane-vector of VW floats: one 16/8/4-byte load per lane per row
template <int VW>
struct LaneVec {
    float v[VW];
    __device__ __forceinline__ void load(const float *p) {
        if constexpr (VW == 4) {
            const float4 x = *reinterpret_cast<const float4 *>(p);
            v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        } else if constexpr (VW == 2) {
            const float2 x = *reinterpret_cast<const float2 *>(p);
            v[0] = x.x; v[1] = x.y;
        } else {
            v[0] = *p;
        }
    }
};

template <int K>
__global__ void __launch_bounds__(256)
    agg_pool_kernel(const float *__restrict__ T, const int32_t *__restrict__ users, int64_t n,
                    const int64_t *__restrict__ off, const int32_t *__restrict__ hist,
                    int64_t max_history, float one_minus_gamma, float *__restrict__ P) {
    constexpr int VW = K >= 32 ? K / 32 : 1;
    constexpr int ACT = K >= 32 ? 32 : K;
    constexpr int U = 8;  // rows in flight per lane
    const int lane = threadIdx.x & 31;
    const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (m >= n || lane >= ACT) return;
    const int64_t u = users[m];
    const int64_t hb = off[u];
    const int64_t he = imin64(off[u + 1], hb + max_history);
    float acc[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) acc[i] = 0.f;
    const float *Tl = T + lane * VW;
    int64_t idx = hb;
    for (; idx + U <= he; idx += U) {
        LaneVec<VW> r[U];
#pragma unroll
        for (int q = 0; q < U; ++q) r[q].load(Tl + (int64_t)hist[idx + q] * K);
#pragma unroll
        for (int q = 0; q < U; ++q)
#pragma unroll
            for (int i = 0; i < VW; ++i) acc[i] += r[q].v[i];
    }
    for (; idx < he; ++idx) {
        LaneVec<VW> r;
        r.load(Tl + (int64_t)hist[idx] * K);
#pragma unroll
        for (int i = 0; i < VW; ++i) acc[i] += r.v[i];
    }
    const int64_t len = he - hb;
    const float sc = len > 0 ? one_minus_gamma / (float)len : 0.f;
#pragma unroll
    for (int i = 0; i < VW; ++i) P[m * K + lane * VW + i] = acc[i] * sc;
}

// ---- 2 / 5a. out = A . B (+ add_scale * addend[rows[m]]) ------------------------
// A: n x K row-major; B(k, j) = W[k*K + j] (TRANS_B = false) or W[j*K + k].
// CTA: TM = 4096/K rows x all K columns, 256 threads, 4 rows x 4 columns each.
// All of B (K x K) and the transposed A tile are staged in shared memory with
// every 16-byte load of a thread issued before the first use (one L2 round
// trip per CTA instead of one per loop iteration).
template <int K>
constexpr size_t agg_gemm_smem() {
    return sizeof(float) * ((size_t)K * K + (size_t)K * (4096 / K + 4));
}

template <int K, bool TRANS_B>
__global__ void __launch_bounds__(256)
    agg_gemm_kernel(const float *__restrict__ A, const float *__restrict__ W, int64_t n,
                    float *__restrict__ out, const float *__restrict__ addend,
                    const int32_t *__restrict__ add_rows, float add_scale) {
    constexpr int TM = 4096 / K;
    constexpr int LDA = TM + 4;
    constexpr int CG = K / 4;  // column groups of 4
    constexpr int NWV = K * K / 4;                // float4 of B
    constexpr int WV = (NWV + 255) / 256;         // per thread
    constexpr int AV = TM * K / 4 / 256;  // float4 of A per thread (= 4)
    extern __shared__ __align__(16) float gsm[];
    float *Ws = gsm;           // [K][K]: Ws[k*K + j] = B(k, j)
    float *As = gsm + K * K;   // [K][LDA]: As[k*LDA + r] = A[m0 + r][k]
    const int t = threadIdx.x;
    const int cg = t % CG, rg = t / CG;
    const int64_t m0 = (int64_t)blockIdx.x * TM;
    {
        float4 wv[WV];
        float4 av[AV];
#pragma unroll
        for (int q = 0; q < WV; ++q)
            if (t + q * 256 < NWV) wv[q] = reinterpret_cast<const float4 *>(W)[t + q * 256];
#pragma unroll
        for (int q = 0; q < AV; ++q) {
            const int f = t + q * 256;  // float4 index in the TM x K tile
            const int r = f / CG;
            const int64_t m = m0 + r;
            av[q] = m < n ? reinterpret_cast<const float4 *>(A + m * K)[f % CG]
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < WV; ++q) {
            const int f = t + q * 256;
            if (f >= NWV) break;
            const int row = f / CG, c = (f % CG) * 4;  // W[row][c..c+3]
            if (TRANS_B) {  // B(k, j) = W[j][k]: W[row][c+i] -> Ws[(c+i)*K + row]
                Ws[(c + 0) * K + row] = wv[q].x;
                Ws[(c + 1) * K + row] = wv[q].y;
                Ws[(c + 2) * K + row] = wv[q].z;
                Ws[(c + 3) * K + row] = wv[q].w;
            } else {
                *reinterpret_cast<float4 *>(Ws + row * K + c) = wv[q];
            }
        }
#pragma unroll
        for (int q = 0; q < AV; ++q) {
            const int f = t + q * 256;
            const int r = f / CG, c = (f % CG) * 4;
            As[(c + 0) * LDA + r] = av[q].x;
            As[(c + 1) * LDA + r] = av[q].y;
            As[(c + 2) * LDA + r] = av[q].z;
            As[(c + 3) * LDA + r] = av[q].w;
        }
    }
    __syncthreads();
    float acc[4][4] = {};
#pragma unroll 8
    for (int kk = 0; kk < K; ++kk) {
        const float4 a4 = *reinterpret_cast<const float4 *>(As + kk * LDA + rg * 4);
        const float4 b4 = *reinterpret_cast<const float4 *>(Ws + kk * K + cg * 4);
        const float av[4] = {a4.x, a4.y, a4.z, a4.w};
        const float bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + rg * 4 + i;
        if (m >= n) continue;
        float4 o = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (addend) {
            const float4 s =
                *reinterpret_cast<const float4 *>(addend + (int64_t)add_rows[m] * K + cg * 4);
            o.x = fmaf(add_scale, s.x, o.x);
            o.y = fmaf(add_scale, s.y, o.y);
            o.z = fmaf(add_scale, s.z, o.z);
            o.w = fmaf(add_scale, s.w, o.w);
        }
        *reinterpret_cast<float4 *>(out + m * K + cg * 4) = o;
    }
}

// ---- 4. W += scale * P^T . G ----------------------------------------------------
// grid.x = output tiles of TA x TA (TA = 16R), grid.y = chunks of RC pairs;
// a 16 x 16 thread grid, R x R outputs per thread, partial sums added with
// vector reductions.
// TO_ACCU: the partial sums go, unscaled, into the fp64 pending accumulator
// (pairs of a mini-batch that has not completed yet) instead of into W.
template <int K, bool TO_ACCU>
__global__ void __launch_bounds__(256)
    agg_wgrad_kernel(const float *__restrict__ P, const float *__restrict__ G, int64_t n,
                     int64_t rows_per_cta, float *__restrict__ W, double *__restrict__ accu,
                     float scale) {
    constexpr int R = K >= 64 ? 4 : (K == 32 ? 2 : 1);
    constexpr int TA = 16 * R;
    constexpr int TILES = K / TA;
    constexpr int MC = 32;
    __shared__ __align__(16) float Ps[MC][TA];
    __shared__ __align__(16) float Gs[MC][TA];
    const int t = threadIdx.x;
    const int ty = t / 16, tx = t % 16;
    const int a0 = (blockIdx.x / TILES) * TA, b0 = (blockIdx.x % TILES) * TA;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per_cta;
    const int64_t r1 = imin64(n, r0 + rows_per_cta);
    float acc[R][R] = {};
    constexpr int QV = MC * TA / 4 / 256 > 0 ? MC * TA / 4 / 256 : 1;  // float4 per thread
    constexpr int TV = TA / 4;
    for (int64_t mc = r0; mc < r1; mc += MC) {
        float4 pv[QV], gv[QV];
#pragma unroll
        for (int q = 0; q < QV; ++q) {
            const int f = t + q * 256;
            const int r = f / TV, c = (f % TV) * 4;
            const int64_t m = mc + r;
            const bool ok = f < MC * TV && m < r1;
            pv[q] = ok ? *reinterpret_cast<const float4 *>(P + m * K + a0 + c)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
            gv[q] = ok ? *reinterpret_cast<const float4 *>(G + m * K + b0 + c)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < QV; ++q) {
            const int f = t + q * 256;
            if (f < MC * TV) {
                const int r = f / TV, c = (f % TV) * 4;
                *reinterpret_cast<float4 *>(&Ps[r][c]) = pv[q];
                *reinterpret_cast<float4 *>(&Gs[r][c]) = gv[q];
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int r = 0; r < MC; ++r) {
            float av[R], bv[R];
#pragma unroll
            for (int i = 0; i < R; ++i) {
                av[i] = Ps[r][ty * R + i];
                bv[i] = Gs[r][tx * R + i];
            }
#pragma unroll
            for (int i = 0; i < R; ++i)
#pragma unroll
                for (int j = 0; j < R; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    if constexpr (TO_ACCU) {
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
            for (int j = 0; j < R; ++j)
                atomicAdd(accu + (int64_t)(a0 + ty * R + i) * K + b0 + tx * R + j,
                          (double)acc[i][j]);
        return;
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
        float *dst = W + (int64_t)(a0 + ty * R + i) * K + b0 + tx * R;
        if constexpr (R == 4) {
            red_add4(dst, scale * acc[i][0], scale * acc[i][1], scale * acc[i][2],
                     scale * acc[i][3]);
        } else if constexpr (R == 2) {
            red_add2(dst, scale * acc[i][0], scale * acc[i][1]);
        } else {
            atomicAdd(dst, scale * acc[i][0]);
        }
    }
}

// ---- 4a. flush of the pending accumulator once its mini-batch completes ----
// W = f32(f64(W) + scale * accu), accu = 0 (trainer.py:310-316)
__global__ void agg_flush_kernel(float *__restrict__ W, double *__restrict__ accu, int kk,
                                 double scale) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= kk) return;
    W[i] = (float)((double)W[i] + scale * accu[i]);
    accu[i] = 0.0;
}

// ---- 5b. history rows: T[h] -= lr * ((1-gamma)/len * WH[m] + l2 * T[h]) ---------
template <int K>
__global__ void __launch_bounds__(256)
    agg_hist_kernel(float *__restrict__ T, const int32_t *__restrict__ users, int64_t n,
                    const int64_t *__restrict__ off, const int32_t *__restrict__ hist,
                    int64_t max_history, float one_minus_gamma, const float *__restrict__ WH,
                    float lr, float l2) {
    constexpr int VW = K >= 32 ? K / 32 : 1;
    constexpr int ACT = K >= 32 ? 32 : K;
    const int lane = threadIdx.x & 31;
    const int64_t m = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (m >= n || lane >= ACT) return;
    const int64_t u = users[m];
    const int64_t hb = off[u];
    const int64_t he = imin64(off[u + 1], hb + max_history);
    if (he <= hb) return;
    const float sc = one_minus_gamma / (float)(he - hb);
    float wh[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) wh[i] = sc * WH[m * K + lane * VW + i];
    for (int64_t idx = hb; idx < he; ++idx) {
        float *row = T + (int64_t)hist[idx] * K + lane * VW;
        float d[VW];
#pragma unroll
        for (int i = 0; i < VW; ++i) d[i] = -lr * (wh[i] + (l2 != 0.f ? l2 * row[i] : 0.f));
        if constexpr (VW == 4) {
            red_add4(row, d[0], d[1], d[2], d[3]);
        } else if constexpr (VW == 2) {
            red_add2(row, d[0], d[1]);
        } else {
            atomicAdd(row, d[0]);
        }
    }
}

static int agg_step(int window) { return window > 0 ? window : 4096; }

size_t agg_hogwild_scratch_bytes(int K, int window) {
    // P, Q (reused for W.G), G: step x K float32 each
    return (size_t)3 * (size_t)agg_step(window) * (size_t)K * sizeof(float) + 256;
}

template <int K>
static cudaError_t run_agg(const HogwildArgs &base, const heat_agg_params &agg, void *scratch,
                           cudaStream_t st) {
    // the dynamic shared-memory opt-in is per device context: kernel_occupancy
    // applies it once per (device, kernel, size), under its lock
    cudaError_t oe;
    kernel_occupancy((const void *)agg_gemm_kernel<K, false>, 256, agg_gemm_smem<K>(), &oe);
    if (oe != cudaSuccess) return oe;
    kernel_occupancy((const void *)agg_gemm_kernel<K, true>, 256, agg_gemm_smem<K>(), &oe);
    if (oe != cudaSuccess) return oe;
    const int64_t C = agg_step(base.window);
    float *P = reinterpret_cast<float *>(scratch);
    float *Q = P + C * K;
    float *G = Q + C * K;
    const float omg = (float)(1.0 - agg.gamma);
    const float wscale = (float)(-agg.lr / (double)agg.mini_batch);
    for (int64_t s = base.start; s < base.stop; s += C) {
        const int64_t n = imin64(C, base.stop - s);
        const int32_t *us = base.users + s;
        const unsigned wblocks = (unsigned)((n + 7) / 8);
        agg_pool_kernel<K><<<wblocks, 256, 0, st>>>(base.T, us, n, agg.tr_offsets, agg.tr_items,
                                                    agg.max_history, omg, P);
        constexpr int TM = 4096 / K;
        constexpr size_t GSM = agg_gemm_smem<K>();
        const unsigned gblocks = (unsigned)((n + TM - 1) / TM);
        agg_gemm_kernel<K, false><<<gblocks, 256, GSM, st>>>(P, agg.W, n, Q, base.S, us,
                                                             (float)agg.gamma);
        HogwildArgs a = base;
        a.start = s;
        a.stop = s + n;
        a.window = (int)n;  // the whole step in flight: W is frozen within it
        a.query = Q;
        a.ugrad_out = G;
        a.ugamma = (float)agg.gamma;
        cudaError_t e = launch_hogwild_staged(a, st, nullptr, false);
        if (e != cudaSuccess) return e;
        constexpr int R = K >= 64 ? 4 : (K == 32 ? 2 : 1);
        constexpr int TILES = K / (16 * R);
        // ~2 CTAs per SM over the output tiles x pair chunks
        const int64_t want = std::max<int64_t>(1, 2 * sm_count() / (TILES * TILES));
        // the reference's flush schedule (trainer.py:300-316, one accumulator):
        // pair q of the epoch joins mini-batch q / mini_batch, whose
        // contributions reach W only once it is complete; an incomplete
        // batch waits in the fp64 accumulator (dropped at the epoch's end,
        // like the reference's per-epoch thread state).  c0 pairs of the
        // current batch precede this step.
        const int64_t mb = agg.mini_batch;
        const int64_t c0 = s % mb;
        const int64_t cut = std::min<int64_t>(n, std::max<int64_t>(0, (c0 + n) / mb * mb - c0));
        if (c0 > 0 && c0 + n >= mb && agg.accu) {  // the pending batch completes here
            const int kk = K * K;
            agg_flush_kernel<<<(kk + 255) / 256, 256, 0, st>>>(agg.W, agg.accu, kk,
                                                               -agg.lr / (double)mb);
        }
        auto wgrad = [&](int64_t r0, int64_t rn, bool to_accu) {
            if (rn <= 0) return;
            int64_t rpc = std::max<int64_t>(32, (rn + want - 1) / want);
            rpc = (rpc + 31) / 32 * 32;
            const dim3 wg((unsigned)(TILES * TILES), (unsigned)((rn + rpc - 1) / rpc));
            if (to_accu)
                agg_wgrad_kernel<K, true><<<wg, 256, 0, st>>>(P + r0 * K, G + r0 * K, rn, rpc,
                                                              agg.W, agg.accu, 1.f);
            else
                agg_wgrad_kernel<K, false><<<wg, 256, 0, st>>>(P + r0 * K, G + r0 * K, rn, rpc,
                                                               agg.W, nullptr, wscale);
        };
        if (agg.accu) {
            wgrad(0, cut, false);
            wgrad(cut, n - cut, true);
        } else {  // no accumulator given: every pair straight into W
            wgrad(0, n, false);
        }
        if (agg.history_grad) {
            agg_gemm_kernel<K, true><<<gblocks, 256, GSM, st>>>(G, agg.W, n, Q, nullptr,
                                                                nullptr, 0.f);
            agg_hist_kernel<K><<<wblocks, 256, 0, st>>>(base.T, us, n, agg.tr_offsets,
                                                        agg.tr_items, agg.max_history, omg, Q,
                                                        base.lr, base.l2);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_agg_hogwild(const HogwildArgs &base, const heat_agg_params &agg,
                               void *scratch, cudaStream_t st) {
    if (base.stop <= base.start) return cudaSuccess;
    if (((uintptr_t)base.S | (uintptr_t)base.T | (uintptr_t)agg.W | (uintptr_t)scratch) % 16)
        return cudaErrorNotSupported;
    switch (base.K) {
    case 16: return run_agg<16>(base, agg, scratch, st);
    case 32: return run_agg<32>(base, agg, scratch, st);
    case 64: return run_agg<64>(base, agg, scratch, st);
    case 128: return run_agg<128>(base, agg, scratch, st);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace heat
