// heat_eval.cu — Recall@K / NDCG@K over the full catalog.
//
// Restates /root/reference/pkg/src/heatcf/evaluator.py:140-172 for the
// non-aggregated query: binary64 cosine (or dot) scores of every item for a
// user, the user's train positives masked (evaluator.py:64-65), the top k
// ranked by (score desc, item id asc) (evaluator.py:61-73), hits against the
// sorted test slice, recall = hits / n_test, NDCG = sum over hit ranks of
// 1/log2(r+1) / IDCG[min(k, n_test)] (evaluator.py:164-172; the two weight
// tables come from the host in the reference's arithmetic).
//
// One CTA scores UB users against 64-item tiles of T staged in shared memory
// (fp64 FMA dot products; scores are a pure function of (user, item), so
// exact ties stay exact ties), then each warp merges its users' candidates
// into a sorted top-k list kept in shared memory.  Items stream in increasing
// id order, so a candidate that ties the current k-th score never displaces
// it (the incumbent has the lower id) — exactly the reference's tie rule.
#include <cfloat>
#include <cstdint>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

constexpr int kEvalThreads = 256;
constexpr int kEvalWarps = kEvalThreads / 32;
constexpr int kIT = 64;  // items per tile

template <int UB>
struct EvalLayout {
    static constexpr int TPU = kEvalThreads / UB;  // threads per user in scoring
    static constexpr int IPT = kIT / TPU;          // items per thread
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

template <int UB>
__host__ __device__ inline size_t eval_smem_bytes(int K, int k) {
    size_t b = 0;
    b += align16(sizeof(double) * UB * (K + 1));    // uvec (padded rows)
    b += align16(sizeof(double) * UB);              // unorm
    b += align16(sizeof(float) * kIT * (K + 1));    // item tile (padded rows)
    b += align16(sizeof(double) * kIT);             // inorm
    b += align16(sizeof(double) * UB * kIT);        // scores
    b += align16(sizeof(double) * UB * k);          // list scores
    b += align16(sizeof(int32_t) * UB * k);         // list ids
    b += align16(sizeof(int32_t) * UB);             // list sizes
    b += align16(sizeof(int64_t) * UB);             // exclusion cursors
    return b;
}

template <int UB>
__global__ void __launch_bounds__(kEvalThreads)
    eval_kernel(const void *__restrict__ S, int s_f64, const float *__restrict__ T, int64_t t_rows,
                int K,
                const int32_t *__restrict__ users, int64_t n_users,
                const int64_t *__restrict__ tr_off, const int32_t *__restrict__ tr_items,
                int64_t tr_num_users, const int64_t *__restrict__ te_off,
                const int32_t *__restrict__ te_items, int k, int cosine,
                const double *__restrict__ dcg_w, const double *__restrict__ idcg,
                int32_t *__restrict__ topk, double *__restrict__ recall,
                double *__restrict__ ndcg) {
    using L = EvalLayout<UB>;
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char *ptr = smem;
    double *uvec = reinterpret_cast<double *>(ptr); ptr += align16(sizeof(double) * UB * (K + 1));
    double *unorm = reinterpret_cast<double *>(ptr); ptr += align16(sizeof(double) * UB);
    float *tile = reinterpret_cast<float *>(ptr); ptr += align16(sizeof(float) * kIT * (K + 1));
    double *inorm = reinterpret_cast<double *>(ptr); ptr += align16(sizeof(double) * kIT);
    double *scores = reinterpret_cast<double *>(ptr); ptr += align16(sizeof(double) * UB * kIT);
    double *ls = reinterpret_cast<double *>(ptr); ptr += align16(sizeof(double) * UB * k);
    int32_t *lid = reinterpret_cast<int32_t *>(ptr); ptr += align16(sizeof(int32_t) * UB * k);
    int32_t *ln = reinterpret_cast<int32_t *>(ptr); ptr += align16(sizeof(int32_t) * UB);
    int64_t *cur = reinterpret_cast<int64_t *>(ptr);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ubase = (int64_t)blockIdx.x * UB;
    const int nub = (int)imin64(UB, n_users - ubase);

    // user vectors (binary64), norms, list state, exclusion cursors
    for (int i = tid; i < UB * K; i += kEvalThreads) {
        int b = i / K, c = i % K;
        if (b < nub) {
            const int64_t off = (int64_t)users[ubase + b] * K + c;
            uvec[b * (K + 1) + c] = s_f64 ? reinterpret_cast<const double *>(S)[off]
                                          : (double)reinterpret_cast<const float *>(S)[off];
        } else {
            uvec[b * (K + 1) + c] = 0.0;
        }
    }
    __syncthreads();
    if (tid < UB) {
        double a = 0.0;
        for (int c = 0; c < K; ++c) a = fma(uvec[tid * (K + 1) + c], uvec[tid * (K + 1) + c], a);
        unorm[tid] = sqrt(a);
        ln[tid] = 0;
        int64_t u = tid < nub ? users[ubase + tid] : 0;
        cur[tid] = (tid < nub && u < tr_num_users) ? tr_off[u] : 0;
    }

    const int ub_s = tid / L::TPU;  // scoring: my user
    const int q = tid % L::TPU;     // scoring: my item lane

    for (int64_t i0 = 0; i0 < t_rows; i0 += kIT) {
        __syncthreads();
        // stage the item tile (coalesced rows) and its norms
        const int nit = (int)imin64(kIT, t_rows - i0);
        for (int i = tid; i < kIT * K; i += kEvalThreads) {
            int r = i / K, c = i % K;
            tile[r * (K + 1) + c] = r < nit ? T[(i0 + r) * K + c] : 0.f;
        }
        __syncthreads();
        if (tid < kIT) {
            double a = 0.0;
            for (int c = 0; c < K; ++c) {
                double x = (double)tile[tid * (K + 1) + c];
                a = fma(x, x, a);
            }
            inorm[tid] = sqrt(a);
        }
        // scores
        double acc[L::IPT];
#pragma unroll
        for (int m = 0; m < L::IPT; ++m) acc[m] = 0.0;
        const double *uv = uvec + ub_s * (K + 1);
        for (int c = 0; c < K; ++c) {
            const double x = uv[c];
#pragma unroll
            for (int m = 0; m < L::IPT; ++m)
                acc[m] = fma(x, (double)tile[(q + L::TPU * m) * (K + 1) + c], acc[m]);
        }
        __syncthreads();  // inorm ready
#pragma unroll
        for (int m = 0; m < L::IPT; ++m) {
            const int it = q + L::TPU * m;
            double s = acc[m];
            if (cosine) {
                const double un = unorm[ub_s], in = inorm[it];
                s = (un == 0.0 || in == 0.0) ? 0.0 : s / (un * in);
            }
            if (it >= nit) s = -INFINITY;
            scores[ub_s * kIT + it] = s;
        }
        __syncthreads();
        // per-user: mask train positives in this tile, merge candidates
        for (int b = warp; b < nub; b += kEvalWarps) {
            const int64_t u = users[ubase + b];
            double *srow = scores + b * kIT;
            if (u < tr_num_users) {
                const int64_t end = tr_off[u + 1];
                int64_t c0 = cur[b];
                while (true) {
                    int64_t idx = c0 + lane;
                    int64_t item = idx < end ? (int64_t)tr_items[idx] : INT64_MAX;
                    bool in_tile = item < i0 + kIT;
                    if (in_tile) srow[item - i0] = -INFINITY;
                    unsigned m = __ballot_sync(0xffffffffu, in_tile);
                    c0 += __popc(m);
                    if (m != 0xffffffffu) break;
                }
                __syncwarp();
                if (lane == 0) cur[b] = c0;
            }
            double *lsb = ls + b * k;
            int32_t *lidb = lid + b * k;
            int n = ln[b];
            for (int qq = 0; qq < kIT / 32; ++qq) {
                const int it = lane + 32 * qq;
                const double s = srow[it];
                const double kth = n == k ? lsb[k - 1] : -INFINITY;
                bool cand = s != -INFINITY && (n < k || s > kth);
                unsigned m = __ballot_sync(0xffffffffu, cand);
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const double cs = __shfl_sync(0xffffffffu, s, src);
                    const int32_t cid = (int32_t)(i0 + src + 32 * qq);
                    if (n == k && !(cs > lsb[k - 1])) continue;
                    // insertion point: entries strictly better than (cs, cid)
                    int posn = 0;
                    for (int e0 = 0; e0 < n; e0 += 32) {
                        int e = e0 + lane;
                        bool better = e < n && (lsb[e] > cs || (lsb[e] == cs && lidb[e] < cid));
                        posn += __popc(__ballot_sync(0xffffffffu, better));
                    }
                    const int newn = n < k ? n + 1 : k;
                    // shift [posn, newn-1) up by one, top chunk first
                    for (int hi = newn - 1; hi > posn; hi -= 32) {
                        int dst = hi - lane;
                        bool mv = dst > posn;
                        double vs = 0.0;
                        int32_t vi = 0;
                        if (mv) { vs = lsb[dst - 1]; vi = lidb[dst - 1]; }
                        __syncwarp();
                        if (mv) { lsb[dst] = vs; lidb[dst] = vi; }
                        __syncwarp();
                    }
                    if (lane == 0 && posn < k) { lsb[posn] = cs; lidb[posn] = cid; }
                    __syncwarp();
                    n = newn;
                }
            }
            if (lane == 0) ln[b] = n;
            __syncwarp();
        }
    }
    __syncthreads();
    // hits / recall / NDCG, one warp per user; ranks summed in order
    for (int b = warp; b < nub; b += kEvalWarps) {
        const int64_t ug = ubase + b;
        const int64_t u = users[ug];
        const int n = ln[b];
        if (topk)
            for (int e = lane; e < k; e += 32) topk[ug * k + e] = e < n ? lid[b * k + e] : -1;
        if (lane == 0) {
            const int64_t tb = te_off[u], te = te_off[u + 1];
            const int64_t nt = te - tb;
            int hits = 0;
            double dcg = 0.0;
            for (int r = 0; r < n; ++r) {
                const int32_t item = lid[b * k + r];
                int64_t lo = tb, hi2 = te;
                while (lo < hi2) {
                    int64_t mid = (lo + hi2) >> 1;
                    if (te_items[mid] < item) lo = mid + 1; else hi2 = mid;
                }
                if (lo < te && te_items[lo] == item) {
                    ++hits;
                    dcg += dcg_w[r];
                }
            }
            recall[ug] = (double)hits / (double)nt;
            ndcg[ug] = dcg / idcg[(k < nt ? k : nt) - 1];
        }
    }
}

template <int UB>
static cudaError_t launch_eval_ub(const void *S, int s_f64, const float *T, int64_t t_rows, int K,
                                  const int32_t *users, int64_t n_users, const int64_t *tr_off,
                                  const int32_t *tr_items, int64_t tr_nu, const int64_t *te_off,
                                  const int32_t *te_items, int k, int cosine, const double *dw,
                                  const double *idcg, int32_t *topk, double *rec, double *nd,
                                  cudaStream_t st) {
    size_t smem = eval_smem_bytes<UB>(K, k);
    cudaError_t e = cudaFuncSetAttribute(eval_kernel<UB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t blocks = (n_users + UB - 1) / UB;
    eval_kernel<UB><<<(unsigned)blocks, kEvalThreads, smem, st>>>(
        S, s_f64, T, t_rows, K, users, n_users, tr_off, tr_items, tr_nu, te_off, te_items, k, cosine, dw,
        idcg, topk, rec, nd);
    return cudaGetLastError();
}

cudaError_t launch_eval(const void *S, int s_f64, const float *T, int64_t t_rows, int K,
                        const int32_t *users, int64_t n_users, const int64_t *tr_offsets,
                        const int32_t *tr_items, int64_t tr_num_users, const int64_t *te_offsets,
                        const int32_t *te_items, int k, int cosine, const double *dcg_w,
                        const double *idcg, int32_t *topk, double *recall, double *ndcg,
                        cudaStream_t stream) {
    if (n_users == 0) return cudaSuccess;
    const size_t cap = 200 * 1024;
    if (eval_smem_bytes<32>(K, k) <= cap)
        return launch_eval_ub<32>(S, s_f64, T, t_rows, K, users, n_users, tr_offsets, tr_items,
                                  tr_num_users, te_offsets, te_items, k, cosine, dcg_w, idcg,
                                  topk, recall, ndcg, stream);
    if (eval_smem_bytes<8>(K, k) <= cap)
        return launch_eval_ub<8>(S, s_f64, T, t_rows, K, users, n_users, tr_offsets, tr_items,
                                 tr_num_users, te_offsets, te_items, k, cosine, dcg_w, idcg,
                                 topk, recall, ndcg, stream);
    return cudaErrorInvalidValue;
}

// Aggregated query vectors for evaluation (evaluator.py:91-110):
// out[u] = gamma*S[u] + (1-gamma) * mean(first max_history train rows) . W,
// binary64, one CTA per user.
__global__ void aggregate_users_kernel(const float *__restrict__ S, const float *__restrict__ T,
                                       const float *__restrict__ W,
                                       const int64_t *__restrict__ tr_off,
                                       const int32_t *__restrict__ tr_items, int64_t tr_num_users,
                                       int K, double gamma, int64_t max_history,
                                       double *__restrict__ out) {
    extern __shared__ double pooled[];
    const int64_t u = blockIdx.x;
    int64_t hb = 0, n = 0;
    if (u < tr_num_users) {
        hb = tr_off[u];
        n = tr_off[u + 1] - hb;
        if (n > max_history) n = max_history;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        double a = 0.0;
        for (int64_t i = 0; i < n; ++i) a += (double)T[(int64_t)tr_items[hb + i] * K + k];
        pooled[k] = n > 0 ? a / (double)n : 0.0;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        double a = 0.0;
        for (int k = 0; k < K; ++k) a = fma(pooled[k], (double)W[k * K + j], a);
        out[u * K + j] = gamma * (double)S[u * K + j] + (1.0 - gamma) * a;
    }
}

cudaError_t launch_aggregate_users(const float *S, const float *T, const float *W,
                                   const int64_t *tr_off, const int32_t *tr_items,
                                   int64_t n_users, int64_t tr_num_users, int K, double gamma,
                                   int64_t max_history, double *out, cudaStream_t st) {
    if (n_users == 0) return cudaSuccess;
    int threads = K < 128 ? 64 : 128;
    aggregate_users_kernel<<<(unsigned)n_users, threads, K * sizeof(double), st>>>(
        S, T, W, tr_off, tr_items, tr_num_users, K, gamma, max_history, out);
    return cudaGetLastError();
}

size_t eval_max_k_supported(int K) {
    size_t k = 1;
    while (eval_smem_bytes<8>(K, (int)(k * 2)) <= 200 * 1024 && k < (1u << 20)) k *= 2;
    return k;
}

}  // namespace heat
