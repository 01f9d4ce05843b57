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
// Three kernels, the fastest that fits is launched (launch_eval):
//  * eval_fr_kernel (default, K % 4 == 0 and K <= 128): FP64 tensor path
//    (mma.sync m8n8k4), a warp owns 8 users, scores screened in registers,
//    lists merged by eval_finish_kernel when the catalog is cut into ranges;
//  * eval_rb_kernel (HEAT_EVAL_RB=1): round 1's register-blocked kernel, the
//    scores of a 32 x 128 tile through shared memory;
//  * eval_kernel: the plain one below, for any K and k.
// The plain kernel: one CTA scores UB users against 64-item tiles of T staged
// in shared memory (fp64 FMA dot products; scores are a pure function of
// (user, item), so exact ties stay exact ties), then each warp merges its
// users' candidates into a sorted top-k list kept in shared memory.  Items
// stream in increasing id order, so a candidate that ties the current k-th
// score never displaces it (the incumbent has the lower id) — exactly the
// reference's tie rule.
#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

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

// ---- register-blocked variant (K <= 128): warp w scores users 4w..4w+3
// against a 128-item tile, lane owns items lane + 32 m (m < 4): 16 binary64
// dot products per thread, 16 DFMA per 6 shared loads.  The warp merges its
// own users straight from registers (no score buffer, two barriers per tile).
// A candidate is screened by score * (1/unorm) * (1/inorm) against the list's
// k-th score; only survivors get the exact s / (unorm * inorm) of
// evaluator.py:48-58, so the list holds exactly the values the plain kernel
// computes (and the reference's division).  The next tile is prefetched
// into registers while the current one is scored.
constexpr int kRbUsers = 32;
constexpr int kRbItems = 128;
// The MMA variant keeps the tile in binary64 (converted once when it is
// stored, not once per fragment load: every tile element is a B operand of
// four warps) and, so that this costs no shared memory, writes the tile's
// scores over the tile itself once every warp has finished its products.
// EVAL_TILE_F32=1 restores the float tile with a separate score buffer.
#ifndef EVAL_TILE_F32
#define EVAL_TILE_F32 0
#endif
template <bool MMA>
using RbTile = std::conditional_t<MMA && EVAL_TILE_F32 == 0, double, float>;
template <bool MMA>
constexpr bool kRbAlias = MMA && EVAL_TILE_F32 == 0;

// MMA variant: the 32 x 128 x K product of a tile on the FP64 tensor path
// (mma.sync m8n8k4 f64; tcgen05 has no binary64 kind), the user matrix and
// the tile padded so fragment loads are bank-conflict-free, and the scores
// through shared memory into the same merge.
template <bool MMA>
__host__ __device__ constexpr int rb_ldu() { return MMA ? kRbUsers + 4 : kRbUsers; }
template <bool MMA>
__host__ __device__ inline int rb_ldt(int K) { return MMA ? K + 4 : K + 1; }
// tile-score rows padded by 64 B: a quarter-warp's 16-byte stores (two users,
// four column pairs) land in distinct banks
constexpr int kRbScoreLd = kRbItems + 8;

template <bool MMA = false>
__host__ __device__ inline size_t eval_rb_smem_bytes(int K, int k) {
    size_t b = 0;
    b += align16(sizeof(double) * K * rb_ldu<MMA>());        // user vectors, transposed
    const size_t tile = align16(sizeof(RbTile<MMA>) * kRbItems * rb_ldt<MMA>(K));  // padded rows
    const size_t score = MMA ? align16(sizeof(double) * kRbUsers * kRbScoreLd) : 0;
    b += kRbAlias<MMA> ? (tile > score ? tile : score) : tile + score;  // (scores over the tile)
    b += align16(sizeof(double) * kRbUsers * k);     // list scores
    b += align16(sizeof(int32_t) * kRbUsers * k);    // list ids
    b += align16(sizeof(uint32_t) * kRbUsers * 4);   // train-positive mask of the tile
    b += align16(sizeof(double) * kRbUsers * 2);     // user norms and reciprocals
    b += align16(sizeof(int64_t) * kRbUsers * 3);    // train cursors, ends, next train item
    return b;
}

__global__ void item_norms_kernel(const float *__restrict__ T, int64_t t_rows, int K,
                                  double *__restrict__ norm, double *__restrict__ rnorm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= t_rows) return;
    double a = 0.0;
    for (int c = 0; c < K; ++c) {
        const double x = (double)T[i * K + c];
        a = fma(x, x, a);
    }
    const double n = sqrt(a);
    norm[i] = n;
    rnorm[i] = n > 0.0 ? 1.0 / n : 0.0;
}

template <int KC, bool MMA>  // KC: K rounded up to a multiple of 4 for the staging loads
__global__ void __launch_bounds__(256)
    eval_rb_kernel(const void *__restrict__ S, int s_f64, const float *__restrict__ T,
                   int64_t t_rows, int K, const double *__restrict__ inorm_g,
                   const double *__restrict__ rinorm_g, const int32_t *__restrict__ users,
                   int64_t n_users, const int64_t *__restrict__ tr_off,
                   const int32_t *__restrict__ tr_items, int64_t tr_num_users,
                   const int64_t *__restrict__ te_off, const int32_t *__restrict__ te_items,
                   int k, int cosine, const double *__restrict__ dcg_w,
                   const double *__restrict__ idcg, int32_t *__restrict__ topk,
                   double *__restrict__ recall, double *__restrict__ ndcg) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char *ptr = smem;
    constexpr int LDU = rb_ldu<MMA>();
    const int LDT = rb_ldt<MMA>(K);
    double *uT = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * K * LDU);
    using TileT = RbTile<MMA>;
    TileT *tile = reinterpret_cast<TileT *>(ptr);
    double *tscore = reinterpret_cast<double *>(ptr);  // MMA: [32 users][128 items]
    {
        const size_t tb = align16(sizeof(TileT) * kRbItems * LDT);
        const size_t sb = MMA ? align16(sizeof(double) * kRbUsers * kRbScoreLd) : 0;
        if constexpr (kRbAlias<MMA>) {
            ptr += tb > sb ? tb : sb;
        } else {
            tscore = reinterpret_cast<double *>(ptr + tb);
            ptr += tb + sb;
        }
    }
    double *ls = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * kRbUsers * k);
    int32_t *lid = reinterpret_cast<int32_t *>(ptr);
    ptr += align16(sizeof(int32_t) * kRbUsers * k);
    uint32_t *pmask = reinterpret_cast<uint32_t *>(ptr);
    ptr += align16(sizeof(uint32_t) * kRbUsers * 4);
    double *unv = reinterpret_cast<double *>(ptr);  // [0, 32) norms, [32, 64) reciprocals
    ptr += align16(sizeof(double) * kRbUsers * 2);
    // [0, 32) cursors, [32, 64) ends, [64, 96) the item at the cursor
    // (INT64_MAX when exhausted): a tile below it has no train positive
    int64_t *curv = reinterpret_cast<int64_t *>(ptr);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t ubase = (int64_t)blockIdx.x * kRbUsers;
    const int nub = (int)imin64(kRbUsers, n_users - ubase);
    for (int i = tid; i < kRbUsers * K; i += 256) {
        const int b = i / K, c = i % K;
        double v = 0.0;
        if (b < nub) {
            const int64_t off = (int64_t)users[ubase + b] * K + c;
            v = s_f64 ? reinterpret_cast<const double *>(S)[off]
                      : (double)reinterpret_cast<const float *>(S)[off];
        }
        uT[c * LDU + b] = v;
    }
    __syncthreads();
    // user norms, train cursors (shared), list sizes (registers)
    if (tid < kRbUsers) {
        const int b = tid;
        double a = 0.0;
        for (int c = 0; c < K; ++c) a = fma(uT[c * LDU + b], uT[c * LDU + b], a);
        const double n = sqrt(a);
        unv[b] = n;
        unv[kRbUsers + b] = n > 0.0 ? 1.0 / n : 0.0;
        const int64_t u = b < nub ? users[ubase + b] : 0;
        const bool has = b < nub && u < tr_num_users;
        curv[b] = has ? tr_off[u] : 0;
        curv[kRbUsers + b] = has ? tr_off[u + 1] : 0;
        curv[2 * kRbUsers + b] =
            (has && tr_off[u] < tr_off[u + 1]) ? (int64_t)tr_items[tr_off[u]] : INT64_MAX;
    }
    int n_l[4] = {0, 0, 0, 0};
    // tile staging: 128 rows x K floats, float4 loads held in registers
    constexpr int PER = (kRbItems * KC / 4 + 255) / 256;  // float4 per thread
    float4 pre[PER];
    auto load_tile = [&](int64_t i0) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int f = tid + q * 256;  // float4 index within the tile
            const int r = f / (KC / 4), c4 = f % (KC / 4);
            const int64_t row = i0 + r;
            pre[q] = (r < kRbItems && row < t_rows && c4 * 4 < K)
                         ? *reinterpret_cast<const float4 *>(T + row * K + c4 * 4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_tile = [&]() {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int f = tid + q * 256;
            const int r = f / (KC / 4), c = (f % (KC / 4)) * 4;
            if (r < kRbItems && c < K) {
                TileT *d = tile + r * LDT + c;
                if constexpr (sizeof(TileT) == 8) {  // (LDT even, c % 4 == 0: 16-byte aligned)
                    *reinterpret_cast<double2 *>(d) = make_double2(pre[q].x, pre[q].y);
                    *reinterpret_cast<double2 *>(d + 2) = make_double2(pre[q].z, pre[q].w);
                } else {
                    d[0] = pre[q].x; d[1] = pre[q].y; d[2] = pre[q].z; d[3] = pre[q].w;
                }
            }
        }
    };
    load_tile(0);
    for (int64_t i0 = 0; i0 < t_rows; i0 += kRbItems) {
        __syncthreads();  // previous tile consumed
        store_tile();
        // this tile's train positives per user -> 128-bit masks
        if (lane < 4)
            for (int j = 0; j < 4; ++j) pmask[(warp * 4 + j) * 4 + lane] = 0u;
        __syncthreads();
        if (i0 + kRbItems < t_rows) load_tile(i0 + kRbItems);  // overlaps the scoring
        for (int j = 0; j < 4; ++j) {
            const int b = warp * 4 + j;
            if (curv[2 * kRbUsers + b] >= i0 + kRbItems) continue;  // (warp-uniform)
            int64_t c0 = curv[b];
            const int64_t cend = curv[kRbUsers + b];
            while (c0 < cend) {
                const int64_t idx = c0 + lane;
                const int64_t item = idx < cend ? (int64_t)tr_items[idx] : INT64_MAX;
                const bool in_tile = item < i0 + kRbItems;
                if (in_tile) {
                    const int o = (int)(item - i0);
                    atomicOr(&pmask[(warp * 4 + j) * 4 + (o >> 5)], 1u << (o & 31));
                }
                const unsigned m = __ballot_sync(0xffffffffu, in_tile);
                c0 += __popc(m);
                if (m != 0xffffffffu) break;
            }
            __syncwarp();
            if (lane == 0) {
                curv[b] = c0;
                curv[2 * kRbUsers + b] = c0 < cend ? (int64_t)tr_items[c0] : INT64_MAX;
            }
        }
        __syncwarp();
        // 4 users x 4 items of dot products per lane
        double acc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[j][m] = 0.0;
        if constexpr (MMA) {
            // warp w: users 8*(w/2) .. +7, items 64*(w%2) .. +63 as 8 m8n8k4 tiles
            const int g = lane >> 2, tq = lane & 3;
            const int ub = warp >> 1, ih = warp & 1;
            double c0[8], c1[8];
#pragma unroll
            for (int ni = 0; ni < 8; ++ni) c0[ni] = c1[ni] = 0.0;
            const double *ucol = uT + 8 * ub + g;
            const TileT *trow = tile + (size_t)(64 * ih + g) * LDT + tq;
            for (int k0 = 0; k0 < K; k0 += 4) {
                const double av = ucol[(k0 + tq) * LDU];  // A[user g][k0 + tq]
#pragma unroll
                for (int ni = 0; ni < 8; ++ni) {
                    const double bv = (double)trow[(size_t)8 * ni * LDT + k0];  // B[k][item]
                    asm volatile(
                        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
                        "{%0, %1};"
                        : "+d"(c0[ni]), "+d"(c1[ni])
                        : "d"(av), "d"(bv));
                }
            }
            if constexpr (kRbAlias<MMA>) __syncthreads();  // every warp is done with the tile
            double *srow = tscore + (size_t)(8 * ub + g) * kRbScoreLd + 64 * ih + 2 * tq;
#pragma unroll
            for (int ni = 0; ni < 8; ++ni)
                *reinterpret_cast<double2 *>(srow + 8 * ni) = make_double2(c0[ni], c1[ni]);
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    acc[j][m] = tscore[(warp * 4 + j) * kRbScoreLd + lane + 32 * m];
        } else {
            const double *ucol = uT + warp * 4;
            for (int c = 0; c < K; ++c) {
                const double2 ua = *reinterpret_cast<const double2 *>(ucol + c * LDU);
                const double2 ub = *reinterpret_cast<const double2 *>(ucol + c * LDU + 2);
                const double uv[4] = {ua.x, ua.y, ub.x, ub.y};
                double iv[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) iv[m] = (double)tile[(lane + 32 * m) * LDT + c];
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int m = 0; m < 4; ++m) acc[j][m] = fma(uv[j], iv[m], acc[j][m]);
            }
        }
        __syncwarp();
        // this lane's four items of the tile: reciprocal norms for the screen
        // (0 past the table: such a slot can only pass the screen when the
        // k-th score is <= 0, and the merge below rejects it as invalid)
        double rin[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int64_t item = i0 + lane + 32 * m;
            rin[m] = (cosine && item < t_rows) ? rinorm_g[item] : 0.0;
        }
        // merge, one user at a time (items in increasing id order per lane
        // group; the tie rule keeps the lower id, so order of arrival within
        // equal scores does not matter: the insertion point compares ids)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int b = warp * 4 + j;
            if (b >= nub) continue;
            double *lsb = ls + b * k;
            int32_t *lidb = lid + b * k;
            int n = n_l[j];
            // Screen of the whole tile for this user, before anything else is
            // looked at: once the list is full almost no tile holds a score
            // near the k-th one.  The test is the merge's own approximate
            // screen (same expression, same slack) without the validity and
            // mask lookups, so it passes a superset of the merge's candidates.
            if (n == k) {
                const double lim = lsb[k - 1] - 1e-9;
                const double run = cosine ? unv[kRbUsers + b] : 1.0;
                bool any = false;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const double approx = cosine ? acc[j][m] * run * rin[m] : acc[j][m];
                    any |= !(approx < lim);
                }
                if (!__any_sync(0xffffffffu, any)) continue;
            }
            for (int m = 0; m < 4; ++m) {
                const int o = lane + 32 * m;
                const int64_t item = i0 + o;
                const bool valid = item < t_rows &&
                                   !((pmask[b * 4 + (o >> 5)] >> (o & 31)) & 1u);
                double s = acc[j][m];
                const double kth = n == k ? lsb[k - 1] : -INFINITY;
                bool cand = valid;
                if (cand && n == k && cosine) {  // screen: approximate cosine
                    const double approx = s * unv[kRbUsers + b] * rinorm_g[item];
                    cand = approx >= kth - 1e-9;
                }
                double ex = s;
                if (cand && cosine) {
                    const double in = inorm_g[item], un = unv[b];
                    ex = (un == 0.0 || in == 0.0) ? 0.0 : s / (un * in);
                }
                if (cand && n == k) cand = ex > kth || (ex == kth && false);
                unsigned mk = __ballot_sync(0xffffffffu, cand);
                while (mk) {
                    const int src = __ffs(mk) - 1;
                    mk &= mk - 1;
                    const double cs = __shfl_sync(0xffffffffu, ex, src);
                    const int32_t cid = (int32_t)(i0 + src + 32 * m);
                    if (n == k && !(cs > lsb[k - 1] ||
                                    (cs == lsb[k - 1] && cid < lidb[k - 1])))
                        continue;
                    int posn = 0;
                    for (int e0 = 0; e0 < n; e0 += 32) {
                        const int e = e0 + lane;
                        const bool better = e < n && (lsb[e] > cs || (lsb[e] == cs && lidb[e] < cid));
                        posn += __popc(__ballot_sync(0xffffffffu, better));
                    }
                    const int newn = n < k ? n + 1 : k;
                    for (int hi = newn - 1; hi > posn; hi -= 32) {
                        const int dst = hi - lane;
                        const bool mv = dst > posn;
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
            n_l[j] = n;
        }
    }
    // hits / recall / NDCG, one lane per user of the warp; ranks in order
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int b = warp * 4 + j;
        if (b >= nub) continue;
        const int64_t ug = ubase + b;
        const int64_t u = users[ug];
        const int n = n_l[j];
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
                    const int64_t mid = (lo + hi2) >> 1;
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

// ---- fragment-resident variant (K % 4 == 0, K <= 128; the default) ----------
// The same FP64 tensor-path product, re-tiled so that the scores never leave
// the registers: a CTA holds 64 users, warp w OWNS users 8w .. 8w+7 and
// scores them against a 64-item tile (8 m8n8k4 tiles, 16 accumulators per
// thread), the tile kept in binary64 (converted once when stored).  Each
// thread screens its own 16 scores of user 8w + (lane >> 2) against that
// user's limit — (k-th score - 2e-9) / (1 / |u|), so one multiply by the
// item's reciprocal norm and one compare per score — and only a warp with a
// survivor enters the merge, which is the register-blocked kernel's (exact
// cosine s / (|u| |v|) as evaluator.py:48-58 divides it, order (score desc,
// id asc), train positives masked).  A warp is the only writer of its users'
// lists, so a tile costs two CTA barriers (tile stored / tile consumed) and
// no score buffer: the register-blocked kernel above spent a quarter of its
// stall samples on four barriers per 128 items (profiles/r02_ncu_eval.txt).
constexpr int kFrUsers = 64;
constexpr int kFrItems = 64;

__host__ __device__ inline size_t eval_fr_smem_bytes(int K, int k) {
    size_t b = 0;
    b += align16(sizeof(double) * K * (kFrUsers + 4));  // user vectors, transposed
    b += align16(sizeof(double) * kFrItems * (K + 4));  // item tile, binary64, padded rows
    b += align16(sizeof(double) * kFrItems);            // reciprocal item norms of the tile
    b += align16(sizeof(double) * kFrUsers * k);        // list scores
    b += align16(sizeof(int32_t) * kFrUsers * k);       // list ids
    b += align16(sizeof(uint32_t) * kFrUsers * 2);      // train-positive mask of the tile
    b += align16(sizeof(double) * kFrUsers * 3);        // user norm, reciprocal, screen limit
    b += align16(sizeof(int64_t) * kFrUsers * 3);       // train cursor, end, item at the cursor
    b += align16(sizeof(int32_t) * kFrUsers);           // list sizes
    return b;
}

template <int KC>
__global__ void __launch_bounds__(256, 2)
    eval_fr_kernel(const void *__restrict__ S, int s_f64, const float *__restrict__ T,
                   int64_t t_rows, int K, const double *__restrict__ inorm_g,
                   const double *__restrict__ rinorm_g, const int32_t *__restrict__ users,
                   int64_t n_users, const int64_t *__restrict__ tr_off,
                   const int32_t *__restrict__ tr_items, int64_t tr_num_users,
                   const int64_t *__restrict__ te_off, const int32_t *__restrict__ te_items,
                   int k, int cosine, int nsplit, int64_t split_items,
                   double *__restrict__ part_scores, int32_t *__restrict__ part_ids,
                   int32_t *__restrict__ part_n) {
    extern __shared__ __align__(16) unsigned char smem[];
    unsigned char *ptr = smem;
    constexpr int LDU = kFrUsers + 4;
    const int LDT = K + 4;
    double *uT = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * K * LDU);
    double *tile = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * kFrItems * LDT);
    double *rin = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * kFrItems);
    double *ls = reinterpret_cast<double *>(ptr);
    ptr += align16(sizeof(double) * kFrUsers * k);
    int32_t *lid = reinterpret_cast<int32_t *>(ptr);
    ptr += align16(sizeof(int32_t) * kFrUsers * k);
    uint32_t *pmask = reinterpret_cast<uint32_t *>(ptr);
    ptr += align16(sizeof(uint32_t) * kFrUsers * 2);
    double *unv = reinterpret_cast<double *>(ptr);  // [0,64) norm, [64,128) 1/norm, [128,192) limit
    ptr += align16(sizeof(double) * kFrUsers * 3);
    int64_t *curv = reinterpret_cast<int64_t *>(ptr);  // cursor, end, item at the cursor
    ptr += align16(sizeof(int64_t) * kFrUsers * 3);
    int32_t *nl = reinterpret_cast<int32_t *>(ptr);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tq = lane & 3;
    // CTA = (user block, item range): the catalog is cut into nsplit ranges
    // of whole tiles so that the grid fills the SMs evenly (and small user
    // sets still use every SM); eval_finish_kernel merges the ranges' lists
    const int split = (int)(blockIdx.x % (unsigned)nsplit);
    const int64_t ubase = (int64_t)(blockIdx.x / (unsigned)nsplit) * kFrUsers;
    const int64_t i_begin = (int64_t)split * split_items;
    const int64_t i_end = imin64(t_rows, i_begin + split_items);
    const int nub = (int)imin64(kFrUsers, n_users - ubase);
    for (int i = tid; i < kFrUsers * K; i += 256) {
        const int b = i / K, c = i % K;
        double v = 0.0;
        if (b < nub) {
            const int64_t off = (int64_t)users[ubase + b] * K + c;
            v = s_f64 ? reinterpret_cast<const double *>(S)[off]
                      : (double)reinterpret_cast<const float *>(S)[off];
        }
        uT[c * LDU + b] = v;
    }
    __syncthreads();
    // the limit a score (times the item's reciprocal norm) must reach to be
    // looked at: -inf while the list is short (or the user's norm is zero:
    // every cosine is then 0 and the merge decides), +inf for a padding slot
    auto limit_of = [&](int b, double kth) -> double {
        if (!cosine) return kth - 2e-9;
        const double run = unv[kFrUsers + b];
        return run > 0.0 ? (kth - 2e-9) * unv[b] : -INFINITY;
    };
    if (tid < kFrUsers) {
        const int b = tid;
        double a = 0.0;
        for (int c = 0; c < K; ++c) a = fma(uT[c * LDU + b], uT[c * LDU + b], a);
        const double n = sqrt(a);
        unv[b] = n;
        unv[kFrUsers + b] = n > 0.0 ? 1.0 / n : 0.0;
        unv[2 * kFrUsers + b] = b < nub ? -INFINITY : INFINITY;
        const int64_t u = b < nub ? users[ubase + b] : 0;
        const bool has = b < nub && u < tr_num_users;
        int64_t lo = has ? tr_off[u] : 0;
        const int64_t cend = has ? tr_off[u + 1] : 0;
        for (int64_t hi = cend; lo < hi;) {  // first train positive inside the item range
            const int64_t mid = (lo + hi) >> 1;
            if (tr_items[mid] < i_begin) lo = mid + 1; else hi = mid;
        }
        curv[b] = lo;
        curv[kFrUsers + b] = cend;
        curv[2 * kFrUsers + b] = lo < cend ? (int64_t)tr_items[lo] : INT64_MAX;
        nl[b] = 0;
    }
    constexpr int PER = (kFrItems * KC / 4 + 255) / 256;  // float4 per thread
    float4 pre[PER];
    auto load_tile = [&](int64_t i0) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int f = tid + q * 256;
            const int r = f / (KC / 4), c4 = f % (KC / 4);
            const int64_t row = i0 + r;
            pre[q] = (r < kFrItems && row < t_rows && c4 * 4 < K)
                         ? *reinterpret_cast<const float4 *>(T + row * K + c4 * 4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    auto store_tile = [&]() {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int f = tid + q * 256;
            const int r = f / (KC / 4), c = (f % (KC / 4)) * 4;
            if (r < kFrItems && c < K) {
                double *d = tile + r * LDT + c;  // (LDT even, c % 4 == 0: 16-byte aligned)
                *reinterpret_cast<double2 *>(d) = make_double2(pre[q].x, pre[q].y);
                *reinterpret_cast<double2 *>(d + 2) = make_double2(pre[q].z, pre[q].w);
            }
        }
    };
    load_tile(i_begin);
    for (int64_t i0 = i_begin; i0 < i_end; i0 += kFrItems) {
        __syncthreads();  // previous tile consumed (its products, masks and norms)
        store_tile();
        if (tid < kFrItems) {
            const int64_t item = i0 + tid;
            rin[tid] = item < t_rows ? (cosine ? rinorm_g[item] : 1.0) : 0.0;
        }
        if (lane < 16) pmask[warp * 16 + lane] = 0u;  // the warp's 8 users x 2 words
        __syncthreads();
        if (i0 + kFrItems < i_end) load_tile(i0 + kFrItems);  // overlaps the scoring
        // this tile's train positives of the warp's users -> 64-bit masks
        for (int j = 0; j < 8; ++j) {
            const int b = warp * 8 + j;
            if (curv[2 * kFrUsers + b] >= i0 + kFrItems) continue;  // (warp-uniform)
            int64_t c0 = curv[b];
            const int64_t cend = curv[kFrUsers + b];
            while (c0 < cend) {
                const int64_t idx = c0 + lane;
                const int64_t item = idx < cend ? (int64_t)tr_items[idx] : INT64_MAX;
                const bool in_tile = item < i0 + kFrItems;
                if (in_tile) {
                    const int o = (int)(item - i0);
                    atomicOr(&pmask[b * 2 + (o >> 5)], 1u << (o & 31));
                }
                const unsigned m = __ballot_sync(0xffffffffu, in_tile);
                c0 += __popc(m);
                if (m != 0xffffffffu) break;
            }
            __syncwarp();
            if (lane == 0) {
                curv[b] = c0;
                curv[2 * kFrUsers + b] = c0 < cend ? (int64_t)tr_items[c0] : INT64_MAX;
            }
        }
        __syncwarp();
        // users 8w .. 8w+7 x the tile's 64 items: 8 m8n8k4 tiles per k-step.
        // Thread (g, tq) ends with scores of user 8w + g for items
        // 8 ni + 2 tq and 8 ni + 2 tq + 1.
        double c0[8], c1[8];
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) c0[ni] = c1[ni] = 0.0;
        {
            const double *ucol = uT + 8 * warp + g;
            const double *trow = tile + (size_t)g * LDT + tq;
            for (int k0 = 0; k0 < K; k0 += 4) {
                const double av = ucol[(k0 + tq) * LDU];  // A[user g][k0 + tq]
#pragma unroll
                for (int ni = 0; ni < 8; ++ni) {
                    const double bv = trow[(size_t)8 * ni * LDT + k0];  // B[k0 + tq][item 8 ni + g]
                    asm volatile(
                        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, "
                        "{%0, %1};"
                        : "+d"(c0[ni]), "+d"(c1[ni])
                        : "d"(av), "d"(bv));
                }
            }
        }
        // screen in registers
        const double lim = unv[2 * kFrUsers + warp * 8 + g];
        bool any = false;
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) {
            const double2 r2 = *reinterpret_cast<const double2 *>(rin + 8 * ni + 2 * tq);
            any |= !(c0[ni] * r2.x < lim);
            any |= !(c1[ni] * r2.y < lim);
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        // merge the survivors (any order: the insertion point compares ids).
        // ONE copy of the merge code, looped over the 16 score slots: sixteen
        // unrolled copies thrashed the instruction cache (no_instructions was
        // 18 % of the stall samples).
        unsigned mine = 0;  // bit 2 ni + e: my score in slot (ni, e) passed the screen
#pragma unroll
        for (int ni = 0; ni < 8; ++ni) {
            const double2 r2 = *reinterpret_cast<const double2 *>(rin + 8 * ni + 2 * tq);
            mine |= (!(c0[ni] * r2.x < lim) ? 1u : 0u) << (2 * ni);
            mine |= (!(c1[ni] * r2.y < lim) ? 1u : 0u) << (2 * ni + 1);
        }
        unsigned slots = __reduce_or_sync(0xffffffffu, mine);
#pragma unroll 1
        while (slots) {
            const int slot = __ffs(slots) - 1;
            slots &= slots - 1;
            const int ni = slot >> 1, e = slot & 1;
            double s = 0.0;  // my score of the slot (register select, no local memory)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q == ni) s = e ? c1[q] : c0[q];
            }
            unsigned mk = __ballot_sync(0xffffffffu, (mine >> slot) & 1u);
#pragma unroll 1
            while (mk) {
                const int src = __ffs(mk) - 1;
                mk &= mk - 1;
                const double sr = __shfl_sync(0xffffffffu, s, src);
                const int b = warp * 8 + (src >> 2);
                const int o = 8 * ni + 2 * (src & 3) + e;
                const int64_t item = i0 + o;
                if (b >= nub || item >= t_rows || ((pmask[b * 2 + (o >> 5)] >> (o & 31)) & 1u))
                    continue;
                double cs = sr;
                if (cosine) {
                    const double in = inorm_g[item], un = unv[b];
                    cs = (un == 0.0 || in == 0.0) ? 0.0 : sr / (un * in);
                }
                const int32_t cid = (int32_t)item;
                double *lsb = ls + b * k;
                int32_t *lidb = lid + b * k;
                const int n = nl[b];
                const int newn = n < k ? n + 1 : k;
                if (k <= 32) {
                    // the list across the lanes: lane l holds entry l; the
                    // entries behind the insertion point move up one lane
                    const bool in_list = lane < n;
                    const double own = in_list ? lsb[lane] : 0.0;
                    const int32_t oid = in_list ? lidb[lane] : 0;
                    const bool better = in_list && (own > cs || (own == cs && oid < cid));
                    const int posn = __popc(__ballot_sync(0xffffffffu, better));
                    const double up = __shfl_up_sync(0xffffffffu, own, 1);
                    const int32_t upid = __shfl_up_sync(0xffffffffu, oid, 1);
                    if (posn < k) {  // (a full list whose last entry beats the candidate: no change)
                        if (lane == posn) { lsb[lane] = cs; lidb[lane] = cid; }
                        else if (lane > posn && lane < newn) { lsb[lane] = up; lidb[lane] = upid; }
                        if (lane == 0) nl[b] = newn;
                    }
                    __syncwarp();
                    if (posn < k && newn == k && lane == 0)
                        unv[2 * kFrUsers + b] = limit_of(b, lsb[k - 1]);
                    __syncwarp();
                    continue;
                }
                if (n == k && !(cs > lsb[k - 1] || (cs == lsb[k - 1] && cid < lidb[k - 1])))
                    continue;
                int posn = 0;
                for (int e0 = 0; e0 < n; e0 += 32) {
                    const int q = e0 + lane;
                    const bool better = q < n && (lsb[q] > cs || (lsb[q] == cs && lidb[q] < cid));
                    posn += __popc(__ballot_sync(0xffffffffu, better));
                }
                for (int hi = newn - 1; hi > posn; hi -= 32) {
                    const int dst = hi - lane;
                    const bool mv = dst > posn;
                    double vs = 0.0;
                    int32_t vi = 0;
                    if (mv) { vs = lsb[dst - 1]; vi = lidb[dst - 1]; }
                    __syncwarp();
                    if (mv) { lsb[dst] = vs; lidb[dst] = vi; }
                    __syncwarp();
                }
                if (lane == 0 && posn < k) { lsb[posn] = cs; lidb[posn] = cid; }
                __syncwarp();
                if (lane == 0) {
                    nl[b] = newn;
                    if (newn == k) unv[2 * kFrUsers + b] = limit_of(b, lsb[k - 1]);
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    // this range's lists out (scores, ids, sizes), merged by eval_finish_kernel
    for (int j = 0; j < 8; ++j) {
        const int b = warp * 8 + j;
        if (b >= nub) continue;
        const int64_t slot = (int64_t)split * n_users + ubase + b;
        const int n = nl[b];
        for (int e = lane; e < n; e += 32) {
            part_scores[slot * k + e] = ls[b * k + e];
            part_ids[slot * k + e] = lid[b * k + e];
        }
        if (lane == 0) part_n[slot] = n;
    }
}

// One thread per user: the k best of the item ranges' lists under (score
// desc, id asc) — each list is sorted that way, so a k-step selection over
// the list heads — then hits / recall / NDCG as evaluator.py:164-172.
__global__ void eval_finish_kernel(const double *__restrict__ part_scores,
                                   const int32_t *__restrict__ part_ids,
                                   const int32_t *__restrict__ part_n, int nsplit,
                                   const int32_t *__restrict__ users, int64_t n_users,
                                   const int64_t *__restrict__ te_off,
                                   const int32_t *__restrict__ te_items, int k,
                                   const double *__restrict__ dcg_w,
                                   const double *__restrict__ idcg, int32_t *__restrict__ topk,
                                   double *__restrict__ recall, double *__restrict__ ndcg) {
    const int64_t ug = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ug >= n_users) return;
    constexpr int kMaxSplit = 32;
    int head[kMaxSplit];
    for (int q = 0; q < nsplit; ++q) head[q] = 0;
    const int64_t u = users[ug];
    const int64_t tb = te_off[u], te = te_off[u + 1];
    const int64_t nt = te - tb;
    int hits = 0;
    double dcg = 0.0;
    for (int r = 0; r < k; ++r) {
        int best = -1;
        double bs = 0.0;
        int32_t bi = 0;
        for (int q = 0; q < nsplit; ++q) {
            const int64_t slot = (int64_t)q * n_users + ug;
            if (head[q] >= part_n[slot]) continue;
            const double cs = part_scores[slot * k + head[q]];
            const int32_t ci = part_ids[slot * k + head[q]];
            if (best < 0 || cs > bs || (cs == bs && ci < bi)) { best = q; bs = cs; bi = ci; }
        }
        if (best < 0) {
            if (topk)
                for (int e = r; e < k; ++e) topk[ug * k + e] = -1;
            break;
        }
        ++head[best];
        if (topk) topk[ug * k + r] = bi;
        int64_t lo = tb, hi2 = te;
        while (lo < hi2) {
            const int64_t mid = (lo + hi2) >> 1;
            if (te_items[mid] < bi) lo = mid + 1; else hi2 = mid;
        }
        if (lo < te && te_items[lo] == bi) {
            ++hits;
            dcg += dcg_w[r];
        }
    }
    recall[ug] = (double)hits / (double)nt;
    ndcg[ug] = dcg / idcg[(k < nt ? k : nt) - 1];
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


template <int KC>
static cudaError_t launch_eval_fr(const void *S, int s_f64, const float *T, int64_t t_rows,
                                  int K, const int32_t *users, int64_t n_users,
                                  const int64_t *tr_off, const int32_t *tr_items, int64_t tr_nu,
                                  const int64_t *te_off, const int32_t *te_items, int k,
                                  int cosine, const double *dw, const double *idcg, int32_t *topk,
                                  double *rec, double *nd, cudaStream_t st) {
    const size_t smem = eval_fr_smem_bytes(K, k);
    cudaError_t e = cudaFuncSetAttribute(eval_fr_kernel<KC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // item norms and reciprocals, once per call (evaluator.py:140-141)
    double *norms = static_cast<double *>(stream_scratch(2, (size_t)t_rows * 16, st));
    if (!norms) return cudaErrorMemoryAllocation;
    item_norms_kernel<<<(unsigned)((t_rows + 255) / 256), 256, 0, st>>>(T, t_rows, K, norms,
                                                                        norms + t_rows);
    // Item ranges: one, unless the user blocks alone leave SMs idle (small
    // user sets) — then as many ranges (at most 32, at least 16 tiles each) as
    // fill two CTAs per SM.  Measured on c2 (434 blocks on 296 slots): 10.2 ms
    // unsplit, 10.6 / 12.5 / 13.3 ms at 2 / 3 / 4 ranges — every range builds
    // its own list from scratch (k ln(n / k) insertions each) and a lone CTA
    // on an SM runs faster, so evening out the waves does not pay.
    const int64_t blocks = (n_users + kFrUsers - 1) / kFrUsers;
    const int64_t tiles = (t_rows + kFrItems - 1) / kFrItems;
    const int64_t slots = 2 * (int64_t)sm_count();
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(32, tiles / 16),
                                                             slots / blocks));
    if (const char *f = getenv("HEAT_EVAL_SPLIT")) nsplit = std::min(std::max(atoi(f), 1), 32);
    const int64_t split_items = ((tiles + nsplit - 1) / nsplit) * kFrItems;
    const size_t per = (size_t)nsplit * (size_t)n_users;
    unsigned char *part = static_cast<unsigned char *>(
        stream_scratch(4, per * (size_t)k * 12 + per * 4 + 64, st));
    if (!part) return cudaErrorMemoryAllocation;
    double *part_scores = reinterpret_cast<double *>(part);
    int32_t *part_ids = reinterpret_cast<int32_t *>(part + per * (size_t)k * 8);
    int32_t *part_n = part_ids + per * (size_t)k;
    eval_fr_kernel<KC><<<(unsigned)(blocks * nsplit), 256, smem, st>>>(
        S, s_f64, T, t_rows, K, norms, norms + t_rows, users, n_users, tr_off, tr_items, tr_nu,
        te_off, te_items, k, cosine, nsplit, split_items, part_scores, part_ids, part_n);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    eval_finish_kernel<<<(unsigned)((n_users + 127) / 128), 128, 0, st>>>(
        part_scores, part_ids, part_n, nsplit, users, n_users, te_off, te_items, k, dw, idcg, topk,
        rec, nd);
    return cudaGetLastError();
}

template <int KC, bool MMA>
static cudaError_t launch_eval_rb(const void *S, int s_f64, const float *T, int64_t t_rows,
                                  int K, const int32_t *users, int64_t n_users,
                                  const int64_t *tr_off, const int32_t *tr_items, int64_t tr_nu,
                                  const int64_t *te_off, const int32_t *te_items, int k,
                                  int cosine, const double *dw, const double *idcg, int32_t *topk,
                                  double *rec, double *nd, cudaStream_t st) {
    const size_t smem = eval_rb_smem_bytes<MMA>(K, k);
    cudaError_t e = cudaFuncSetAttribute(eval_rb_kernel<KC, MMA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // item norms and reciprocals, once per call (evaluator.py:140-141)
    double *norms = static_cast<double *>(stream_scratch(2, (size_t)t_rows * 16, st));
    if (!norms) return cudaErrorMemoryAllocation;
    item_norms_kernel<<<(unsigned)((t_rows + 255) / 256), 256, 0, st>>>(T, t_rows, K, norms,
                                                                        norms + t_rows);
    const int64_t blocks = (n_users + kRbUsers - 1) / kRbUsers;
    eval_rb_kernel<KC, MMA><<<(unsigned)blocks, 256, smem, st>>>(
        S, s_f64, T, t_rows, K, norms, norms + t_rows, users, n_users, tr_off, tr_items, tr_nu,
        te_off, te_items, k, cosine, dw, idcg, topk, rec, nd);
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
    const bool mma = !getenv("HEAT_EVAL_FMA") && eval_rb_smem_bytes<true>(K, k) <= cap;
    const bool rb_ok = K % 4 == 0 && eval_rb_smem_bytes<false>(K, k) <= cap &&
                       !getenv("HEAT_EVAL_PLAIN");
#define HEAT_EVAL_RB(KCV)                                                                        \
    return mma ? launch_eval_rb<KCV, true>(S, s_f64, T, t_rows, K, users, n_users, tr_offsets,  \
                                           tr_items, tr_num_users, te_offsets, te_items, k,     \
                                           cosine, dcg_w, idcg, topk, recall, ndcg, stream)     \
               : launch_eval_rb<KCV, false>(S, s_f64, T, t_rows, K, users, n_users, tr_offsets, \
                                            tr_items, tr_num_users, te_offsets, te_items, k,    \
                                            cosine, dcg_w, idcg, topk, recall, ndcg, stream)
    // the fragment-resident kernel (default; HEAT_EVAL_RB=1 selects the register-blocked one)
    const bool fr_ok = mma && rb_ok && K % 4 == 0 && !getenv("HEAT_EVAL_RB") &&
                       eval_fr_smem_bytes(K, k) <= cap;
#define HEAT_EVAL_FR(KCV)                                                                    \
    return launch_eval_fr<KCV>(S, s_f64, T, t_rows, K, users, n_users, tr_offsets, tr_items, \
                               tr_num_users, te_offsets, te_items, k, cosine, dcg_w, idcg,   \
                               topk, recall, ndcg, stream)
    if (fr_ok && K <= 32) HEAT_EVAL_FR(32);
    if (fr_ok && K <= 64) HEAT_EVAL_FR(64);
    if (fr_ok && K <= 128) HEAT_EVAL_FR(128);
#undef HEAT_EVAL_FR
    if (rb_ok && K <= 32) HEAT_EVAL_RB(32);
    if (rb_ok && K <= 64) HEAT_EVAL_RB(64);
    if (rb_ok && K <= 128) HEAT_EVAL_RB(128);
#undef HEAT_EVAL_RB
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
