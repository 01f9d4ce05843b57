// heat_capi.cu — the C ABI declared in include/heat_b200.h.
//
// Host-side validation mirrors the reference's error behaviour: bad shapes
// and options are rejected before any device work (trainer.py:366-382, the
// dataclass checks of trainer.py:55-59,79-87 and kernels.py:50-54), and
// options outside the built path (tiling sampler, aggregator) are rejected by
// the Python layer with ValueError — there is no CPU fallback.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>
#include <string>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

static thread_local std::string g_err;

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

static int cuda_fail(cudaError_t e, const char *what) {
    return fail(HEAT_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 1;
    }
    return cached[dev];
}

// Library-owned scratch when the caller passes none: one buffer per
// (purpose, device, stream), so kernels queued on different streams never
// share it.  Grown on demand; growth waits for the device to go idle.
void *stream_scratch(int purpose, size_t bytes, cudaStream_t stream) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, cudaStream_t>, std::pair<void *, size_t>> bufs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto &b = bufs[std::make_tuple(purpose, dev, stream)];
    if (b.second < bytes) {
        if (b.first) {
            cudaDeviceSynchronize();
            cudaFree(b.first);
        }
        b = {nullptr, 0};
        if (cudaMalloc(&b.first, bytes) != cudaSuccess) {
            cudaGetLastError();
            b.first = nullptr;
            return nullptr;
        }
        b.second = bytes;
    }
    return b.first;
}

// Resident CTAs per SM of `kern` at `threads` and `smem` dynamic bytes, with
// the dynamic shared-memory opt-in applied once: both calls cost microseconds
// of host time, which a short step (the sharded runtime launches one kernel
// per few-microsecond step) cannot afford on every launch.
int kernel_occupancy(const void *kern, int threads, size_t smem, cudaError_t *err) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, size_t>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, kern, threads, smem);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *err = cudaSuccess;
            return it->second;
        }
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    *err = e;
    if (e != cudaSuccess) return 0;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = per_sm;
    return per_sm;
}

static void *get_scratch(size_t bytes, cudaStream_t stream) {
    return stream_scratch(0, bytes, stream);
}

// ---- ordered / atomic item-delta application (multi-GPU exchange) --------
// ordered: ids sorted ascending (stable), each run of equal ids summed in
// index order by one warp and added once -> bit-identical on every replica.
__global__ void apply_deltas_ordered(float *__restrict__ T, int K, const int32_t *__restrict__ ids,
                                     const float *__restrict__ rows, const int64_t *count_p,
                                     int64_t capacity) {
    const int64_t count = imin64(*count_p, capacity);
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (; w < count; w += nw) {
        const int32_t id = ids[w];
        if (w > 0 && ids[w - 1] == id) continue;  // not a run head
        for (int k0 = 0; k0 < K; k0 += 32) {
            int k = k0 + lane;
            if (k >= K) break;
            float acc = 0.f;
            for (int64_t i = w; i < count && ids[i] == id; ++i) acc += rows[i * K + k];
            T[(int64_t)id * K + k] += acc;
        }
    }
}

__global__ void apply_deltas_atomic(float *__restrict__ T, int K, const int32_t *__restrict__ ids,
                                    const float *__restrict__ rows, const int64_t *count_p,
                                    int64_t capacity) {
    const int64_t count = imin64(*count_p, capacity);
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < count * K; i += stride) {
        int64_t r = i / K;
        int k = (int)(i % K);
        atomicAdd(T + (int64_t)ids[r] * K + k, rows[i]);
    }
}

// ---- order-independent (fixed-point) application ---------------------------------
// Entries e < world*stride, valid when e % stride < counts[e / stride].  Pass 1
// adds round(delta * 2^40) into an int64 accumulator per (row, column) —
// integer addition commutes, so the sum is the same whatever order the
// atomics land in — and flags the row; pass 2 converts each flagged row once:
// T += float(acc * 2^-40), acc = 0.  Every replica that applies the same
// gathered logs therefore computes bit-identical rows, with no sort.
constexpr double kFixScale = 1099511627776.0;  // 2^40: resolution 9.1e-13, range +-8.4e6

__global__ void apply_deltas_fixed_acc(int K, const int32_t *__restrict__ ids,
                                       const float *__restrict__ rows,
                                       const int64_t *__restrict__ counts, int world,
                                       int64_t stride, long long *__restrict__ acc,
                                       int32_t *__restrict__ flags) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = (int64_t)world * stride;
    for (; w < total; w += nw) {
        if (w % stride >= counts[w / stride]) continue;
        const int64_t id = ids[w];
        if (lane == 0) flags[id] = 1;
        for (int k = lane; k < K; k += 32) {
            const long long q = __double2ll_rn((double)rows[w * K + k] * kFixScale);
            atomicAdd(reinterpret_cast<unsigned long long *>(acc + id * K + k),
                      (unsigned long long)q);
        }
    }
}

__global__ void apply_deltas_fixed_cvt(float *__restrict__ T, int K,
                                       const int32_t *__restrict__ ids,
                                       const int64_t *__restrict__ counts, int world,
                                       int64_t stride, long long *__restrict__ acc,
                                       int32_t *__restrict__ flags) {
    const int lane = threadIdx.x & 31;
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t total = (int64_t)world * stride;
    for (; w < total; w += nw) {
        if (w % stride >= counts[w / stride]) continue;
        const int64_t id = ids[w];
        int mine = 0;
        if (lane == 0) mine = atomicExch(flags + id, 0);
        mine = __shfl_sync(0xffffffffu, mine, 0);
        if (!mine) continue;  // another warp converts this row
        for (int k = lane; k < K; k += 32) {
            const long long q = acc[id * K + k];
            acc[id * K + k] = 0;
            T[id * K + k] += (float)((double)q * (1.0 / kFixScale));
        }
    }
}

cudaError_t launch_apply_deltas_fixed(float *T, int K, const int32_t *ids, const float *rows,
                                      const int64_t *counts, int world, int64_t stride,
                                      long long *acc, int32_t *flags, cudaStream_t st) {
    const int64_t total = (int64_t)world * stride;
    if (total <= 0) return cudaSuccess;
    const int64_t warps = std::min<int64_t>(total, (int64_t)sm_count() * 64);
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    apply_deltas_fixed_acc<<<blocks, 256, 0, st>>>(K, ids, rows, counts, world, stride, acc,
                                                   flags);
    apply_deltas_fixed_cvt<<<blocks, 256, 0, st>>>(T, K, ids, counts, world, stride, acc, flags);
    return cudaGetLastError();
}

cudaError_t launch_apply_deltas(float *T, int64_t t_rows, int K, const int32_t *ids,
                                const float *rows, const int64_t *count, int64_t capacity,
                                int ordered, cudaStream_t stream) {
    (void)t_rows;
    int blocks = sm_count() * 4;
    if (ordered)
        apply_deltas_ordered<<<blocks, 256, 0, stream>>>(T, K, ids, rows, count, capacity);
    else
        apply_deltas_atomic<<<blocks, 256, 0, stream>>>(T, K, ids, rows, count, capacity);
    return cudaGetLastError();
}

}  // namespace heat

using namespace heat;

__global__ void l2_probe_kernel(const float4 *__restrict__ a, long long n4, int passes,
                                float *sink) {
    float acc = 0.f;
    for (int p = 0; p < passes; ++p)
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
             i += (long long)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + i);
            acc += (v.x + v.y) + (v.z + v.w);
        }
    if (acc == 1234.5f) sink[0] = acc;  // keeps the loads live
}

// Random-row gather probe: the access pattern of the training kernels'
// reads (8 lanes per row, V float4 per lane, two groups of 4 rows in flight
// per warp, rows drawn by a hash), with no arithmetic beyond a sum.  It
// measures what this GPU's L2 delivers to gathers of dim-float rows — the
// ceiling a gather-bound kernel is compared against (scripts/gather_ceiling.cu
// sweeps the configurations; 28 one-warp CTAs per SM is the best of them).
template <int V>
__global__ void __launch_bounds__(32) l2_gather_probe_kernel(const float4 *__restrict__ T,
                                                             unsigned rows, int iters,
                                                             float *sink) {
    const int lane = threadIdx.x, g = lane >> 3, c = lane & 7;
    unsigned h = blockIdx.x * 0x9E3779B9u + 0x7F4A7C15u;
    auto row = [&](int it, int u) {
        unsigned x = h + (unsigned)(it * 2 + u) * 4u + (unsigned)g;
        x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
        return T + (size_t)(x % rows) * (V * 8) + c;
    };
    float acc = 0.f;
    float4 b[2][V];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) b[u][j] = __ldcg(row(0, u) + 8 * j);
    for (int it = 1; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
#pragma unroll
            for (int j = 0; j < V; ++j) acc += (b[u][j].x + b[u][j].y) + (b[u][j].z + b[u][j].w);
#pragma unroll
            for (int j = 0; j < V; ++j) b[u][j] = __ldcg(row(it, u) + 8 * j);
        }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc += b[u][j].x;
    if (acc == 1234.5f) sink[0] = acc;
}

extern "C" {

const char *heat_last_error(void) { return g_err.c_str(); }

/* Random-row gather probe over a rows x dim table (dim 64 or 128): one-warp
 * CTAs, 28 per SM, each `iters` x 8 rows; *rows_read gets the row count. */
int heat_probe_l2_gather(const float *table, int64_t rows, int32_t dim, int32_t iters,
                         float *sink, int64_t *rows_read, void *stream) {
    if (!table || !sink || rows < 1 || rows > 0xFFFFFFFFll || iters < 2 ||
        (dim != 64 && dim != 128))
        return fail(HEAT_ERR_INVALID, "bad gather probe args");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 28;
    const float4 *t4 = reinterpret_cast<const float4 *>(table);
    if (dim == 128)
        l2_gather_probe_kernel<4><<<grid, 32, 0, (cudaStream_t)stream>>>(t4, (unsigned)rows, iters,
                                                                         sink);
    else
        l2_gather_probe_kernel<2><<<grid, 32, 0, (cudaStream_t)stream>>>(t4, (unsigned)rows, iters,
                                                                         sink);
    if (rows_read) *rows_read = (int64_t)grid * iters * 8;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "gather probe launch");
}

int heat_version(void) { return 1; }

// ---- phase profile (trainer.py:120-331 collect_phases, timing.py:20-53)
static std::mutex g_phase_mu;
static unsigned long long *g_phase = nullptr;
static int g_phase_dev = -1;
static bool g_phase_on = false;

}  // extern "C"
namespace heat {
unsigned long long *phase_buffer() {
    std::lock_guard<std::mutex> lk(g_phase_mu);
    if (!g_phase_on || !g_phase) return nullptr;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev != g_phase_dev) return nullptr;
    return g_phase;
}
}  // namespace heat
extern "C" {

int heat_phase_collect(int32_t on) {
    std::lock_guard<std::mutex> lk(g_phase_mu);
    if (!on) {
        g_phase_on = false;
        return HEAT_OK;
    }
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "phase profile: device");
    if (g_phase && g_phase_dev != dev) {
        int cur = dev;
        cudaSetDevice(g_phase_dev);
        cudaFree(g_phase);
        cudaSetDevice(cur);
        g_phase = nullptr;
    }
    if (!g_phase) {
        e = cudaMalloc(&g_phase, heat::kPhaseWords * sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_fail(e, "phase profile: allocation");
        e = cudaMemset(g_phase, 0, heat::kPhaseWords * sizeof(unsigned long long));
        if (e != cudaSuccess) return cuda_fail(e, "phase profile: zero");
        g_phase_dev = dev;
    }
    g_phase_on = true;
    return HEAT_OK;
}

int heat_phase_read(double *seconds, int64_t *workers, int64_t *pairs, int32_t reset) {
    if (!seconds) return fail(HEAT_ERR_INVALID, "phase profile: NULL output");
    std::lock_guard<std::mutex> lk(g_phase_mu);
    for (int i = 0; i < 6; ++i) seconds[i] = 0.0;
    if (workers) *workers = 0;
    if (pairs) *pairs = 0;
    if (!g_phase) return HEAT_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g_phase_dev) cudaSetDevice(g_phase_dev);
    unsigned long long v[heat::kPhaseWords];
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(v, g_phase, sizeof(v), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && reset) e = cudaMemset(g_phase, 0, sizeof(v));
    if (cur != g_phase_dev) cudaSetDevice(cur);
    if (e != cudaSuccess) return cuda_fail(e, "phase profile: read");
    // seconds per phase averaged over the workers, as the reference averages
    // its threads' cycle counts (trainer.py:452-455); clocks -> seconds with
    // the workers' own clock/globaltimer ratio (timing.py:39-53 calibrates
    // rdtsc against perf_counter the same way)
    const double hz = v[7] ? (double)v[6] / ((double)v[7] * 1e-9) : 0.0;
    if (v[8] && hz > 0.0)
        for (int i = 0; i < 6; ++i) seconds[i] = (double)v[i] / (double)v[8] / hz;
    if (workers) *workers = (int64_t)v[8];
    if (pairs) *pairs = (int64_t)v[9];
    return HEAT_OK;
}

/* Diagnostics of the parallel deterministic kernel (not part of the
 * reference interface): clock64 totals [speculate, token wait, commit],
 * [partial recomputes, full recomputes, pairs]; `reset` zeroes them. */
int heat_exact_stats(unsigned long long *out, int reset) {
    exact_spec_stats(out, reset != 0);
    return HEAT_OK;
}

int64_t heat_scratch_bytes(int32_t n_neg, int32_t dim, int64_t s_rows, int64_t t_rows) {
    const int64_t serial = (int64_t)n_neg * (int64_t)dim * (int64_t)sizeof(float) + 256;
    const int64_t spec = (int64_t)exact_spec_scratch_bytes(dim, n_neg, s_rows, t_rows);
    return serial > spec ? serial : spec;
}

int64_t heat_agg_scratch_bytes(int32_t dim, int32_t window) {
    return (int64_t)agg_hogwild_scratch_bytes(dim, window);
}

int heat_sample_negatives(uint64_t stream_base, int64_t first_pair, int64_t npairs,
                          int32_t n_neg, int64_t num_items, int32_t *out, void *stream) {
    if (n_neg < 1) return fail(HEAT_ERR_INVALID, "num_negatives must be >= 1, got %d", n_neg);
    if (num_items < 1 || num_items >= (int64_t)1 << 31)
        return fail(HEAT_ERR_INVALID, "num_items must be in [1, 2^31), got %lld",
                    (long long)num_items);
    if (npairs < 0 || first_pair < 0) return fail(HEAT_ERR_INVALID, "negative pair range");
    if (npairs > 0 && !out) return fail(HEAT_ERR_INVALID, "null output");
    cudaError_t e = launch_sample(stream_base, first_pair, npairs, n_neg, num_items, out,
                                  (cudaStream_t)stream);
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "sample_negatives launch");
}

static int train_range_core(float *S, int64_t s_rows, float *T, int64_t t_rows,
                            const int32_t *ep_users, const int32_t *ep_items, int64_t start,
                            int64_t stop, const heat_sgd_params *p, heat_counters *counters,
                            int32_t *delta_ids, float *delta_rows, int64_t *delta_count,
                            int64_t delta_capacity, const int64_t *pair_index,
                            const heat_agg_params *agg, void *scratch, void *stream,
                            const int64_t *range_dev, const uint64_t *s0_dev) {
    if (!p) return fail(HEAT_ERR_INVALID, "null params");
    if (!S || !T || !counters) return fail(HEAT_ERR_INVALID, "null table or counters pointer");
    if (p->dim < 1) return fail(HEAT_ERR_INVALID, "dim must be >= 1, got %d", p->dim);
    if (p->n_neg < 1)
        return fail(HEAT_ERR_INVALID, "num_negatives must be >= 1, got %d", p->n_neg);
    if (!(p->lr > 0)) return fail(HEAT_ERR_INVALID, "learning_rate must be positive");
    if (p->mu < 0) return fail(HEAT_ERR_INVALID, "mu must be >= 0, got %g", p->mu);
    if (!(p->theta >= -1.0 && p->theta <= 1.0))
        return fail(HEAT_ERR_INVALID, "theta must be in [-1, 1], got %g", p->theta);
    if (s_rows < 1 || t_rows < 1) return fail(HEAT_ERR_INVALID, "empty embedding table");
    if (t_rows >= (int64_t)1 << 31) return fail(HEAT_ERR_INVALID, "item table too large");
    if (start < 0 || stop < start) return fail(HEAT_ERR_INVALID, "bad pair range");
    if (stop > start && (!ep_users || !ep_items)) return fail(HEAT_ERR_INVALID, "null pairs");
    cudaStream_t st = (cudaStream_t)stream;
    if (agg) {
        if (p->mode == HEAT_MODE_DELTA)
            return fail(HEAT_ERR_UNSUPPORTED, "aggregation is not implemented in DELTA mode");
        if (!agg->W || !agg->tr_offsets || !agg->tr_items)
            return fail(HEAT_ERR_INVALID, "aggregation needs W and the train CSR");
        if (p->mode == HEAT_MODE_EXACT && (!agg->accu || !agg->counter))
            return fail(HEAT_ERR_INVALID, "EXACT aggregation needs the accumulator and counter");
        if (p->mode == HEAT_MODE_HOGWILD && p->dim != 16 && p->dim != 32 && p->dim != 64 &&
            p->dim != 128)
            return fail(HEAT_ERR_UNSUPPORTED,
                        "hogwild aggregation supports dim in {16, 32, 64, 128}, got %d", p->dim);
        if (!(agg->gamma >= 0.0 && agg->gamma <= 1.0))
            return fail(HEAT_ERR_INVALID, "gamma must be in [0, 1], got %g", agg->gamma);
        if (agg->mini_batch < 1 || agg->max_history < 0)
            return fail(HEAT_ERR_INVALID, "mini_batch_size >= 1 and max_history >= 0 required");
    }
    if (stop == start) return HEAT_OK;
    cudaError_t e;
    switch (p->mode) {
    case HEAT_MODE_EXACT: {
        // speculative in-order-commit kernel (parallel, bit-identical) unless
        // the shape or the aggregator needs the serial one
        // (a phase profile runs the serial kernel: its phases are the
        // reference's, one pair at a time; results are the same bits)
        unsigned long long *ph = phase_buffer();
        if (!agg && !ph && exact_spec_supported(p->dim, p->n_neg) && !getenv("HEAT_EXACT_SERIAL")) {
            void *sc = scratch ? scratch
                               : get_scratch((size_t)heat_scratch_bytes(p->n_neg, p->dim, s_rows,
                                                                        t_rows), st);
            if (!sc) return fail(HEAT_ERR_CUDA, "exact mode: scratch allocation failed");
            e = launch_exact_spec(S, s_rows, T, t_rows, ep_users, ep_items, start, stop, p->dim,
                                  p->n_neg, p->use_cosine, p->lr, p->l2, p->mu, p->theta,
                                  p->stream_base, counters, sc, pair_index, st);
            break;
        }
        if (exact_smem_bytes(p->dim, p->n_neg) > 220 * 1024)
            return fail(HEAT_ERR_UNSUPPORTED, "exact mode: n_neg=%d dim=%d exceeds shared memory",
                        p->n_neg, p->dim);
        void *snap = scratch ? scratch
                             : get_scratch((size_t)heat_scratch_bytes(p->n_neg, p->dim, s_rows,
                                                                      t_rows), st);
        if (!snap) return fail(HEAT_ERR_CUDA, "exact mode: scratch allocation failed");
        e = launch_exact(S, T, ep_users, ep_items, start, stop, p->dim, p->n_neg, p->use_cosine,
                         p->lr, p->l2, p->mu, p->theta, p->stream_base, t_rows, counters,
                         (float *)snap, pair_index, agg, st, ph);
        break;
    }
    case HEAT_MODE_HOGWILD:
    case HEAT_MODE_DELTA: {
        if (p->dim > 512)
            return fail(HEAT_ERR_UNSUPPORTED, "hogwild mode supports dim <= 512, got %d", p->dim);
        if (p->mode == HEAT_MODE_DELTA && (!delta_ids || !delta_rows || !delta_count))
            return fail(HEAT_ERR_INVALID, "delta mode needs delta buffers");
        HogwildArgs a;
        a.S = S; a.T = T; a.users = ep_users; a.items = ep_items;
        a.start = start; a.stop = stop;
        a.K = p->dim; a.N = p->n_neg; a.cosine = p->use_cosine;
        a.lr = (float)p->lr; a.l2 = (float)p->l2; a.mu = p->mu; a.theta = p->theta;
        a.s0 = p->stream_base; a.num_items = t_rows; a.ctr = counters; a.s_rows = s_rows;
        a.window = p->window; a.fp64 = p->flags & 1;
        a.delta_ids = p->mode == HEAT_MODE_DELTA ? delta_ids : nullptr;
        a.delta_rows = delta_rows; a.delta_count = delta_count;
        a.delta_capacity = delta_capacity;
        a.pair_index = pair_index;
        a.range_dev = range_dev;
        a.s0_dev = s0_dev;
        if (!range_dev && p->mode == HEAT_MODE_HOGWILD) a.phase = phase_buffer();
        if (agg) {
            if (range_dev) return fail(HEAT_ERR_UNSUPPORTED, "aggregation with a device range");
            void *sc = scratch ? scratch
                               : get_scratch(agg_hogwild_scratch_bytes(p->dim, p->window), st);
            if (!sc) return fail(HEAT_ERR_CUDA, "aggregation: scratch allocation failed");
            e = launch_agg_hogwild(a, *agg, sc, st);
            if (e == cudaErrorNotSupported)
                return fail(HEAT_ERR_UNSUPPORTED, "hogwild aggregation: unaligned tables/scratch");
            break;
        }
        e = launch_hogwild(a, st, nullptr);
        if (range_dev && e == cudaErrorNotSupported)
            return fail(HEAT_ERR_UNSUPPORTED, "no kernel family for a device range at dim %d",
                        p->dim);
        break;
    }
    default:
        return fail(HEAT_ERR_INVALID, "unknown mode %d", p->mode);
    }
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "train_range launch");
}

int heat_train_range(float *S, int64_t s_rows, float *T, int64_t t_rows,
                     const int32_t *ep_users, const int32_t *ep_items, int64_t start,
                     int64_t stop, const heat_sgd_params *p, heat_counters *counters,
                     int32_t *delta_ids, float *delta_rows, int64_t *delta_count,
                     int64_t delta_capacity, const int64_t *pair_index,
                     const heat_agg_params *agg, void *scratch, void *stream) {
    return train_range_core(S, s_rows, T, t_rows, ep_users, ep_items, start, stop, p, counters,
                            delta_ids, delta_rows, delta_count, delta_capacity, pair_index, agg,
                            scratch, stream, nullptr, nullptr);
}

int heat_eval_users(const void *S, int32_t s_f64, const float *T, int64_t t_rows, int32_t dim,
                    const int32_t *users, int64_t n_users, const int64_t *tr_offsets,
                    const int32_t *tr_items, int64_t tr_num_users, const int64_t *te_offsets,
                    const int32_t *te_items, int32_t k, int32_t use_cosine,
                    const double *dcg_weights, const double *idcg, int32_t *topk,
                    double *recall, double *ndcg, void *stream) {
    if (k < 1) return fail(HEAT_ERR_INVALID, "k must be >= 1, got %d", k);
    if (dim < 1 || dim > 512) return fail(HEAT_ERR_UNSUPPORTED, "eval supports 1 <= dim <= 512");
    if (t_rows < 1 || t_rows >= (int64_t)1 << 31) return fail(HEAT_ERR_INVALID, "bad t_rows");
    if (n_users < 0) return fail(HEAT_ERR_INVALID, "negative user count");
    if (n_users > 0 && (!S || !T || !users || !te_offsets || !te_items || !dcg_weights || !idcg ||
                        !recall || !ndcg))
        return fail(HEAT_ERR_INVALID, "null pointer argument");
    if (tr_num_users > 0 && (!tr_offsets || !tr_items))
        return fail(HEAT_ERR_INVALID, "null train CSR");
    cudaError_t e = launch_eval(S, s_f64, T, t_rows, dim, users, n_users, tr_offsets, tr_items,
                                tr_num_users, te_offsets, te_items, k, use_cosine, dcg_weights,
                                idcg, topk, recall, ndcg, (cudaStream_t)stream);
    if (e == cudaErrorInvalidValue)
        return fail(HEAT_ERR_UNSUPPORTED, "eval: k=%d with dim=%d exceeds shared memory", k, dim);
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "eval launch");
}

int heat_aggregate_users(const float *S, int64_t s_rows, const float *T, const float *W,
                         int32_t dim, const int64_t *tr_offsets, const int32_t *tr_items,
                         int64_t tr_num_users, double gamma, int64_t max_history, double *out,
                         void *stream) {
    if (dim < 1) return fail(HEAT_ERR_INVALID, "dim must be >= 1");
    if (!(gamma >= 0.0 && gamma <= 1.0)) return fail(HEAT_ERR_INVALID, "gamma must be in [0, 1]");
    if (s_rows > 0 && (!S || !T || !W || !out)) return fail(HEAT_ERR_INVALID, "null pointer");
    if (tr_num_users > 0 && (!tr_offsets || !tr_items)) return fail(HEAT_ERR_INVALID, "null CSR");
    cudaError_t e = launch_aggregate_users(S, T, W, tr_offsets, tr_items, s_rows, tr_num_users,
                                           dim, gamma, max_history, out, (cudaStream_t)stream);
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "aggregate_users launch");
}

int heat_apply_row_deltas(float *T, int64_t t_rows, int32_t dim, const int32_t *ids,
                          const float *rows, const int64_t *count, int64_t capacity,
                          int32_t ordered, void *stream) {
    if (!T || !ids || !rows || !count) return fail(HEAT_ERR_INVALID, "null pointer argument");
    if (dim < 1) return fail(HEAT_ERR_INVALID, "dim must be >= 1");
    cudaError_t e = launch_apply_deltas(T, t_rows, dim, ids, rows, count, capacity, ordered,
                                        (cudaStream_t)stream);
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "apply_row_deltas launch");
}

/* Order-independent replica update for the multi-GPU exchange: the gathered
 * logs of `world` ranks, rank r's entries at [r*stride, r*stride+counts[r]).
 * acc: t_rows*dim int64 and flags: t_rows int32, zero on first use and left
 * zero on return. */
int heat_apply_row_deltas_fixed(float *T, int64_t t_rows, int32_t dim, const int32_t *ids,
                                const float *rows, const int64_t *counts, int32_t world,
                                int64_t stride, int64_t *acc, int32_t *flags, void *stream) {
    if (!T || !counts || !acc || !flags) return fail(HEAT_ERR_INVALID, "null pointer argument");
    if (world < 1 || stride < 0) return fail(HEAT_ERR_INVALID, "bad world / stride");
    if (stride > 0 && (!ids || !rows)) return fail(HEAT_ERR_INVALID, "null log");
    if (dim < 1 || t_rows < 1) return fail(HEAT_ERR_INVALID, "bad table shape");
    cudaError_t e = launch_apply_deltas_fixed(T, dim, ids, rows, counts, world, stride,
                                              reinterpret_cast<long long *>(acc), flags,
                                              (cudaStream_t)stream);
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "apply_row_deltas_fixed launch");
}

/* Diagnostic (not part of the reference interface): streaming read of
 * `n` floats `passes` times, 16-byte vectors at L2 (ld.global.cg), 8 CTAs of
 * 512 threads per SM.  bench.py times it with events to measure the L2
 * ceiling of the L2-resident configurations on the box it runs on. */
int heat_probe_l2_read(const float *buf, int64_t n, int32_t passes, float *sink, void *stream) {
    if (!buf || !sink || n < 4 || passes < 1) return fail(HEAT_ERR_INVALID, "bad probe args");
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    l2_probe_kernel<<<sms * 8, 512, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const float4 *>(buf), n / 4, passes, sink);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HEAT_OK : cuda_fail(e, "l2 probe launch");
}

}  // extern "C"

namespace heat {

int train_range_device_step(float *S, int64_t s_rows, float *T, int64_t t_rows,
                            const int32_t *users, const int32_t *items,
                            const heat_sgd_params *p, heat_counters *counters, int32_t *delta_ids,
                            float *delta_rows, int64_t *delta_count, int64_t delta_capacity,
                            const int64_t *pair_index, const int64_t *range_dev,
                            const uint64_t *s0_dev, void *stream) {
    // grid sized for the window (start/stop only bound it); the kernel reads
    // the step's real range and stream base from range_dev / s0_dev
    return train_range_core(S, s_rows, T, t_rows, users, items, 0, (int64_t)1 << 40, p, counters,
                            delta_ids, delta_rows, delta_count, delta_capacity, pair_index,
                            nullptr, nullptr, stream, range_dev, s0_dev);
}

bool device_step_supported(const heat_sgd_params *p, const float *S, const float *T) {
    if (!p || p->mode != HEAT_MODE_DELTA) return false;
    if (p->dim != 16 && p->dim != 32 && p->dim != 64 && p->dim != 128) return false;
    if (((uintptr_t)S % 16) || ((uintptr_t)T % 16)) return false;
    const char *impl = getenv("HEAT_HOGWILD_IMPL");
    if (getenv("HEAT_FORCE_GENERIC")) return false;
    return !impl || impl[0] == 'r' || impl[0] == 'm' || impl[0] == 's' || impl[0] == 't' ||
           impl[0] == 'w';
}

}  // namespace heat
