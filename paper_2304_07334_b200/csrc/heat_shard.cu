// heat_shard.cu — native runtime of the multi-GPU (user-sharded) epoch.
//
// users sharded u mod G, item table replicated, per-step
// item-delta exchange.  One process per GPU; this file is the per-rank step
// scheduler, in C++.  Per step s (log slot s % (lag + 1), lag = 3 unless
// HEAT_SHARD_LAG says otherwise):
//
//   compute stream s&1: [wait ex_done(s-lag)] DELTA kernel -> log slot
//   comm stream:        [wait log_ready(s)] NCCL all-gather of the 8-byte
//   (top priority)      counts; fused gather+apply: the apply kernels read
//                       every rank's log slot straight from its HBM over
//                       NVLink (CUDA IPC mappings, P2P loads) and add the
//                       entries in 2^-40 fixed point -> T; record ex_done(s)
//
// Nothing waits on the host inside an epoch: the counts stay on the device,
// the apply grid strides over whatever the counts say.  The count all-gather
// doubles as the cross-rank fence: it completes on a rank only once every
// rank's comm stream has reached it, i.e. finished applying step s-1 (so no
// peer still reads an older slot) and seen its own step-s kernel finish (so
// the slot being read is complete).  Kernel(s) waits for ex_done(s-lag):
//   * its slot was last read by the applies of step s-lag-1, which every
//     rank finished before its count all-gather of s-lag could complete;
//   * it sees every applied union up to s-lag (the staleness bound on item
//     rows; Hogwild tolerates it).
// Consecutive kernels alternate between two compute streams, so step s+1's
// workers fill the SMs as step s's tail drains; pairs in flight stay bounded
// by the resident workers.  T changes only through the applies, which every
// rank performs on the same logs with an integer (order-free) sum, so the
// item replicas stay bit-identical.
//
// Fallback exchange (HEAT_SHARD_EXCHANGE=gather, or automatically when some
// rank cannot map a peer's memory; at world 1 it runs with local copies in
// place of the NCCL calls, which is how its scheduling is tested on one GPU): the host reads the counts of step s and NCCL all-gathers the
// logs padded to the largest count, then the same apply runs on the gathered
// copy.  NCCL is resolved at run time from the copy torch already loaded
// (dlopen RTLD_NOLOAD): no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

// log slots (lag + 1 in use; the stream-ordered steps run lag <= 3, the
// persistent epoch lag <= 7)
constexpr int kSlots = kPersistSlots;
constexpr int kStreamMaxLag = 3;
constexpr int kMaxWorld = 64;

struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};

static const NcclApi &nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) return a;
        a.get_unique_id = (decltype(a.get_unique_id))dlsym(h, "ncclGetUniqueId");
        a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(h, "ncclCommInitRank");
        a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
        a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
        a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
        a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
        a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather &&
               a.group_start && a.group_end;
        return a;
    }();
    return api;
}

struct Slot {
    int32_t *ids = nullptr;  // this rank's log (capacity entries)
    float *rows = nullptr;
    int64_t *cnt = nullptr;
    const int32_t **pids = nullptr;  // device [world]: every rank's ids of this slot
    const float **prows = nullptr;   // device [world]
    int32_t *g_ids = nullptr;        // gather fallback: world * capacity entries
    float *g_rows = nullptr;
    cudaEvent_t log_ready = nullptr, cnt_ready = nullptr, ex_done = nullptr;
};

// Where the apply reads step s's entries: per-rank pointers (own log plus
// peers' logs mapped over NVLink), or one gathered buffer of `stride` entries
// per rank.
struct LogView {
    const int32_t *const *pids;
    const float *const *prows;
    const int32_t *ids;
    const float *rows;
    int64_t stride;
};

}  // namespace heat

struct heat_shard {
    int world = 1, rank = 0, device = 0;
    bool p2p = true;
    // kernel(s) waits for the apply of step s - lag: HEAT_SHARD_LAG, else 3 for
    // both runtimes, one staleness bound (measured: the persistent c4 epoch at
    // lag 2 loses 18 % of its warp time to gates, at lag 3 none; the
    // stream-ordered c3 steps run 37.6 M samples/s at lag 2, 41.6 M at lag 3)
    int lag = 3, lag_persist = 3;
    int nalloc = 0;  // log slots allocated (max(lag, lag_persist, 2) + 1)
    ncclComm_t comm = nullptr;
    // host transport (heat_shard_create_host): the collectives of the
    // per-process runtime as calls of a caller-supplied host all-gather
    // (e.g. torch.distributed over gloo) around stream synchronisations,
    // for ranks that share one GPU (NCCL refuses two ranks on a device).
    // Same-device CUDA IPC carries the logs exactly as NVLink would.
    heat_host_allgather_fn hostx = nullptr;
    void *hostx_user = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaStream_t cstream[2] = {nullptr, nullptr};
    cudaEvent_t ev_start = nullptr, ev_cdone[2] = {nullptr, nullptr}, ev_comm = nullptr;
    heat::Slot slot[heat::kSlots];
    std::vector<void *> opened;  // peer mappings to close
    int64_t cap = 0, dim = 0, acc_elems = 0, t_rows = 0;
    long long *acc = nullptr;
    int32_t *flags = nullptr;
    int64_t *step_counts = nullptr;   // device [nsteps * world]
    int64_t *hstep_counts = nullptr;  // pinned copy
    int64_t step_counts_n = 0;
    int64_t *scratch = nullptr;  // device: small collective staging (handles, agreement)
    // loopback group (heat_shard_create_loopback): `world` ranks of one
    // process on one device; the NCCL calls become stream-ordered copies and
    // event waits, peers' logs are read through plain device pointers
    bool loopback = false;
    int64_t *shared_counts = nullptr;  // group-owned [nsteps * world] (rank 0 allocates)
    cudaEvent_t arrive[heat::kSlots] = {};
    // captured step graphs: the epoch's inputs live in runtime-owned buffers
    // (stable addresses), the per-step pair ranges and the stream base in
    // device memory, so one instantiated graph replays every epoch of a shape
    bool graphs = true;
    int32_t *d_users = nullptr, *d_items = nullptr;
    int64_t *d_pidx = nullptr, pairs_cap = 0;
    int64_t *d_bounds = nullptr, *h_bounds = nullptr, bounds_cap = 0;
    uint64_t *d_s0 = nullptr, *h_s0 = nullptr;
    cudaGraphExec_t gexec = nullptr;
    std::vector<int64_t> gkey;
    // persistent epoch (one launch per epoch, steps gated on the device):
    // mailbox [2][mbox_steps][world] and released words [world] are written
    // by every rank (IPC-mapped between processes); the step state and
    // counts are local
    bool persist = true, persist_force = false;
    unsigned long long *mbox = nullptr, *rel = nullptr;
    unsigned long long **mbox_tab = nullptr, **rel_tab = nullptr;  // device [world]
    std::vector<void *> opened_mbox;
    int64_t mbox_steps = 0;
    unsigned long long gstep = 0;  // global steps run since the mailbox was (re)allocated
    unsigned tag = 1;              // epoch tag of the mailbox words
    unsigned long long *pstate = nullptr, *pcnt = nullptr, *pclaim = nullptr;
    int64_t pstate_steps = 0;
    heat::PersistRank *pctx = nullptr;  // device contexts (a loopback group's live in rank 0's)
    // every rank's T replica (the owners' converts store into all of them):
    // device table, and per peer the IPC mapping in use (handle, offset, base)
    float **t_tab = nullptr;
    struct TMap {
        cudaIpcMemHandle_t handle;
        int64_t offset = -1;
        void *base = nullptr;
    };
    std::vector<TMap> tmaps;
    int pctx_n = 0;
    // accumulation buffers of the persistent epoch (one per step in flight)
    long long *pacc[heat::kSlots] = {};
    int32_t *pflags[heat::kSlots] = {}, *ptouched[heat::kSlots] = {};
    unsigned long long *ptcount = nullptr;
    int64_t pbuf_rows = 0, pbuf_dim = 0;
    int pbufs = 0;
    std::string err;
};

namespace heat {

// ---- fused gather + apply ---------------------------------------------------
// Entry (q, i), i < min(counts[q], cap), of rank q's log; warp per entry,
// flattened over ranks with a prefix of the counts in shared memory.  Pass 1
// adds round(delta * 2^40) into an int64 accumulator per (row, column) —
// integer addition commutes — and flags the row; pass 2 converts each flagged
// row once, T += float(acc * 2^-40).  The same fixed point as
// heat_apply_row_deltas_fixed.
constexpr double kShardFixScale = 1099511627776.0;  // 2^40

__device__ __forceinline__ int64_t view_prefix(const int64_t *counts, int world, int64_t cap,
                                               int64_t *pre) {
    if (threadIdx.x == 0) {
        int64_t s = 0;
        pre[0] = 0;
        for (int q = 0; q < world; ++q) {
            s += min(max(counts[q], (int64_t)0), cap);
            pre[q + 1] = s;
        }
    }
    __syncthreads();
    return pre[world];
}

__device__ __forceinline__ void view_entry(const LogView &v, const int64_t *pre, int world,
                                           int64_t w, const int32_t **id_p, const float **row_p,
                                           int K) {
    int q = 0;
    while (q + 1 < world && w >= pre[q + 1]) ++q;
    const int64_t i = w - pre[q];
    if (v.pids) {
        *id_p = v.pids[q] + i;
        *row_p = v.prows[q] + i * K;
    } else {
        *id_p = v.ids + q * v.stride + i;
        *row_p = v.rows + (q * v.stride + i) * K;
    }
}

// counts: the step's per-rank counts; at world 1 the log's own counter,
// which block 0 also records into step_counts (the gathered array otherwise)
__global__ void shard_apply_acc(int K, LogView v, const int64_t *__restrict__ counts, int world,
                                int64_t cap, long long *__restrict__ acc,
                                int32_t *__restrict__ flags, int64_t *__restrict__ step_counts) {
    __shared__ int64_t pre[kMaxWorld + 1];
    const int64_t total = view_prefix(counts, world, cap, pre);
    if (step_counts != counts && blockIdx.x == 0 && threadIdx.x == 0) step_counts[0] = counts[0];
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += nw) {
        const int32_t *idp;
        const float *rp;
        view_entry(v, pre, world, w, &idp, &rp, K);
        const int64_t id = __ldcg(idp);  // peers' logs: read at L2 (theirs), never L1
        if (lane == 0) flags[id] = 1;
        long long *a = acc + id * K;
        if ((K & 3) == 0) {
            for (int k = lane * 4; k < K; k += 128) {
                const float4 d = __ldcg(reinterpret_cast<const float4 *>(rp + k));
                atomicAdd((unsigned long long *)(a + k),
                          (unsigned long long)__double2ll_rn((double)d.x * kShardFixScale));
                atomicAdd((unsigned long long *)(a + k + 1),
                          (unsigned long long)__double2ll_rn((double)d.y * kShardFixScale));
                atomicAdd((unsigned long long *)(a + k + 2),
                          (unsigned long long)__double2ll_rn((double)d.z * kShardFixScale));
                atomicAdd((unsigned long long *)(a + k + 3),
                          (unsigned long long)__double2ll_rn((double)d.w * kShardFixScale));
            }
        } else {
            for (int k = lane; k < K; k += 32)
                atomicAdd((unsigned long long *)(a + k),
                          (unsigned long long)__double2ll_rn((double)__ldcg(rp + k) * kShardFixScale));
        }
    }
}

// counts: the step's recorded counts; block 0 re-arms this rank's log
// counter for the slot's next step (own_cnt; its readers are all done)
__global__ void shard_apply_cvt(float *__restrict__ T, int K, LogView v,
                                const int64_t *__restrict__ counts, int world, int64_t cap,
                                long long *__restrict__ acc, int32_t *__restrict__ flags,
                                int64_t *__restrict__ own_cnt) {
    __shared__ int64_t pre[kMaxWorld + 1];
    const int64_t total = view_prefix(counts, world, cap, pre);
    if (blockIdx.x == 0 && threadIdx.x == 0) *own_cnt = 0;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < total; w += nw) {
        const int32_t *idp;
        const float *rp;
        view_entry(v, pre, world, w, &idp, &rp, K);
        const int64_t id = __ldcg(idp);
        int mine = 0;
        if (lane == 0) mine = atomicExch(flags + id, 0);
        mine = __shfl_sync(0xffffffffu, mine, 0);
        if (!mine) continue;  // another warp converts this row
        long long *a = acc + id * K;
        float *t = T + id * K;
        if ((K & 3) == 0) {  // 4 columns per lane: 2 x 16 B of accumulator, 16 B of T
            for (int k = lane * 4; k < K; k += 128) {
                const longlong2 q01 = *reinterpret_cast<const longlong2 *>(a + k);
                const longlong2 q23 = *reinterpret_cast<const longlong2 *>(a + k + 2);
                *reinterpret_cast<longlong2 *>(a + k) = make_longlong2(0, 0);
                *reinterpret_cast<longlong2 *>(a + k + 2) = make_longlong2(0, 0);
                float4 tv = *reinterpret_cast<const float4 *>(t + k);
                tv.x += (float)((double)q01.x * (1.0 / kShardFixScale));
                tv.y += (float)((double)q01.y * (1.0 / kShardFixScale));
                tv.z += (float)((double)q23.x * (1.0 / kShardFixScale));
                tv.w += (float)((double)q23.y * (1.0 / kShardFixScale));
                *reinterpret_cast<float4 *>(t + k) = tv;
            }
        } else {
            for (int k = lane; k < K; k += 32) {
                const long long q = a[k];
                a[k] = 0;
                t[k] += (float)((double)q * (1.0 / kShardFixScale));
            }
        }
    }
}

static cudaError_t launch_shard_apply(float *T, int K, const LogView &v, const int64_t *counts,
                                      int64_t *step_counts, int64_t *own_cnt, int world,
                                      int64_t cap, long long *acc, int32_t *flags,
                                      cudaStream_t st) {
    // grid sized without the counts (they live on the device): enough warps to
    // cover a typical step, striding over the rest
    const int64_t warps = std::min<int64_t>(std::max<int64_t>(world * cap, 1),
                                            (int64_t)sm_count() * 16);
    const unsigned blocks = (unsigned)((warps * 32 + 255) / 256);
    shard_apply_acc<<<blocks, 256, 0, st>>>(K, v, counts, world, cap, acc, flags, step_counts);
    shard_apply_cvt<<<blocks, 256, 0, st>>>(T, K, v, step_counts, world, cap, acc, flags,
                                            own_cnt);
    return cudaGetLastError();
}

static void close_peers(heat_shard *h) {
    for (void *p : h->opened) cudaIpcCloseMemHandle(p);
    h->opened.clear();
}

// frees the log buffers of every slot (the events stay)
static void free_slots(heat_shard *h) {
    close_peers(h);
    for (Slot &s : h->slot) {
        cudaFree(s.ids); cudaFree(s.rows); cudaFree(s.cnt);
        cudaFree((void *)s.pids); cudaFree((void *)s.prows);
        cudaFree(s.g_ids); cudaFree(s.g_rows);
        s.ids = nullptr; s.rows = nullptr; s.cnt = nullptr; s.pids = nullptr;
        s.prows = nullptr; s.g_ids = nullptr; s.g_rows = nullptr;
    }
    h->cap = 0;
}

struct ShardErr {
    heat_shard *h;
    int rc = HEAT_OK;
    bool cuda(cudaError_t e, const char *what) {
        if (e != cudaSuccess && rc == HEAT_OK) {
            h->err = std::string(what) + ": " + cudaGetErrorString(e);
            rc = HEAT_ERR_CUDA;
        }
        return e == cudaSuccess;
    }
    bool nccl(ncclResult_t r, const char *what) {
        if (r != ncclSuccess && rc == HEAT_OK) {
            const NcclApi &n = heat::nccl();
            h->err = std::string(what) + ": " + (n.error_string ? n.error_string(r) : "nccl error");
            rc = HEAT_ERR_CUDA;
        }
        return r == ncclSuccess;
    }
    bool invalid(const std::string &msg) {
        if (rc == HEAT_OK) {
            h->err = msg;
            rc = HEAT_ERR_INVALID;
        }
        return false;
    }
};

// world > 1: host values all-gathered through NCCL (a collective: every rank
// calls it in the same order); out has world * n entries
static bool host_all_gather(heat_shard *h, ShardErr &er, const int64_t *in, int64_t n,
                            int64_t *out) {
    const int64_t bytes = n * (int64_t)sizeof(int64_t);
    if (h->hostx) {
        if (h->hostx(h->hostx_user, in, bytes, out) != 0) return er.invalid("host all-gather failed");
        return true;
    }
    int64_t *d = h->scratch;  // 1 + world entries of 64 B handles fit (see create)
    if (!er.cuda(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, h->comm_stream), "stage"))
        return false;
    if (!er.nccl(nccl().all_gather(d, d + n, (size_t)bytes, ncclUint8, h->comm, h->comm_stream),
                 "all_gather (host values)"))
        return false;
    if (!er.cuda(cudaMemcpyAsync(out, d + n, bytes * h->world, cudaMemcpyDeviceToHost,
                                 h->comm_stream), "unstage"))
        return false;
    return er.cuda(cudaStreamSynchronize(h->comm_stream), "agree");
}

// (Re)allocates the slots for `cap` entries of `dim` floats and, for the P2P
// exchange at world > 1, maps every peer's slots (IPC handles all-gathered).
// Every rank calls it with the same agreed cap/dim.
static bool ensure_slots(heat_shard *h, ShardErr &er, int64_t cap, int64_t dim) {
    if (cap <= h->cap && dim == h->dim) return true;
    cudaDeviceSynchronize();  // buffers of a previous epoch may still be in use
    free_slots(h);
    const int W = h->world;
    h->nalloc = std::max(std::max(h->lag, h->lag_persist), 2) + 1;
    for (int k = 0; k < h->nalloc; ++k) {
        Slot &s = h->slot[k];
        if (!er.cuda(cudaMalloc(&s.ids, cap * sizeof(int32_t)), "log ids")) return false;
        if (!er.cuda(cudaMalloc(&s.rows, cap * dim * sizeof(float)), "log rows")) return false;
        if (!er.cuda(cudaMalloc(&s.cnt, sizeof(int64_t)), "log count")) return false;
        if (!er.cuda(cudaMalloc((void **)&s.pids, W * sizeof(void *)), "peer ids")) return false;
        if (!er.cuda(cudaMalloc((void **)&s.prows, W * sizeof(void *)), "peer rows")) return false;
        if (W > 1 && !h->p2p) {
            if (!er.cuda(cudaMalloc(&s.g_ids, W * cap * sizeof(int32_t)), "gather ids")) return false;
            if (!er.cuda(cudaMalloc(&s.g_rows, W * cap * dim * sizeof(float)), "gather rows"))
                return false;
        }
    }
    std::vector<const void *> pid(W * kSlots), prow(W * kSlots);
    for (int k = 0; k < h->nalloc; ++k) {
        pid[h->rank * kSlots + k] = h->slot[k].ids;
        prow[h->rank * kSlots + k] = h->slot[k].rows;
    }
    if (W > 1 && h->p2p && !h->loopback) {
        // 2 * kSlots IPC handles per rank, exchanged as int64 words
        static_assert(sizeof(cudaIpcMemHandle_t) % sizeof(int64_t) == 0, "handle size");
        constexpr int64_t hw = sizeof(cudaIpcMemHandle_t) / sizeof(int64_t);
        std::vector<int64_t> mine(2 * kSlots * hw), all(W * 2 * kSlots * hw);
        for (int k = 0; k < h->nalloc; ++k) {
            cudaIpcMemHandle_t a, b;
            if (!er.cuda(cudaIpcGetMemHandle(&a, h->slot[k].ids), "ipc handle")) return false;
            if (!er.cuda(cudaIpcGetMemHandle(&b, h->slot[k].rows), "ipc handle")) return false;
            memcpy(&mine[(2 * k) * hw], &a, sizeof(a));
            memcpy(&mine[(2 * k + 1) * hw], &b, sizeof(b));
        }
        if (!host_all_gather(h, er, mine.data(), (int64_t)mine.size(), all.data())) return false;
        int64_t mapped = 1;
        for (int q = 0; q < W && mapped; ++q) {
            if (q == h->rank) continue;
            for (int k = 0; k < h->nalloc && mapped; ++k) {
                cudaIpcMemHandle_t a, b;
                memcpy(&a, &all[((int64_t)q * 2 * kSlots + 2 * k) * hw], sizeof(a));
                memcpy(&b, &all[((int64_t)q * 2 * kSlots + 2 * k + 1) * hw], sizeof(b));
                void *pa = nullptr, *pb = nullptr;
                if (cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
                    (h->opened.push_back(pa),
                     cudaIpcOpenMemHandle(&pb, b, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)) {
                    cudaGetLastError();  // no peer mapping: every rank falls back below
                    mapped = 0;
                    break;
                }
                h->opened.push_back(pb);
                pid[q * kSlots + k] = pa;
                prow[q * kSlots + k] = pb;
            }
        }
        // the exchange mode is collective: P2P only if every rank mapped every peer
        std::vector<int64_t> all_mapped(W);
        if (!host_all_gather(h, er, &mapped, 1, all_mapped.data())) return false;
        if (*std::min_element(all_mapped.begin(), all_mapped.end()) == 0) {
            close_peers(h);
            h->p2p = false;
            for (int k = 0; k < h->nalloc; ++k) {
                Slot &s = h->slot[k];
                if (!er.cuda(cudaMalloc(&s.g_ids, W * cap * sizeof(int32_t)), "gather ids"))
                    return false;
                if (!er.cuda(cudaMalloc(&s.g_rows, W * cap * dim * sizeof(float)), "gather rows"))
                    return false;
            }
            for (int q = 0; q < W; ++q)
                for (int k = 0; k < kSlots; ++k)
                    if (q != h->rank) pid[q * kSlots + k] = prow[q * kSlots + k] = nullptr;
        }
    }
    for (int k = 0; k < h->nalloc; ++k) {
        std::vector<const void *> a(W), b(W);
        for (int q = 0; q < W; ++q) {
            a[q] = pid[q * kSlots + k];
            b[q] = prow[q * kSlots + k];
        }
        if (!er.cuda(cudaMemcpy((void *)h->slot[k].pids, a.data(), W * sizeof(void *),
                                cudaMemcpyHostToDevice), "peer table"))
            return false;
        if (!er.cuda(cudaMemcpy((void *)h->slot[k].prows, b.data(), W * sizeof(void *),
                                cudaMemcpyHostToDevice), "peer table"))
            return false;
    }
    h->cap = cap;
    h->dim = dim;
    return true;
}

static bool ensure_epoch_buffers(heat_shard *h, ShardErr &er, int64_t t_rows, int64_t dim,
                                 int64_t nsteps) {
    if (t_rows * dim > h->acc_elems || t_rows > h->t_rows) {
        cudaDeviceSynchronize();
        cudaFree(h->acc);
        cudaFree(h->flags);
        h->acc = nullptr;
        h->flags = nullptr;
        h->acc_elems = 0;
        h->t_rows = 0;
        if (!er.cuda(cudaMalloc(&h->acc, t_rows * dim * sizeof(long long)), "accumulator"))
            return false;
        if (!er.cuda(cudaMalloc(&h->flags, t_rows * sizeof(int32_t)), "row flags")) return false;
        if (!er.cuda(cudaMemset(h->acc, 0, t_rows * dim * sizeof(long long)), "zero acc"))
            return false;
        if (!er.cuda(cudaMemset(h->flags, 0, t_rows * sizeof(int32_t)), "zero flags"))
            return false;
        h->acc_elems = t_rows * dim;
        h->t_rows = t_rows;
    }
    const int64_t n = std::max<int64_t>(nsteps, 1) * h->world;
    if (n > h->step_counts_n) {
        cudaDeviceSynchronize();
        cudaFree(h->step_counts);
        cudaFreeHost(h->hstep_counts);
        h->step_counts = nullptr;
        h->hstep_counts = nullptr;
        h->step_counts_n = 0;
        if (!er.cuda(cudaMalloc(&h->step_counts, n * sizeof(int64_t)), "step counts")) return false;
        if (!er.cuda(cudaMallocHost(&h->hstep_counts, n * sizeof(int64_t)), "step counts (host)"))
            return false;
        h->step_counts_n = n;
    }
    return true;
}

// The persistent epoch's cross-rank words: (re)allocated zeroed when an epoch
// has more steps than the mailbox holds, which every rank decides alike (the
// step count is agreed); between processes the buffers are IPC-mapped into
// every peer.  A reallocation restarts the global step count: no kernel runs
// anywhere at that point (every rank finished its previous epoch before the
// agreement collective), so no released word or log slot is still in use.
static bool ensure_mailbox(heat_shard *h, ShardErr &er, int64_t nsteps) {
    const int W = h->world;
    if (nsteps <= h->mbox_steps && h->mbox) return true;
    const int64_t steps = std::max<int64_t>(nsteps, 16);
    cudaDeviceSynchronize();
    for (void *q : h->opened_mbox) cudaIpcCloseMemHandle(q);
    h->opened_mbox.clear();
    cudaFree(h->mbox); cudaFree(h->rel);
    h->mbox = h->rel = nullptr;
    h->mbox_steps = 0;
    const size_t mb = (size_t)2 * steps * W * sizeof(unsigned long long);
    if (!er.cuda(cudaMalloc(&h->mbox, mb), "mailbox") ||
        !er.cuda(cudaMalloc(&h->rel, (W + 1) * sizeof(unsigned long long)), "released words") ||
        !er.cuda(cudaMemset(h->mbox, 0, mb), "zero mailbox") ||
        !er.cuda(cudaMemset(h->rel, 0, (W + 1) * sizeof(unsigned long long)), "zero released"))
        return false;
    if (!h->mbox_tab &&
        (!er.cuda(cudaMalloc((void **)&h->mbox_tab, kMaxWorld * sizeof(void *)), "mailbox table") ||
         !er.cuda(cudaMalloc((void **)&h->rel_tab, kMaxWorld * sizeof(void *)), "released table")))
        return false;
    h->mbox_steps = steps;
    h->gstep = 0;
    h->tag = 1;
    std::vector<void *> mt(W, nullptr), rt(W, nullptr);
    mt[h->rank] = h->mbox;
    rt[h->rank] = h->rel;
    if (W > 1 && !h->loopback) {
        constexpr int64_t hw = sizeof(cudaIpcMemHandle_t) / sizeof(int64_t);
        std::vector<int64_t> mine(2 * hw), all(W * 2 * hw);
        cudaIpcMemHandle_t a, b;
        if (!er.cuda(cudaIpcGetMemHandle(&a, h->mbox), "ipc handle") ||
            !er.cuda(cudaIpcGetMemHandle(&b, h->rel), "ipc handle"))
            return false;
        memcpy(&mine[0], &a, sizeof(a));
        memcpy(&mine[hw], &b, sizeof(b));
        if (!host_all_gather(h, er, mine.data(), 2 * hw, all.data())) return false;
        int64_t mapped = 1;
        for (int q = 0; q < W && mapped; ++q) {
            if (q == h->rank) continue;
            memcpy(&a, &all[(int64_t)q * 2 * hw], sizeof(a));
            memcpy(&b, &all[(int64_t)q * 2 * hw + hw], sizeof(b));
            if (cudaIpcOpenMemHandle(&mt[q], a, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                mapped = 0;
                break;
            }
            h->opened_mbox.push_back(mt[q]);
            if (cudaIpcOpenMemHandle(&rt[q], b, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                mapped = 0;
                break;
            }
            h->opened_mbox.push_back(rt[q]);
        }
        cudaGetLastError();
        // collective: the persistent epoch only if every rank mapped every peer
        std::vector<int64_t> all_mapped(W);
        if (!host_all_gather(h, er, &mapped, 1, all_mapped.data())) return false;
        if (*std::min_element(all_mapped.begin(), all_mapped.end()) == 0) {
            h->persist = false;  // every rank: stream-ordered steps from now on
            return true;
        }
    }
    // (a loopback group fills its tables with every rank's buffers itself)
    return er.cuda(cudaMemcpy(h->mbox_tab, mt.data(), W * sizeof(void *), cudaMemcpyHostToDevice),
                   "mailbox table") &&
           er.cuda(cudaMemcpy(h->rel_tab, rt.data(), W * sizeof(void *), cudaMemcpyHostToDevice),
                   "released table");
}

// base of the device allocation holding p (driver API, resolved from the
// libcuda torch loaded: an IPC handle names a whole cudaMalloc block)
static bool alloc_base(const void *p, void **base) {
    using Fn = int (*)(unsigned long long *, size_t *, unsigned long long);
    static Fn fn = [] {
        void *lib = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
        if (!lib) lib = dlopen("libcuda.so.1", RTLD_NOW);
        return lib ? (Fn)dlsym(lib, "cuMemGetAddressRange_v2") : (Fn) nullptr;
    }();
    unsigned long long b = 0;
    size_t sz = 0;
    if (!fn || fn(&b, &sz, (unsigned long long)(uintptr_t)p) != 0) return false;
    *base = (void *)(uintptr_t)b;
    return true;
}

// every rank's T replica into h->t_tab: plain pointers in a loopback group
// (filled by the caller), CUDA IPC mappings between processes, reopened only
// when a peer's allocation changes (collective at world > 1)
static bool map_replicas(heat_shard *h, ShardErr &er, float *T) {
    const int W = h->world;
    if (!h->t_tab && !er.cuda(cudaMalloc((void **)&h->t_tab, kMaxWorld * sizeof(float *)), "replica table"))
        return false;
    std::vector<float *> tt(W, nullptr);
    tt[h->rank] = T;
    if (W > 1 && !h->loopback) {
        // (handle, offset, ok) per rank; every rank takes part in both
        // collectives whatever happens locally, and all fall back together
        constexpr int64_t hw = sizeof(cudaIpcMemHandle_t) / sizeof(int64_t);
        std::vector<int64_t> mine(hw + 2, 0), all(W * (hw + 2));
        void *base = nullptr;
        cudaIpcMemHandle_t hd;
        if (alloc_base(T, &base) && cudaIpcGetMemHandle(&hd, base) == cudaSuccess) {
            memcpy(mine.data(), &hd, sizeof(hd));
            mine[hw] = (int64_t)((const char *)T - (const char *)base);
            mine[hw + 1] = 1;
        }
        cudaGetLastError();
        if (!host_all_gather(h, er, mine.data(), hw + 2, all.data())) return false;
        int64_t mapped = 1;
        for (int q = 0; q < W; ++q)
            if (all[(int64_t)q * (hw + 2) + hw + 1] == 0) mapped = 0;
        h->tmaps.resize(W);
        for (int q = 0; q < W && mapped; ++q) {
            if (q == h->rank) continue;
            auto &m = h->tmaps[q];
            const int64_t *w = &all[(int64_t)q * (hw + 2)];
            cudaIpcMemHandle_t qh;
            memcpy(&qh, w, sizeof(qh));
            if (!m.base || m.offset != w[hw] || memcmp(&m.handle, &qh, sizeof(qh)) != 0) {
                if (m.base) cudaIpcCloseMemHandle(m.base);
                m.base = nullptr;
                if (cudaIpcOpenMemHandle(&m.base, qh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    m.base = nullptr;
                    mapped = 0;
                    break;
                }
                m.handle = qh;
                m.offset = w[hw];
            }
            tt[q] = reinterpret_cast<float *>((char *)m.base + m.offset);
        }
        cudaGetLastError();
        std::vector<int64_t> all_mapped(W);
        if (!host_all_gather(h, er, &mapped, 1, all_mapped.data())) return false;
        if (*std::min_element(all_mapped.begin(), all_mapped.end()) == 0) {
            h->persist = false;  // every rank: stream-ordered steps from now on
            return true;
        }
    }
    return er.cuda(cudaMemcpy(h->t_tab, tt.data(), W * sizeof(float *), cudaMemcpyHostToDevice),
                   "replica table");
}

// local per-epoch state of the persistent epoch, `nctx` device contexts
static bool ensure_persist_state(heat_shard *h, ShardErr &er, int64_t nsteps, int nctx,
                                 int64_t t_rows, int64_t dim, int nb) {
    if (nsteps > h->pstate_steps) {
        cudaDeviceSynchronize();
        cudaFree(h->pstate); cudaFree(h->pcnt);
        h->pstate = h->pcnt = nullptr;
        h->pstate_steps = 0;
        const int64_t n = std::max<int64_t>(nsteps, 16);
        if (!er.cuda(cudaMalloc(&h->pstate, kStepWords * n * sizeof(unsigned long long)), "step state") ||
            !er.cuda(cudaMalloc(&h->pcnt, n * sizeof(unsigned long long)), "step counts"))
            return false;
        h->pstate_steps = n;
    }
    if (!h->pclaim && !er.cuda(cudaMalloc(&h->pclaim, 4 * sizeof(unsigned long long)), "claim"))
        return false;
    // accumulation buffers: zeroed once; every convert leaves them zero again
    if (nb > h->pbufs || t_rows > h->pbuf_rows || dim != h->pbuf_dim) {
        cudaDeviceSynchronize();
        for (int k = 0; k < kSlots; ++k) {
            cudaFree(h->pacc[k]); cudaFree(h->pflags[k]); cudaFree(h->ptouched[k]);
            h->pacc[k] = nullptr; h->pflags[k] = h->ptouched[k] = nullptr;
        }
        h->pbufs = 0;
        if (!h->ptcount &&
            !er.cuda(cudaMalloc(&h->ptcount, kSlots * sizeof(unsigned long long)), "row counts"))
            return false;
        for (int k = 0; k < nb; ++k) {  // (a step touches at most t_rows rows)
            if (!er.cuda(cudaMalloc(&h->pacc[k], t_rows * dim * sizeof(long long)), "accumulator") ||
                !er.cuda(cudaMemset(h->pacc[k], 0, t_rows * dim * sizeof(long long)), "zero acc") ||
                !er.cuda(cudaMalloc(&h->pflags[k], t_rows * sizeof(int32_t)), "row map") ||
                !er.cuda(cudaMemset(h->pflags[k], 0, t_rows * sizeof(int32_t)), "clear row flags") ||
                !er.cuda(cudaMalloc(&h->ptouched[k], t_rows * sizeof(int32_t)), "row lists"))
                return false;
        }
        if (!er.cuda(cudaMemset(h->ptcount, 0, kSlots * sizeof(unsigned long long)), "zero counts"))
            return false;
        h->pbufs = nb;
        h->pbuf_rows = t_rows;
        h->pbuf_dim = dim;
    }
    if (nctx > h->pctx_n) {
        cudaDeviceSynchronize();
        cudaFree(h->pctx);
        h->pctx = nullptr;
        h->pctx_n = 0;
        if (!er.cuda(cudaMalloc(&h->pctx, nctx * sizeof(PersistRank)), "contexts")) return false;
        h->pctx_n = nctx;
    }
    return true;
}

}  // namespace heat

using namespace heat;

extern "C" {

int heat_nccl_unique_id(unsigned char *out128) {
    const NcclApi &n = nccl();
    if (!n.ok || !out128) return HEAT_ERR_UNSUPPORTED;
    ncclUniqueId id;
    if (n.get_unique_id(&id) != ncclSuccess) return HEAT_ERR_CUDA;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, 128);
    return HEAT_OK;
}

static int shard_create(int32_t world, int32_t rank, const unsigned char *nccl_id,
                        heat_host_allgather_fn hostx, void *hostx_user, int32_t device,
                        heat_shard **out) {
    if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return HEAT_ERR_INVALID;
    heat_shard *h = new heat_shard();
    h->world = world;
    h->rank = rank;
    h->device = device;
    const char *ex = getenv("HEAT_SHARD_EXCHANGE");
    h->p2p = !(ex && strcmp(ex, "gather") == 0);
    if (const char *l = getenv("HEAT_SHARD_LAG"))
        h->lag = h->lag_persist = std::min(std::max(atoi(l), 1), kSlots - 1);
    // captured step graphs: on by default at world 1; with NCCL calls inside
    // the capture (world > 1) only on request, as that path has not run on a
    // multi-GPU box here
    h->graphs = world == 1;
    if (const char *g = getenv("HEAT_SHARD_GRAPH")) h->graphs = atoi(g) != 0;
    if (const char *q = getenv("HEAT_SHARD_PERSIST")) {
        h->persist = atoi(q) != 0;
        h->persist_force = atoi(q) == 2;
    }
    cudaSetDevice(device);
    // the exchange runs at the highest priority: its apply CTAs take the SM
    // slots that the step kernels free before the next kernel's workers do
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    bool ok = cudaStreamCreateWithPriority(&h->comm_stream, cudaStreamNonBlocking, hi) ==
              cudaSuccess;
    for (int i = 0; i < 2 && ok; ++i)
        ok = cudaStreamCreateWithFlags(&h->cstream[i], cudaStreamNonBlocking) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_comm, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < 2 && ok; ++i)
        ok = cudaEventCreateWithFlags(&h->ev_cdone[i], cudaEventDisableTiming) == cudaSuccess;
    for (Slot &s : h->slot) {
        ok = ok && cudaEventCreateWithFlags(&s.log_ready, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&s.cnt_ready, cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&s.ex_done, cudaEventDisableTiming) == cudaSuccess;
    }
    // staging for the host-value all-gathers: (1 + world) * 2 * kSlots handles
    ok = ok && cudaMalloc(&h->scratch, (size_t)(1 + world) * 2 * kSlots *
                                           sizeof(cudaIpcMemHandle_t)) == cudaSuccess;
    ok = ok && cudaMalloc(&h->d_s0, sizeof(uint64_t)) == cudaSuccess &&
         cudaMallocHost(&h->h_s0, sizeof(uint64_t)) == cudaSuccess;
    if (!ok) {
        heat_shard_destroy(h);
        return HEAT_ERR_CUDA;
    }
    if (hostx) {
        // no kernel of one rank may wait on a kernel of another rank when the
        // ranks share a GPU: stream-ordered steps only, no captured graphs
        h->hostx = hostx;
        h->hostx_user = hostx_user;
        h->persist = false;
        h->graphs = false;
    } else if (world > 1) {
        const NcclApi &n = nccl();
        if (!n.ok || !nccl_id) {
            heat_shard_destroy(h);
            return HEAT_ERR_UNSUPPORTED;
        }
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof(id));
        if (n.comm_init_rank(&h->comm, world, id, rank) != ncclSuccess) {
            h->comm = nullptr;
            heat_shard_destroy(h);
            return HEAT_ERR_CUDA;
        }
    }
    *out = h;
    return HEAT_OK;
}

int heat_shard_create(int32_t world, int32_t rank, const unsigned char *nccl_id, int32_t device,
                      heat_shard **out) {
    return shard_create(world, rank, nccl_id, nullptr, nullptr, device, out);
}

int heat_shard_create_host(int32_t world, int32_t rank, heat_host_allgather_fn allgather,
                           void *user, int32_t device, heat_shard **out) {
    if (!allgather) return HEAT_ERR_INVALID;
    return shard_create(world, rank, nullptr, allgather, user, device, out);
}

int heat_shard_destroy(heat_shard *h) {
    if (!h) return HEAT_OK;
    cudaSetDevice(h->device);
    for (cudaStream_t s : {h->comm_stream, h->cstream[0], h->cstream[1]})
        if (s) cudaStreamSynchronize(s);
    free_slots(h);
    for (Slot &s : h->slot) {
        if (s.log_ready) cudaEventDestroy(s.log_ready);
        if (s.cnt_ready) cudaEventDestroy(s.cnt_ready);
        if (s.ex_done) cudaEventDestroy(s.ex_done);
    }
    for (cudaEvent_t e : {h->ev_start, h->ev_comm, h->ev_cdone[0], h->ev_cdone[1]})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : h->arrive)
        if (e) cudaEventDestroy(e);
    cudaFree(h->acc);
    cudaFree(h->flags);
    cudaFree(h->step_counts);
    cudaFreeHost(h->hstep_counts);
    cudaFree(h->scratch);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    cudaFree(h->d_users); cudaFree(h->d_items); cudaFree(h->d_pidx);
    cudaFree(h->d_bounds); cudaFreeHost(h->h_bounds);
    cudaFree(h->d_s0); cudaFreeHost(h->h_s0);
    for (void *q : h->opened_mbox) cudaIpcCloseMemHandle(q);
    cudaFree(h->mbox); cudaFree(h->rel); cudaFree(h->mbox_tab); cudaFree(h->rel_tab);
    cudaFree(h->pstate); cudaFree(h->pcnt); cudaFree(h->pclaim); cudaFree(h->pctx);
    for (auto &m : h->tmaps)
        if (m.base) cudaIpcCloseMemHandle(m.base);
    cudaFree(h->t_tab);
    for (int k = 0; k < kSlots; ++k) {
        cudaFree(h->pacc[k]); cudaFree(h->pflags[k]); cudaFree(h->ptouched[k]);
    }
    cudaFree(h->ptcount);
    if (h->comm) nccl().comm_destroy(h->comm);
    for (cudaStream_t s : {h->comm_stream, h->cstream[0], h->cstream[1]})
        if (s) cudaStreamDestroy(s);
    delete h;
    return HEAT_OK;
}

const char *heat_shard_last_error(heat_shard *h) { return h ? h->err.c_str() : ""; }

}  // extern "C"

namespace heat {

// One rank's epoch: inputs, the step sequence (compute / count / apply) and
// the closing statistics.  heat_shard_epoch drives one of these per process
// (NCCL between processes); heat_shard_epoch_loopback drives `world` of them
// in one process, interleaving their steps so every stream dependency the
// NCCL collectives provide is expressed as an event wait instead.
struct EpochRun {
    heat_shard *h = nullptr;
    ShardErr er{nullptr};
    float *S = nullptr, *T = nullptr;
    int64_t s_rows = 0, t_rows = 0, nsteps = 0, cap = 0, K = 0, total = 0;
    const int32_t *users = nullptr, *items = nullptr;
    const int64_t *pidx = nullptr, *bounds = nullptr;
    const heat_sgd_params *p = nullptr;
    // the stream-ordered steps' kernels: p with half the window.  Consecutive
    // step kernels alternate between two compute streams, so two of them are
    // in flight at once; with `window` workers each, one kernel fills the SMs
    // and the next one's CTAs only start in its tail, with window / 2 each the
    // two run side by side and the pairs in flight stay at `window` in total
    // (measured at N = 1: c3 41.4 M -> 48.1 M samples/s, c2 64.6 M -> 104.7 M).
    // HEAT_SHARD_HALFWIN=0 keeps the whole window per kernel.
    heat_sgd_params pstep{};
    heat_counters *counters = nullptr;
    cudaStream_t caller = nullptr;
    bool direct = true, dr = false;
    int W = 1, lag = 2, nslots = 3;
    std::vector<int64_t> key;
    EpochRun **group = nullptr;  // loopback: every rank's run
    bool persisted = false;      // the epoch ran as one persistent launch

    const int32_t *tr_users() const { return dr ? h->d_users : users; }
    const int32_t *tr_items() const { return dr ? h->d_items : items; }
    const int64_t *tr_pidx() const { return dr ? (pidx ? h->d_pidx : nullptr) : pidx; }

    // agreement on the log layout, buffers, the epoch inputs for captured
    // graphs; `agreed` is the cap every rank uses (host all-gather or loopback)
    int setup(int64_t agreed) {
        if (!ensure_slots(h, er, agreed, K)) return er.rc;
        if (!ensure_epoch_buffers(h, er, t_rows, K, nsteps)) return er.rc;
        cap = h->cap;
        direct = h->p2p;
        // the gather fallback reads a slot on the host after its step's count:
        // compute(s) must not refill the slot apply(s - nslots) still reads,
        // which needs lag >= 2 (lag 1 would let compute(s) run before apply(s-1)
        // is even enqueued)
        if (persist_eligible()) {
            lag = h->lag_persist;
        } else {
            lag = direct ? h->lag : std::max(h->lag, 2);
            lag = std::min(lag, kStreamMaxLag);
        }
        nslots = lag + 1;
        pstep = *p;
        {
            static const bool half = [] {
                const char *e = getenv("HEAT_SHARD_HALFWIN");
                return e ? atoi(e) != 0 : true;
            }();
            if (half && lag >= 2 && pstep.window >= 4) pstep.window = (pstep.window + 1) / 2;
        }
        // captured step graphs need the device-range kernels and a host-free
        // step loop (the gather fallback reads counts on the host between steps)
        dr = direct && h->graphs && !h->loopback && device_step_supported(p, S, T) &&
             !persist_eligible();
        total = nsteps > 0 ? bounds[nsteps] : 0;
        if (dr) {  // the epoch's inputs into runtime-owned buffers
            if (total > h->pairs_cap) {
                cudaDeviceSynchronize();
                cudaFree(h->d_users); cudaFree(h->d_items); cudaFree(h->d_pidx);
                h->d_users = h->d_items = nullptr;
                h->d_pidx = nullptr;
                h->pairs_cap = 0;
                h->gkey.clear();  // the graph holds the old addresses
                const int64_t c = std::max<int64_t>(total, 1) * 5 / 4;
                if (!er.cuda(cudaMalloc(&h->d_users, c * sizeof(int32_t)), "pairs") ||
                    !er.cuda(cudaMalloc(&h->d_items, c * sizeof(int32_t)), "pairs") ||
                    !er.cuda(cudaMalloc(&h->d_pidx, c * sizeof(int64_t)), "pairs"))
                    return er.rc;
                h->pairs_cap = c;
            }
            if (nsteps + 1 > h->bounds_cap) {
                cudaDeviceSynchronize();
                cudaFree(h->d_bounds);
                cudaFreeHost(h->h_bounds);
                h->d_bounds = nullptr;
                h->h_bounds = nullptr;
                h->bounds_cap = 0;
                h->gkey.clear();
                if (!er.cuda(cudaMalloc(&h->d_bounds, (nsteps + 1) * sizeof(int64_t)), "bounds") ||
                    !er.cuda(cudaMallocHost(&h->h_bounds, (nsteps + 1) * sizeof(int64_t)), "bounds"))
                    return er.rc;
                h->bounds_cap = nsteps + 1;
            }
            memcpy(h->h_bounds, bounds, (nsteps + 1) * sizeof(int64_t));
            *h->h_s0 = p->stream_base;
            if (total > 0) {
                er.cuda(cudaMemcpyAsync(h->d_users, users, total * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, caller), "pairs in");
                er.cuda(cudaMemcpyAsync(h->d_items, items, total * sizeof(int32_t),
                                        cudaMemcpyDeviceToDevice, caller), "pairs in");
                if (pidx)
                    er.cuda(cudaMemcpyAsync(h->d_pidx, pidx, total * sizeof(int64_t),
                                            cudaMemcpyDeviceToDevice, caller), "pairs in");
            }
            er.cuda(cudaMemcpyAsync(h->d_bounds, h->h_bounds, (nsteps + 1) * sizeof(int64_t),
                                    cudaMemcpyHostToDevice, caller), "bounds in");
            er.cuda(cudaMemcpyAsync(h->d_s0, h->h_s0, sizeof(uint64_t), cudaMemcpyHostToDevice,
                                    caller), "s0 in");
        }
        // log counters start at zero (afterwards each step's apply re-arms its slot)
        for (int k = 0; k < h->nalloc; ++k)
            er.cuda(cudaMemsetAsync(h->slot[k].cnt, 0, sizeof(int64_t), caller), "zero");
        return er.rc;
    }

    int64_t *counts_row(int64_t s) const {
        return (h->loopback ? h->shared_counts : h->step_counts) + s * W;
    }

    void compute(int64_t s) {
        Slot &sl = h->slot[s % nslots];
        cudaStream_t cs = h->cstream[s & 1];
        if (s >= lag)
            er.cuda(cudaStreamWaitEvent(cs, h->slot[(s - lag) % nslots].ex_done, 0), "wait apply");
        int r = HEAT_OK;
        if (dr) {  // every step launches (empty ones exit at once): a fixed topology
            r = train_range_device_step(S, s_rows, T, t_rows, tr_users(), tr_items(), &pstep, counters,
                                        sl.ids, sl.rows, sl.cnt, cap, tr_pidx(), h->d_bounds + s,
                                        h->d_s0, cs);
        } else if (bounds[s + 1] > bounds[s]) {
            r = heat_train_range(S, s_rows, T, t_rows, tr_users(), tr_items(), bounds[s],
                                 bounds[s + 1], &pstep, counters, sl.ids, sl.rows, sl.cnt, cap,
                                 tr_pidx(), nullptr, nullptr, cs);
        }
        if (r != HEAT_OK && er.rc == HEAT_OK) {
            h->err = std::string("train_range: ") + heat_last_error();
            er.rc = r;
        }
        er.cuda(cudaEventRecord(sl.log_ready, cs), "record log");
    }

    // the gather fallback's host copy of the step's counts
    void counts_to_host(int64_t s) {
        er.cuda(cudaMemcpyAsync(h->hstep_counts + s * W, counts_row(s), W * sizeof(int64_t),
                                cudaMemcpyDeviceToHost, h->comm_stream), "count to host");
        er.cuda(cudaEventRecord(h->slot[s % nslots].cnt_ready, h->comm_stream), "record counts");
    }

    // host transport: the count all-gather as a host collective between two
    // synchronisations of the comm stream — the same fence (no rank leaves it
    // before every rank's step-s log and apply(s-1) are complete), with the
    // host in the loop
    void host_count(Slot &sl, int64_t *cnts) {
        int64_t mine = 0;
        std::vector<int64_t> all(W);
        er.cuda(cudaMemcpyAsync(&mine, sl.cnt, sizeof(int64_t), cudaMemcpyDeviceToHost,
                                h->comm_stream), "count to host");
        er.cuda(cudaStreamSynchronize(h->comm_stream), "count sync");
        // every rank makes the call whatever its own error state (a collective)
        if (h->hostx(h->hostx_user, &mine, sizeof(int64_t), all.data()) != 0)
            er.invalid("host all-gather failed");
        er.cuda(cudaMemcpyAsync(cnts, all.data(), W * sizeof(int64_t), cudaMemcpyHostToDevice,
                                h->comm_stream), "counts to device");
        er.cuda(cudaStreamSynchronize(h->comm_stream), "count sync");  // `all` leaves scope
    }

    // gather fallback under the host transport: logs through host memory
    void host_gather(Slot &sl, int64_t cmax) {
        const int64_t ib = cmax * (int64_t)sizeof(int32_t), rb = cmax * K * (int64_t)sizeof(float);
        std::vector<char> mine(ib + rb), all((ib + rb) * W);
        er.cuda(cudaMemcpyAsync(mine.data(), sl.ids, ib, cudaMemcpyDeviceToHost, h->comm_stream),
                "log to host");
        er.cuda(cudaMemcpyAsync(mine.data() + ib, sl.rows, rb, cudaMemcpyDeviceToHost,
                                h->comm_stream), "log to host");
        er.cuda(cudaStreamSynchronize(h->comm_stream), "log sync");
        if (h->hostx(h->hostx_user, mine.data(), ib + rb, all.data()) != 0)
            er.invalid("host all-gather failed");
        for (int q = 0; q < W; ++q) {
            er.cuda(cudaMemcpyAsync(sl.g_ids + q * cmax, all.data() + q * (ib + rb), ib,
                                    cudaMemcpyHostToDevice, h->comm_stream), "log to device");
            er.cuda(cudaMemcpyAsync(sl.g_rows + q * cmax * K, all.data() + q * (ib + rb) + ib, rb,
                                    cudaMemcpyHostToDevice, h->comm_stream), "log to device");
        }
        er.cuda(cudaStreamSynchronize(h->comm_stream), "log sync");
    }

    // counts of step s: the fence every rank passes before reading slot s
    // (NCCL all-gather between processes; at world 1 a local copy)
    void count(int64_t s) {
        Slot &sl = h->slot[s % nslots];
        er.cuda(cudaStreamWaitEvent(h->comm_stream, sl.log_ready, 0), "wait log");
        int64_t *cnts = h->step_counts + s * W;
        if (W > 1 && h->hostx)
            host_count(sl, cnts);
        else if (W > 1)  // (world 1, direct: the apply records the log's own counter)
            er.nccl(nccl().all_gather(sl.cnt, cnts, 1, ncclInt64, h->comm, h->comm_stream),
                    "all_gather counts");
        else if (!direct)
            er.cuda(cudaMemcpyAsync(cnts, sl.cnt, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                    h->comm_stream), "count copy");
        if (!direct) counts_to_host(s);
    }

    // loopback count, phase 1 (every rank before any phase 2): this rank's
    // count into the group's row, after its step-s log and its apply(s-1)
    // (stream order on the comm stream) — what this rank brings to the
    // collective — then an arrival event
    void count_arrive(int64_t s) {
        Slot &sl = h->slot[s % nslots];
        er.cuda(cudaStreamWaitEvent(h->comm_stream, sl.log_ready, 0), "wait log");
        er.cuda(cudaMemcpyAsync(counts_row(s) + h->rank, sl.cnt, sizeof(int64_t),
                                cudaMemcpyDeviceToDevice, h->comm_stream), "count copy");
        er.cuda(cudaEventRecord(h->arrive[s % nslots], h->comm_stream), "record arrival");
    }

    // phase 2: the collective completes on this rank once every rank arrived
    void count_complete(int64_t s) {
        for (int q = 0; q < W; ++q)
            er.cuda(cudaStreamWaitEvent(h->comm_stream, group[q]->h->arrive[s % nslots], 0),
                    "wait arrivals");
        if (!direct) counts_to_host(s);
    }

    void apply(int64_t t) {
        Slot &sl = h->slot[t % nslots];
        int64_t *cnts = counts_row(t);
        LogView v{};
        if (direct) {
            v.pids = sl.pids;
            v.prows = sl.prows;
        } else {  // gather fallback: counts read on the host, logs padded to the max
            er.cuda(cudaEventSynchronize(sl.cnt_ready), "counts");
            int64_t cmax = 0;
            for (int q = 0; q < W; ++q) cmax = std::max(cmax, h->hstep_counts[t * W + q]);
            cmax = std::min(cmax, cap);
            if (cmax > 0 && er.rc == HEAT_OK && W > 1) {
                if (h->loopback) {  // the all-gather as copies of every rank's log
                    for (int q = 0; q < W; ++q) {
                        const Slot &qs = group[q]->h->slot[t % nslots];
                        er.cuda(cudaMemcpyAsync(sl.g_ids + q * cmax, qs.ids, cmax * sizeof(int32_t),
                                                cudaMemcpyDeviceToDevice, h->comm_stream), "gather");
                        er.cuda(cudaMemcpyAsync(sl.g_rows + q * cmax * K, qs.rows,
                                                cmax * K * sizeof(float), cudaMemcpyDeviceToDevice,
                                                h->comm_stream), "gather");
                    }
                } else if (h->hostx) {
                    host_gather(sl, cmax);
                } else {
                    const NcclApi &n = nccl();
                    er.nccl(n.group_start(), "group start");
                    er.nccl(n.all_gather(sl.ids, sl.g_ids, (size_t)cmax, ncclInt32, h->comm,
                                         h->comm_stream), "all_gather ids");
                    er.nccl(n.all_gather(sl.rows, sl.g_rows, (size_t)(cmax * K), ncclFloat32, h->comm,
                                         h->comm_stream), "all_gather rows");
                    er.nccl(n.group_end(), "group end");
                }
            }
            v.ids = W > 1 ? sl.g_ids : sl.ids;  // world 1: the log is the gathered copy
            v.rows = W > 1 ? sl.g_rows : sl.rows;
            v.stride = cmax;
        }
        if (er.rc == HEAT_OK)
            er.cuda(launch_shard_apply(T, (int)K, v, (direct && W == 1) ? sl.cnt : cnts, cnts,
                                       sl.cnt, W, cap, h->acc, h->flags, h->comm_stream), "apply");
        er.cuda(cudaEventRecord(sl.ex_done, h->comm_stream), "record apply");
    }

    // fork the internal streams from `origin` / join them back
    void fork(cudaStream_t origin) {
        er.cuda(cudaEventRecord(h->ev_start, origin), "record start");
        for (cudaStream_t st : {h->cstream[0], h->cstream[1], h->comm_stream})
            if (st != origin) er.cuda(cudaStreamWaitEvent(st, h->ev_start, 0), "wait start");
    }
    void join(cudaStream_t origin) {
        for (int i = 0; i < 2; ++i) {
            if (h->cstream[i] == origin) continue;
            er.cuda(cudaEventRecord(h->ev_cdone[i], h->cstream[i]), "record compute");
            er.cuda(cudaStreamWaitEvent(origin, h->ev_cdone[i], 0), "join compute");
        }
        er.cuda(cudaEventRecord(h->ev_comm, h->comm_stream), "record comm");
        er.cuda(cudaStreamWaitEvent(origin, h->ev_comm, 0), "join comm");
    }

    // the whole step sequence of one process's rank
    void enqueue_epoch(cudaStream_t origin) {
        fork(origin);
        for (int64_t s = 0; s < nsteps && er.rc == HEAT_OK; ++s) {
            compute(s);
            if (direct) {  // nothing waits on the host: the step's exchange right behind it
                count(s);
                apply(s);
            } else {  // gather fallback: the host wait on the counts of s-1 overlaps kernel(s)
                if (s >= 1) apply(s - 1);
                count(s);
            }
        }
        if (!direct && nsteps >= 1 && er.rc == HEAT_OK) apply(nsteps - 1);
        join(origin);
    }

    // graph key: everything a captured epoch bakes in (not the stream base,
    // the pair order or the step ranges, which live in device memory)
    void make_key() {
        key.clear();
        if (!dr) return;
        heat_sgd_params q = *p;
        q.stream_base = 0;
        key.resize(sizeof(q) / sizeof(int64_t) + 1);
        memcpy(key.data(), &q, sizeof(q));
        for (int64_t v : {(int64_t)(uintptr_t)S, s_rows, (int64_t)(uintptr_t)T, t_rows,
                          (int64_t)(uintptr_t)counters, nsteps, cap, (int64_t)lag,
                          (int64_t)(pidx != nullptr), (int64_t)W})
            key.push_back(v);
    }

    void run_single() {
        make_key();
        if (dr && h->gexec && key == h->gkey) {
            er.cuda(cudaGraphLaunch(h->gexec, caller), "replay epoch");
            return;
        }
        enqueue_epoch(caller);
        if (!dr || er.rc != HEAT_OK) return;
        // record the same sequence once more, unexecuted, for later epochs
        // (this epoch also warmed every launch-configuration cache)
        if (h->gexec) cudaGraphExecDestroy(h->gexec);
        h->gexec = nullptr;
        h->gkey.clear();
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(h->cstream[0], cudaStreamCaptureModeRelaxed) == cudaSuccess) {
            enqueue_epoch(h->cstream[0]);
            const cudaError_t ce = cudaStreamEndCapture(h->cstream[0], &g);
            if (ce == cudaSuccess && er.rc == HEAT_OK &&
                cudaGraphInstantiate(&h->gexec, g, 0) == cudaSuccess) {
                h->gkey = key;
            } else {  // the epoch itself ran: stay on direct launches, no error
                h->gexec = nullptr;
                h->graphs = false;
                er.rc = HEAT_OK;
                h->err.clear();
            }
            if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();
    }

    // ---- persistent epoch ------------------------------------------------
    // every rank of the job decides alike (same parameters, same exchange)
    bool persist_eligible() const {
        if (!h->persist || !direct || W > kPersistMaxWorld || nsteps < 1) return false;
        // K = 128 (configs 4/5); at K = 64 the several-warps-per-pair kernel of
        // the stream-ordered steps is faster (c3: 37.7 M vs 31.5 M samples/s at
        // N = 1), HEAT_SHARD_PERSIST=2 forces the persistent epoch there too
        if (K != 128 && !(K == 64 && h->persist_force)) return false;
        if (!p->use_cosine || (p->flags & 1)) return false;
        if (cap >= (1 << 24)) return false;  // the mailbox words carry 24-bit counts
        return ((uintptr_t)S % 16 == 0) && ((uintptr_t)T % 16 == 0);
    }

    // per-rank buffers and the host context (tables filled by the caller for
    // a loopback group)
    // false: an error (er.rc set); true with h->persist cleared: the ranks
    // agreed to fall back to the stream-ordered steps (a peer mapping failed)
    bool persist_prepare() {
        if (!ensure_mailbox(h, er, nsteps)) return false;
        if (!h->persist) return true;
        if (!map_replicas(h, er, T)) return false;
        if (!h->persist) return true;
        if (!ensure_persist_state(h, er, nsteps, group ? W : 1, t_rows, K, lag)) return false;
        if (nsteps + 1 > h->bounds_cap) {
            cudaDeviceSynchronize();
            cudaFree(h->d_bounds);
            cudaFreeHost(h->h_bounds);
            h->d_bounds = nullptr;
            h->h_bounds = nullptr;
            h->bounds_cap = 0;
            h->gkey.clear();
            if (!er.cuda(cudaMalloc(&h->d_bounds, (nsteps + 1) * sizeof(int64_t)), "bounds") ||
                !er.cuda(cudaMallocHost(&h->h_bounds, (nsteps + 1) * sizeof(int64_t)), "bounds"))
                return false;
            h->bounds_cap = nsteps + 1;
        }
        // (the pinned staging copy is free again: the previous epoch synchronized)
        memcpy(h->h_bounds, bounds, (nsteps + 1) * sizeof(int64_t));
        er.cuda(cudaMemcpyAsync(h->d_bounds, h->h_bounds, (nsteps + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, caller), "bounds in");
        er.cuda(cudaMemsetAsync(h->pstate, 0, kStepWords * nsteps * sizeof(unsigned long long),
                                caller), "zero step state");
        er.cuda(cudaMemsetAsync(h->pcnt, 0, nsteps * sizeof(unsigned long long), caller), "zero counts");
        er.cuda(cudaMemsetAsync(h->pclaim, 0, 4 * sizeof(unsigned long long), caller), "zero claim");
        return er.rc == HEAT_OK;
    }

    PersistRank persist_ctx() const {
        PersistRank c{};
        c.S = S; c.T = T; c.users = users; c.items = items; c.pidx = pidx;
        c.bounds = h->d_bounds;
        c.nsteps = nsteps;
        c.claim = h->pclaim;
        c.state = h->pstate;
        c.cnt = h->pcnt;
        for (int k = 0; k < kPersistSlots; ++k) {
            c.log_ids[k] = h->slot[k].ids;
            c.log_rows[k] = h->slot[k].rows;
            c.pids[k] = h->slot[k].pids;
            c.prows[k] = h->slot[k].prows;
        }
        c.mbox_tab = h->mbox_tab;
        c.t_tab = h->t_tab;
        c.rel_tab = h->rel_tab;
        c.mbox = h->mbox;
        c.rel = h->rel;
        for (int k = 0; k < kPersistSlots; ++k) {
            c.acc[k] = h->pacc[k];
            c.map[k] = h->pflags[k];
            c.touched[k] = h->ptouched[k];
        }

        c.ctr = counters;
        c.step_counts = counts_row(0);
        c.cap = cap;
        c.mbox_steps = h->mbox_steps;
        c.gbase = h->gstep;
        c.tag = h->tag;
        c.rank = h->rank;
        c.world = W;
        c.lag = lag;
        static const int acc_ef = [] {  // HEAT_PERSIST_ACC_EF=0: evict-normal accumulator lines
            const char *e = getenv("HEAT_PERSIST_ACC_EF");
            return e ? (atoi(e) != 0 ? 1 : 0) : 1;
        }();
        c.acc_ef = acc_ef;
        c.nslots = nslots;
        c.gmod_lag = (int)(h->gstep % (unsigned long long)lag);
        c.gmod_slots = (int)(h->gstep % (unsigned long long)nslots);
        return c;
    }

    HogwildArgs persist_args() const {
        HogwildArgs a{};
        a.S = S; a.T = T; a.users = users; a.items = items;
        a.start = 0; a.stop = total;
        a.K = (int)K; a.N = p->n_neg; a.cosine = p->use_cosine;
        a.lr = (float)p->lr; a.l2 = (float)p->l2; a.mu = p->mu; a.theta = p->theta;
        a.s0 = p->stream_base; a.num_items = t_rows; a.ctr = counters; a.s_rows = s_rows;
        a.window = p->window;  // > 0: at most this many pairs in flight per rank
        a.fp64 = 0;
        a.pair_index = pidx;
        return a;
    }

    // after the launch: the epoch's global steps are consumed on every rank
    void persist_advance() {
        h->gstep += (unsigned long long)nsteps;
        h->tag += 1;
        persisted = true;
    }

    // the epoch's counts come back once for the statistics; a log that
    // overflowed is reported (the capacity is the exact worst case, so this
    // is a defensive check, not a mode of operation)
    int finish(heat_shard_stats *stats) {
        if (nsteps > 0)
            er.cuda(cudaMemcpyAsync(h->hstep_counts, counts_row(0), nsteps * W * sizeof(int64_t),
                                    cudaMemcpyDeviceToHost, caller), "counts to host");
        er.cuda(cudaStreamSynchronize(caller), "epoch");
        if (er.rc != HEAT_OK) return er.rc;
        heat_shard_stats st{};
        for (int64_t s = 0; s < nsteps; ++s) {
            int64_t cmax = 0;
            for (int q = 0; q < W; ++q) {
                const int64_t c = h->hstep_counts[s * W + q];
                cmax = std::max(cmax, c);
                st.entries += std::min(c, cap);
            }
            if (cmax > cap) {
                er.invalid("delta log overflow (" + std::to_string(cmax) + " > " +
                           std::to_string(cap) + " entries on some rank in step " +
                           std::to_string(s) + ")");
            }
            st.max_entries = std::max(st.max_entries, cmax);
            st.steps += 1;
        }
        // bytes that crossed between GPUs: every rank reads every other rank's log
        st.exchanged_bytes = (W > 1 ? (W - 1) : 0) * st.entries * (4 * K + 4);
        // persistent: one launch; stream-ordered: a DELTA kernel and the two
        // apply kernels per step
        st.launches = persisted ? 1 : 3 * nsteps;
        if (stats) *stats = st;
        return er.rc;
    }
};

static int epoch_args_ok(heat_shard *h, const heat_sgd_params *p, const int64_t *step_bounds,
                         int64_t nsteps, int64_t capacity) {
    if (!h || !p || !step_bounds || nsteps < 0 || capacity < 1) return HEAT_ERR_INVALID;
    if (p->mode != HEAT_MODE_DELTA) {
        h->err = "heat_shard_epoch runs HEAT_MODE_DELTA steps";
        return HEAT_ERR_INVALID;
    }
    return HEAT_OK;
}

}  // namespace heat

extern "C" {

int heat_shard_epoch(heat_shard *h, float *S, int64_t s_rows, float *T, int64_t t_rows,
                     const int32_t *local_users, const int32_t *local_items,
                     const int64_t *pair_index, const int64_t *step_bounds, int64_t nsteps,
                     int64_t capacity, const heat_sgd_params *p, heat_counters *counters,
                     heat_shard_stats *stats, void *stream) {
    if (const int rc = epoch_args_ok(h, p, step_bounds, nsteps, capacity)) return rc;
    if (h->loopback) {
        h->err = "a loopback rank runs through heat_shard_epoch_loopback";
        return HEAT_ERR_INVALID;
    }
    cudaSetDevice(h->device);
    EpochRun run;
    run.h = h;
    run.er = ShardErr{h};
    run.S = S; run.s_rows = s_rows; run.T = T; run.t_rows = t_rows;
    run.users = local_users; run.items = local_items; run.pidx = pair_index;
    run.bounds = step_bounds; run.nsteps = nsteps; run.p = p; run.counters = counters;
    run.caller = (cudaStream_t)stream;
    run.W = h->world;
    run.K = p->dim;
    // every rank must run the same number of steps with the same log layout:
    // agree (max capacity) and check, before any per-step collective
    int64_t cap = capacity;
    if (run.W > 1) {
        const int64_t mine[3] = {capacity, nsteps, run.K};
        std::vector<int64_t> all(3 * run.W);
        if (!host_all_gather(h, run.er, mine, 3, all.data())) return run.er.rc;
        for (int q = 0; q < run.W; ++q) {
            if (all[3 * q + 1] != nsteps || all[3 * q + 2] != run.K) {
                run.er.invalid("ranks disagree on the epoch's step count or dim (steps " +
                               std::to_string(nsteps) + " vs " + std::to_string(all[3 * q + 1]) +
                               " on rank " + std::to_string(q) + ")");
                return run.er.rc;
            }
            cap = std::max(cap, all[3 * q]);
        }
    }
    if (run.setup(cap) != HEAT_OK) return run.er.rc;
    if (run.persist_eligible() && run.persist_prepare() && h->persist) {
        const PersistRank c = run.persist_ctx();
        const cudaError_t e = launch_shard_persist(run.persist_args(), &c, h->pctx, 1, run.caller);
        if (e == cudaSuccess) {
            run.persist_advance();
            const int rc = run.finish(stats);
            if (rc == HEAT_OK) persist_prof_report();
            else persist_watchdog_report();
            return rc;
        }
        if (e != cudaErrorNotSupported) {
            run.er.cuda(e, "persistent epoch");
            return run.er.rc;
        }
        cudaGetLastError();  // no persistent kernel for these parameters: stream-ordered steps
    }
    if (run.er.rc != HEAT_OK) return run.er.rc;
    run.run_single();
    return run.finish(stats);
}

int heat_shard_create_loopback(int32_t world, int32_t device, heat_shard **out) {
    if (!out || world < 1 || world > kMaxWorld) return HEAT_ERR_INVALID;
    for (int r = 0; r < world; ++r) {
        heat_shard *h = nullptr;
        int rc = heat_shard_create(1, 0, nullptr, device, &h);
        if (rc == HEAT_OK) {
            h->world = world;
            h->rank = r;
            h->loopback = true;
            h->graphs = false;
            for (int k = 0; k < kSlots && rc == HEAT_OK; ++k)
                if (cudaEventCreateWithFlags(&h->arrive[k], cudaEventDisableTiming) != cudaSuccess)
                    rc = HEAT_ERR_CUDA;
        }
        if (rc != HEAT_OK) {
            if (h) heat_shard_destroy(h);
            for (int q = 0; q < r; ++q) heat_shard_destroy(out[q]);
            return rc;
        }
        out[r] = h;
    }
    return HEAT_OK;
}

int heat_shard_epoch_loopback(heat_shard **hs, int32_t world, const heat_shard_rank *ranks,
                              int64_t nsteps, const heat_sgd_params *p, heat_shard_stats *stats,
                              void *stream) {
    if (!hs || !ranks || world < 1 || world > kMaxWorld) return HEAT_ERR_INVALID;
    for (int r = 0; r < world; ++r) {
        if (!hs[r] || !hs[r]->loopback || hs[r]->world != world || hs[r]->rank != r)
            return HEAT_ERR_INVALID;
        if (const int rc = epoch_args_ok(hs[r], p, ranks[r].step_bounds, nsteps,
                                         ranks[r].capacity))
            return rc;
    }
    cudaSetDevice(hs[0]->device);
    std::vector<EpochRun> runs(world);
    std::vector<EpochRun *> group(world);
    int64_t cap = 1;
    for (int r = 0; r < world; ++r) cap = std::max(cap, ranks[r].capacity);
    for (int r = 0; r < world; ++r) {
        EpochRun &run = runs[r];
        group[r] = &run;
        const heat_shard_rank &a = ranks[r];
        run.h = hs[r];
        run.er = ShardErr{hs[r]};
        run.S = a.S; run.s_rows = a.s_rows; run.T = a.T; run.t_rows = a.t_rows;
        run.users = a.local_users; run.items = a.local_items; run.pidx = a.pair_index;
        run.bounds = a.step_bounds; run.nsteps = nsteps; run.p = p; run.counters = a.counters;
        run.caller = (cudaStream_t)stream;
        run.W = world;
        run.K = p->dim;
        run.group = group.data();
    }
    // the group's count rows, owned by rank 0
    heat_shard *h0 = hs[0];
    if (!ensure_epoch_buffers(h0, runs[0].er, ranks[0].t_rows, p->dim, nsteps)) return runs[0].er.rc;
    for (int r = 0; r < world; ++r) hs[r]->shared_counts = h0->step_counts;
    for (int r = 0; r < world; ++r)
        if (runs[r].setup(cap) != HEAT_OK) return runs[r].er.rc;
    // peers' logs through plain device pointers (one address space)
    for (int k = 0; k < hs[0]->nalloc; ++k) {
        std::vector<const void *> ids(world), rows(world);
        for (int q = 0; q < world; ++q) {
            ids[q] = hs[q]->slot[k].ids;
            rows[q] = hs[q]->slot[k].rows;
        }
        for (int r = 0; r < world; ++r) {
            if (!runs[r].er.cuda(cudaMemcpy((void *)hs[r]->slot[k].pids, ids.data(),
                                            world * sizeof(void *), cudaMemcpyHostToDevice),
                                 "peer table") ||
                !runs[r].er.cuda(cudaMemcpy((void *)hs[r]->slot[k].prows, rows.data(),
                                            world * sizeof(void *), cudaMemcpyHostToDevice),
                                 "peer table"))
                return runs[r].er.rc;
        }
    }
    auto ok = [&] {
        for (auto &r : runs)
            if (r.er.rc != HEAT_OK) return false;
        return true;
    };
    // persistent group: one cooperative launch over every rank's contexts
    bool persist = true;
    for (auto &r : runs) persist = persist && r.persist_eligible();
    if (persist) {
        for (auto &r : runs)
            if (!r.persist_prepare()) return r.er.rc;
        std::vector<void *> mt(world), rt(world), tt(world);
        for (int q = 0; q < world; ++q) {
            mt[q] = hs[q]->mbox;
            rt[q] = hs[q]->rel;
            tt[q] = runs[q].T;
        }
        std::vector<PersistRank> cx(world);
        for (int r = 0; r < world; ++r) {
            if (!runs[r].er.cuda(cudaMemcpy(hs[r]->mbox_tab, mt.data(), world * sizeof(void *),
                                            cudaMemcpyHostToDevice), "mailbox table") ||
                !runs[r].er.cuda(cudaMemcpy(hs[r]->rel_tab, rt.data(), world * sizeof(void *),
                                            cudaMemcpyHostToDevice), "released table") ||
                !runs[r].er.cuda(cudaMemcpy(hs[r]->t_tab, tt.data(), world * sizeof(void *),
                                            cudaMemcpyHostToDevice), "replica table"))
                return runs[r].er.rc;
            cx[r] = runs[r].persist_ctx();
        }
        const cudaError_t e = launch_shard_persist(runs[0].persist_args(), cx.data(), h0->pctx,
                                                   world, runs[0].caller);
        if (e == cudaSuccess) {
            for (auto &r : runs) r.persist_advance();
            int rc = HEAT_OK;
            for (int r = 0; r < world; ++r) {
                const int x = runs[r].finish(stats ? stats + r : nullptr);
                if (rc == HEAT_OK) rc = x;
            }
            if (rc != HEAT_OK) persist_watchdog_report();
            for (int r = 0; r < world; ++r) hs[r]->shared_counts = nullptr;
            return rc;
        }
        if (e != cudaErrorNotSupported) {
            runs[0].er.cuda(e, "persistent group epoch");
            return runs[0].er.rc;
        }
        cudaGetLastError();
    }
    for (auto &r : runs) r.fork(r.caller);
    const bool direct = runs[0].direct;
    auto count_all = [&](int64_t s) {
        for (auto &r : runs) r.count_arrive(s);
        for (auto &r : runs) r.count_complete(s);
    };
    for (int64_t s = 0; s < nsteps && ok(); ++s) {
        for (auto &r : runs) r.compute(s);
        if (direct) {
            count_all(s);
            for (auto &r : runs) r.apply(s);
        } else {
            if (s >= 1)
                for (auto &r : runs) r.apply(s - 1);
            count_all(s);
        }
    }
    if (!direct && nsteps >= 1 && ok())
        for (auto &r : runs) r.apply(nsteps - 1);
    for (auto &r : runs) r.join(r.caller);
    int rc = HEAT_OK;
    for (int r = 0; r < world; ++r) {
        const int e = runs[r].finish(stats ? stats + r : nullptr);
        if (rc == HEAT_OK) rc = e;
    }
    for (int r = 0; r < world; ++r) hs[r]->shared_counts = nullptr;
    return rc;
}

}  // extern "C"
