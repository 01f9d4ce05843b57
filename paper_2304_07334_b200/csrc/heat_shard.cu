// heat_shard.cu — native runtime of the multi-GPU (user-sharded) epoch.
//
// users sharded u mod G, item table replicated, per-step
// item-delta exchange.  One process per GPU; this file is the per-rank step
// scheduler, in C++ so the host work between steps (a few event and stream
// calls) stays far below a step's kernel time.  Per step s, slot s%2:
//
//   compute stream:  [wait ex_done(s-2)] memset count; DELTA kernel -> log
//   comm stream:     all-gather counts(s); counts -> pinned host
//   host:            (while kernel(s+1) runs) wait counts(s), cmax = max
//   comm stream:     all-gather logs(s) (cmax entries per rank, one NCCL
//                    group), order-independent fixed-point apply -> T
//
// kernel(s) waits for the apply of s-2 (its log slot and the staleness bound);
// apply(s-1) runs beside kernel(s).  T changes only through the applies, which
// every rank performs on identical gathered logs with an integer (order-free)
// sum, so the item replicas stay bit-identical.  NCCL is resolved at run time
// from the copy torch already loaded (dlopen RTLD_NOLOAD), so the library has
// no link-time NCCL dependency and shares the process's NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

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
    int32_t *ids = nullptr;
    float *rows = nullptr;
    int64_t *cnt = nullptr;
    int64_t *counts = nullptr;   // world, device
    int64_t *hcounts = nullptr;  // world, pinned host
    int32_t *g_ids = nullptr;
    float *g_rows = nullptr;
    cudaEvent_t log_ready = nullptr, cnt_ready = nullptr, ex_done = nullptr;
};

}  // namespace heat

struct heat_shard {
    int world = 1, rank = 0, device = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    heat::Slot slot[2];
    int64_t cap = 0, dim = 0, acc_elems = 0, t_rows = 0;
    long long *acc = nullptr;
    int32_t *flags = nullptr;
    std::string err;
};

namespace heat {

// frees the log buffers of both slots (the events stay)
static void free_slots(heat_shard *h) {
    for (Slot &s : h->slot) {
        cudaFree(s.ids); cudaFree(s.rows); cudaFree(s.cnt); cudaFree(s.counts);
        cudaFreeHost(s.hcounts);
        if (h->world > 1) { cudaFree(s.g_ids); cudaFree(s.g_rows); }
        s.ids = nullptr; s.rows = nullptr; s.cnt = nullptr; s.counts = nullptr;
        s.hcounts = nullptr; s.g_ids = nullptr; s.g_rows = nullptr;
    }
    h->cap = 0;
}

static cudaError_t ensure_buffers(heat_shard *h, int64_t cap, int64_t dim, int64_t t_rows) {
    cudaError_t e = cudaSuccess;
    if (cap > h->cap || dim != h->dim) {
        cudaDeviceSynchronize();  // buffers of a previous epoch may still be in use
        free_slots(h);
        for (Slot &s : h->slot) {
            if ((e = cudaMalloc(&s.ids, cap * sizeof(int32_t)))) return e;
            if ((e = cudaMalloc(&s.rows, cap * dim * sizeof(float)))) return e;
            if ((e = cudaMalloc(&s.cnt, sizeof(int64_t)))) return e;
            if ((e = cudaMalloc(&s.counts, h->world * sizeof(int64_t)))) return e;
            if ((e = cudaMallocHost(&s.hcounts, h->world * sizeof(int64_t)))) return e;
            if (h->world > 1) {
                if ((e = cudaMalloc(&s.g_ids, h->world * cap * sizeof(int32_t)))) return e;
                if ((e = cudaMalloc(&s.g_rows, h->world * cap * dim * sizeof(float)))) return e;
            } else {  // world 1: the gathered log is the log itself
                s.g_ids = s.ids;
                s.g_rows = s.rows;
            }
        }
        h->cap = cap;
        h->dim = dim;
    }
    if (t_rows * dim > h->acc_elems || t_rows > h->t_rows) {
        cudaDeviceSynchronize();
        cudaFree(h->acc);
        cudaFree(h->flags);
        h->acc_elems = t_rows * dim;
        if ((e = cudaMalloc(&h->acc, t_rows * dim * sizeof(long long)))) return e;
        if ((e = cudaMalloc(&h->flags, t_rows * sizeof(int32_t)))) return e;
        if ((e = cudaMemset(h->acc, 0, t_rows * dim * sizeof(long long)))) return e;
        if ((e = cudaMemset(h->flags, 0, t_rows * sizeof(int32_t)))) return e;
        h->t_rows = t_rows;
    }
    return e;
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

int heat_shard_create(int32_t world, int32_t rank, const unsigned char *nccl_id, int32_t device,
                      heat_shard **out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return HEAT_ERR_INVALID;
    heat_shard *h = new heat_shard();
    h->world = world;
    h->rank = rank;
    h->device = device;
    cudaSetDevice(device);
    if (cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return HEAT_ERR_CUDA;
    }
    for (Slot &s : h->slot) {
        cudaEventCreateWithFlags(&s.log_ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.cnt_ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&s.ex_done, cudaEventDisableTiming);
    }
    if (world > 1) {
        const NcclApi &n = nccl();
        if (!n.ok || !nccl_id) {
            delete h;
            return HEAT_ERR_UNSUPPORTED;
        }
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof(id));
        if (n.comm_init_rank(&h->comm, world, id, rank) != ncclSuccess) {
            delete h;
            return HEAT_ERR_CUDA;
        }
    }
    *out = h;
    return HEAT_OK;
}

int heat_shard_destroy(heat_shard *h) {
    if (!h) return HEAT_OK;
    cudaStreamSynchronize(h->comm_stream);
    free_slots(h);
    for (Slot &s : h->slot) {
        cudaEventDestroy(s.log_ready);
        cudaEventDestroy(s.cnt_ready);
        cudaEventDestroy(s.ex_done);
    }
    cudaFree(h->acc);
    cudaFree(h->flags);
    if (h->comm) nccl().comm_destroy(h->comm);
    cudaStreamDestroy(h->comm_stream);
    delete h;
    return HEAT_OK;
}

const char *heat_shard_last_error(heat_shard *h) { return h ? h->err.c_str() : ""; }

int heat_shard_epoch(heat_shard *h, float *S, int64_t s_rows, float *T, int64_t t_rows,
                     const int32_t *local_users, const int32_t *local_items,
                     const int64_t *pair_index, const int64_t *step_bounds, int64_t nsteps,
                     int64_t capacity, const heat_sgd_params *p, heat_counters *counters,
                     heat_shard_stats *stats, void *stream) {
    if (!h || !p || !step_bounds || nsteps < 0 || capacity < 1) return HEAT_ERR_INVALID;
    if (p->mode != HEAT_MODE_DELTA) {
        h->err = "heat_shard_epoch runs HEAT_MODE_DELTA steps";
        return HEAT_ERR_INVALID;
    }
    cudaStream_t cs = (cudaStream_t)stream;
    const int W = h->world;
    const int64_t K = p->dim;
    cudaError_t e = ensure_buffers(h, capacity, K, t_rows);
    if (e != cudaSuccess) {
        h->err = std::string("buffer allocation: ") + cudaGetErrorString(e);
        return HEAT_ERR_CUDA;
    }
    const NcclApi &n = nccl();
    heat_shard_stats st{};
    int rc = HEAT_OK;
    auto check = [&](cudaError_t ce, const char *what) {
        if (ce != cudaSuccess && rc == HEAT_OK) {
            h->err = std::string(what) + ": " + cudaGetErrorString(ce);
            rc = HEAT_ERR_CUDA;
        }
    };
    auto nccl_check = [&](ncclResult_t r, const char *what) {
        if (r != ncclSuccess && rc == HEAT_OK) {
            h->err = std::string(what) + ": " + (n.error_string ? n.error_string(r) : "nccl error");
            rc = HEAT_ERR_CUDA;
        }
    };
    auto launch = [&](int64_t s) {
        Slot &sl = h->slot[s & 1];
        if (s >= 2) check(cudaStreamWaitEvent(cs, sl.ex_done, 0), "wait apply");
        check(cudaMemsetAsync(sl.cnt, 0, sizeof(int64_t), cs), "memset count");
        const int64_t a = step_bounds[s], b = step_bounds[s + 1];
        if (b > a) {
            const int r = heat_train_range(S, s_rows, T, t_rows, local_users, local_items, a, b, p,
                                           counters, sl.ids, sl.rows, sl.cnt, capacity,
                                           pair_index, nullptr, nullptr, cs);
            if (r != HEAT_OK && rc == HEAT_OK) {
                h->err = std::string("train_range: ") + heat_last_error();
                rc = r;
            }
        }
        check(cudaEventRecord(sl.log_ready, cs), "record log");
        check(cudaStreamWaitEvent(h->comm_stream, sl.log_ready, 0), "wait log");
        if (W > 1)
            nccl_check(n.all_gather(sl.cnt, sl.counts, 1, ncclInt64, h->comm, h->comm_stream),
                       "all_gather counts");
        else
            check(cudaMemcpyAsync(sl.counts, sl.cnt, sizeof(int64_t), cudaMemcpyDeviceToDevice,
                                  h->comm_stream), "count copy");
        check(cudaMemcpyAsync(sl.hcounts, sl.counts, W * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              h->comm_stream), "count to host");
        check(cudaEventRecord(sl.cnt_ready, h->comm_stream), "record counts");
    };
    auto exchange = [&](int64_t t) {
        Slot &sl = h->slot[t & 1];
        check(cudaEventSynchronize(sl.cnt_ready), "counts");  // kernel(t+1) already queued
        int64_t cmax = 0, total = 0;
        for (int r = 0; r < W; ++r) {
            cmax = std::max(cmax, sl.hcounts[r]);
            total += sl.hcounts[r];
        }
        if (cmax > capacity && rc == HEAT_OK) {
            h->err = "delta log overflow (" + std::to_string(cmax) + " > " +
                     std::to_string(capacity) + " entries on some rank); raise the capacity";
            rc = HEAT_ERR_INVALID;
        }
        if (cmax > 0 && rc == HEAT_OK) {
            if (W > 1) {
                nccl_check(n.group_start(), "group start");
                nccl_check(n.all_gather(sl.ids, sl.g_ids, (size_t)cmax, ncclInt32, h->comm,
                                        h->comm_stream), "all_gather ids");
                nccl_check(n.all_gather(sl.rows, sl.g_rows, (size_t)(cmax * K), ncclFloat32,
                                        h->comm, h->comm_stream), "all_gather rows");
                nccl_check(n.group_end(), "group end");
            }
            check(launch_apply_deltas_fixed(T, (int)K, sl.g_ids, sl.g_rows, sl.counts, W, cmax,
                                            h->acc, h->flags, h->comm_stream), "apply");
        }
        check(cudaEventRecord(sl.ex_done, h->comm_stream), "record apply");
        st.steps += 1;
        st.entries += total;
        st.exchanged_bytes += (int64_t)W * cmax * (4 * K + 4);
        st.max_entries = std::max(st.max_entries, cmax);
    };
    for (int64_t s = 0; s <= nsteps && rc == HEAT_OK; ++s) {
        if (s < nsteps) launch(s);
        if (s >= 1 && rc == HEAT_OK) exchange(s - 1);
    }
    // later work on the caller's stream sees every applied union
    for (int i = 0; i < 2 && i < nsteps; ++i) check(cudaStreamWaitEvent(cs, h->slot[i].ex_done, 0), "join");
    if (rc != HEAT_OK) {  // drain before reporting so buffers are idle
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(h->comm_stream);
    }
    if (stats) *stats = st;
    return rc;
}

}  // extern "C"
