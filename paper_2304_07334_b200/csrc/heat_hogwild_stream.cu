// heat_hogwild_stream.cu — the throughput SGD kernel for wide pairs
// (K = 64/128, hundreds of negatives: configs 3-5), register-streamed.
//
// Same math and semantics as the other throughput kernels (trainer.py:114-293
// per pair, Hogwild across pairs).  What differs is the data path.  A pair
// reads N+2 rows and writes ~1 + A of them, so the kernel is a gather of
// ~4K(N+2) bytes per pair from L2 (c3/c4: tables L2-resident) or HBM (c5).
// Staging those rows in shared memory (LDGSTS or TMA, then LDS) moves every
// byte through the SM's 128 B/clk shared-memory port twice, which caps a
// staged kernel at the same ~64 B/clk/SM the L2 can feed.  Here the rows go
// straight from L2 into registers:
//
//  * one warp per pair-worker; a row of K floats is read by 8 lanes
//    (K/8 columns each, LDG.128 of 128 contiguous bytes per 8 lanes), so one
//    warp instruction covers a GROUP of 4 rows and every L2 sector is used
//    whole;
//  * a register ring of P groups: group i+P's loads are issued as soon as
//    group i has been consumed, so each warp keeps 4P rows in flight with no
//    shared memory at all (c4: P = 4, 16 rows = 8 KB per warp);
//  * tt = v.v and st = u.v per lane with packed FFMA2, then a transposed
//    8-lane butterfly (4 shuffles per group of 4 rows): lanes 0-3 of a row
//    reduce tt while lanes 4-7 reduce st;
//  * the similarity screen is fp32 (error < 1e-6 for K <= 128; the band is
//    1e-5).  Rows that may be written — every candidate for sim > theta, the
//    positive, rows whose fp32 v.v underflows, decay rows when l2 != 0 — are
//    only RECORDED (id + flags) while streaming, so no row data is held past
//    its FFMA2s;
//  * after the pair's last round the recorded rows are re-read into a per-warp
//    shared-memory snapshot (a per-worker global spill area past its
//    capacity), and the band rows get tt and st in binary64 (warp-cooperative
//    sums; the user's u.u is the reference's sequential binary64 sum), so the
//    margin decisions are binary64 decisions (trainer.py:184-221), not fp32
//    ones.  Then every write is applied (red.global.add.v4, or logged in DELTA
//    mode) — all reads of a pair precede its writes, the reference's snapshot
//    semantics (trainer.py:118-146, 257-293);
//  * workers claim pairs from a per-launch atomic counter in epoch order, so
//    SMs that host fewer workers take more pairs (no tail from the uneven
//    window / 148 split).  Pairs in flight never exceed the worker count,
//    which the launcher caps at the window.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "heat_common.cuh"
#include "heat_internal.h"
#include "heat_row_update.cuh"

namespace heat {

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 0, but the compiler cannot tell: ties a load's address to a value so the
// load is not hoisted above the arithmetic that frees its target registers
__device__ __forceinline__ int32_t opaque_zero(float v) {
    int32_t z;
    asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(__float_as_uint(v)));
    return z;
}

__device__ __forceinline__ float4 ld_row4(const float *p, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// Per (device, stream) pair-claim counters: [0] next pair, [1] finished
// warps.  Zeroed once at allocation; the last warp of every launch re-arms
// them, so graph replays need no memset node.
unsigned long long *stream_claim(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t>, unsigned long long *> ctrs;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto &p = ctrs[std::make_tuple(dev, st)];
    if (!p) {
        if (cudaMalloc(&p, 2 * sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return nullptr;
        }
        cudaMemsetAsync(p, 0, 2 * sizeof(unsigned long long), st);
    }
    return p;
}

__global__ void row_policy_kernel(uint64_t *out) { *out = policy_evict_last(); }

// The evict-last descriptor createpolicy returns on this device (it is an
// opaque 64-bit value; asked from the device once per process and device).
uint64_t stream_row_policy() {
    static std::mutex mu;
    static std::map<int, uint64_t> made;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = made.find(dev);
    if (it != made.end()) return it->second;
    uint64_t v = 0, *d = nullptr;
    // (its own stream; the runtime's captures are relaxed-mode and come after
    // a plain first epoch, so this never runs inside one)
    if (cudaMalloc(&d, sizeof(v)) == cudaSuccess) {
        cudaStream_t s = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess) {
            row_policy_kernel<<<1, 1, 0, s>>>(d);
            if (cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
                cudaStreamSynchronize(s) != cudaSuccess)
                v = 0;
            cudaStreamDestroy(s);
        }
        cudaFree(d);
    }
    cudaGetLastError();
    if (v) made[dev] = v;
    return v;  // 0: no descriptor, the launchers decline
}

}  // namespace

// sum_k a[k]*b[k] over K floats widened to binary64, one k at a time, never
// contracted (trainer.py:177-178, 181-183, 195-197): the reference's value
template <int K>
__device__ __forceinline__ double seq_dot(const float *a, const float *b) {
    double acc = 0.0;
#pragma unroll 2
    for (int k = 0; k < K; k += 4) {
        const float4 x = *reinterpret_cast<const float4 *>(a + k);
        const float4 y = *reinterpret_cast<const float4 *>(b + k);
        acc = __dadd_rn(acc, __dmul_rn((double)x.x, (double)y.x));
        acc = __dadd_rn(acc, __dmul_rn((double)x.y, (double)y.y));
        acc = __dadd_rn(acc, __dmul_rn((double)x.z, (double)y.z));
        acc = __dadd_rn(acc, __dmul_rn((double)x.w, (double)y.w));
    }
    return acc;
}

// ---- persistent sharded epoch (MODE 2) --------------------------------------
// One launch trains a rank's whole epoch of DELTA steps (heat_shard.cu sets
// it up).  Item row id belongs to rank id % world (its OWNER), which alone
// computes the row's new value each step and stores it into every replica.
// Steps are gated on the device instead of by stream order:
//  * a pair of step s (global step g = gbase + s) starts once every rank has
//    applied its rows of every step up to g - lag (which also frees the log
//    slot g % (lag + 1) it will write);
//  * a written row's deltas go, if this rank owns the row, straight into the
//    step's accumulation buffer (g % lag: the steps that can be in flight at
//    once never share one) as 2^-40 fixed-point integer sums, the row joining
//    the buffer's row list; otherwise they are logged.  The warp that
//    finishes a step's last pair publishes the step's counts into every
//    rank's mailbox (one 8-byte store per rank, release at system scope: the
//    log it describes is complete);
//  * every rank applies its rows of each step in step order, the workers
//    doing the work between pairs: the peers' logged entries for its rows are
//    pulled over NVLink into the buffer in claimed chunks, then each touched
//    row is converted once (T += float(sum)) and the new row is stored into
//    every peer's replica.  Integer sums commute and each row has one
//    writer, so the replicas stay bit-identical, and a rank's apply work does
//    not grow with the world size;
//  * a finished apply is published as the rank's released-step count into
//    every rank's `rel` words (monotone, never reset between epochs).
// No warp waits on anything that is not already claimed by a running warp
// (on this rank) or a running kernel (on a peer), so progress needs no
// co-residency within a process; a loopback group (several ranks in one
// launch) is launched cooperatively, since its ranks wait on one another.
constexpr double kFix = 1099511627776.0;  // 2^40, as heat_shard.cu's apply kernels

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <class P>
__device__ __forceinline__ P *shfl_ptr(P *p, int src) {
    return reinterpret_cast<P *>(
        __shfl_sync(kFull, (unsigned long long)reinterpret_cast<uintptr_t>(p), src));
}
// accumulator traffic with an evict-first L2 policy, so it does not displace
// the tables' evict-last lines (HEAT_PERSIST_ACC_EF=0: evict-normal)
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t acc_policy(const PersistRank &R) {
    return R.acc_ef ? policy_evict_first() : policy_evict_normal();
}
__device__ __forceinline__ void red_u64_ef(unsigned long long *p, unsigned long long v, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ longlong2 ld_acc2(const long long *p, uint64_t pol) {
    longlong2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.s64 {%0, %1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void zero_acc2(long long *p, uint64_t pol) {
    asm volatile("st.global.cg.L2::cache_hint.v2.s64 [%0], {%1, %1}, %2;" ::"l"(p), "l"(0ll), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ unsigned long long fix40(float v) {
    return (unsigned long long)__double2ll_rn((double)v * kFix);
}

// per-warp bookkeeping of the persistent kernel (see below) and apply-work
// diagnostics: [8] help calls, [9] calls with nothing to do, [10] clocks in
// accumulate units, [11] clocks in convert units, [12] accumulate units
__shared__ long long s_pw[16];
// phase profile of one warp (PH builds): [0, 6) clocks per phase, [6] the
// last mark, [7] the start clock, [8] the start globaltimer
__shared__ long long s_ph[9];
__device__ __forceinline__ long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
}

// Watchdog of the device-side waits: a wait longer than ~20 s of clocks
// records (site, rank, step, block) in g_watchdog and traps, so a protocol
// bug surfaces as a launch error instead of a hung GPU.
__device__ unsigned long long g_watchdog[4];
__device__ __forceinline__ void watchdog(long long t0, int site, const PersistRank &R, long long s) {
    if (clock64() - t0 > 40000000000ll) {
        g_watchdog[0] = (unsigned long long)site;
        g_watchdog[1] = (unsigned long long)R.rank;
        g_watchdog[2] = (unsigned long long)s;
        g_watchdog[3] = blockIdx.x;
        __threadfence_system();
        __trap();
    }
}

// accumulation buffer and log slot of local step s (32-bit arithmetic on the
// host-computed residues of gbase: a 64-bit % is a call, and a call anywhere
// in the pair loop spills the streaming registers)
__device__ __forceinline__ int persist_buf(const PersistRank &R, long long s) {
    return (int)(((unsigned)R.gmod_lag + (unsigned)s) % (unsigned)R.lag);
}
__device__ __forceinline__ int persist_slot(const PersistRank &R, long long s) {
    return (int)(((unsigned)R.gmod_slots + (unsigned)s) % (unsigned)R.nslots);
}

// may a pair of global step g start? (lane q < world checks rank q's word)
__device__ __forceinline__ bool persist_gate_open(const PersistRank &R, long long g, int lane) {
    bool ok = true;
    if (lane < R.world) {  // every owner applied its rows of step g - lag
        const long long need = g - R.lag + 1;
        if (need > 0) ok = (long long)ld_acquire_sys(R.rel + lane) >= need;
    }
    return __all_sync(kFull, ok);
}

// step s's log on this rank is complete: its count into every rank's mailbox
__device__ __forceinline__ void persist_publish(const PersistRank &R, long long s, int lane) {
    if (R.world == 1) return;  // nobody reads it
    unsigned long long c = 0, wr = 0;
    if (lane == 0) {
        c = ld_acquire_gpu(R.cnt + s);                         // logged
        wr = ld_acquire_gpu(R.state + kWritten * R.nsteps + s);  // written
    }
    c = __shfl_sync(kFull, c, 0);
    wr = __shfl_sync(kFull, wr, 0);
    __threadfence_system();
    __syncwarp();
    if (lane < R.world) {
        const unsigned long long w = ((unsigned long long)(R.tag & 0xffffu) << 48) |
                                     ((wr & 0xffffffull) << 24) | (c & 0xffffffull);
        st_release_sys(R.mbox_tab[lane] + (((long long)(R.tag & 1) * R.mbox_steps + s) * R.world + R.rank), w);
    }
}

// one logged row (this lane's columns 32j + 4c .. +3) into buffer b, when
// `ok` (all lanes of the warp call it, each 8-lane group with its own row).
// The sums are compact: the row's first adder of the step claims the next
// entry of the step's row list (its map word goes 0 -> kMapBusy -> entry + 1)
// and the row's sums live at that entry, so a step's buffer is the rows it
// touched, contiguous and reused step after step (it stays in L2; sums
// indexed by row id spread every step over t_rows * K * 8 bytes and went to
// DRAM: 9 GB of writes per c4 epoch).  A later adder of the same row waits
// only for the first adder's two atomics.
constexpr int32_t kMapBusy = -1;
__device__ __forceinline__ int32_t ld_acquire_gpu_s32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <int K>
__device__ __forceinline__ void persist_accumulate(const PersistRank &R, int b, long long step,
                                                   int32_t id, int c, bool ok,
                                                   const float4 (&d)[K / 32]) {
    int32_t e = 0;
    if (ok && c == 0) {
        int32_t *mw = R.map[b] + id;
        int32_t v = atomicCAS(mw, 0, kMapBusy);
        if (v == 0) {
            e = (int32_t)atomicAdd(R.state + kRows * R.nsteps + step, 1ull);
            R.touched[b][e] = id;
            atomicExch(mw, e + 1);  // (the entry's sums start zeroed)
        } else {
            while (v == kMapBusy) v = ld_acquire_gpu_s32(mw);
            e = v - 1;
        }
    }
    e = __shfl_sync(kFull, e, threadIdx.x & ~7);
    if (!ok) return;
    unsigned long long *ac = reinterpret_cast<unsigned long long *>(R.acc[b] + (int64_t)e * K + 4 * c);
    const uint64_t pol = acc_policy(R);
#pragma unroll
    for (int j = 0; j < K / 32; ++j) {
        red_u64_ef(ac + 32 * j, fix40(d[j].x), pol);
        red_u64_ef(ac + 32 * j + 1, fix40(d[j].y), pol);
        red_u64_ef(ac + 32 * j + 2, fix40(d[j].z), pol);
        red_u64_ef(ac + 32 * j + 3, fix40(d[j].w), pol);
    }
}

// apply of step t finished on this rank (exactly one warp gets here per
// step): statistics, then the released count
__device__ __forceinline__ void persist_finish(const PersistRank &R, long long t, long long c,
                                               int lane) {
    // statistics: the item rows each rank's pairs of the step wrote
    if (lane == R.rank) c = (long long)ld_acquire_gpu(R.state + kWritten * R.nsteps + t);
    if (lane < R.world) R.step_counts[t * R.world + lane] = c;
    __threadfence_system();
    __syncwarp();
    if (lane < R.world) st_release_sys(R.rel_tab[lane] + R.rank, R.gbase + (unsigned long long)t + 1);
}

// claims up to C of a phase's units
__device__ __forceinline__ long long persist_claim(const PersistRank &R, unsigned long long *ctr,
                                                   long long C, long long total, int lane) {
    long long i0 = 0;
    if (lane == 0) i0 = (long long)atomicAdd(ctr, (unsigned long long)C);
    return __shfl_sync(kFull, i0, 0);
}

// One unit of apply work for the lowest unapplied step, if any is available:
// 1 = did work, 0 = nothing claimable now, 2 = every step of the epoch applied.
// A unit is up to kApplyChunk entries or rows, 4 at a time per warp (8 lanes
// each, the kernel's row layout) with every load of a chunk in flight at once.
template <int K>
__device__ __forceinline__ int persist_help(const PersistRank &R, int lane) {
    constexpr int V = K / 32;
    constexpr long long C = kApplyChunk;
    const int g = lane >> 3, c = lane & 7;
    const long long n = R.nsteps;
    if (lane == 0) s_pw[8] += 1;
    const long long t = (long long)ld_acquire_sys(R.rel + R.rank) - (long long)R.gbase;
    if (t >= n) return 2;
    const int b = persist_buf(R, t);
    unsigned long long *st = R.state + t;
    // 1. ready once this rank's pairs of step t are done and every peer's log
    //    of step t is complete
    if ((long long)ld_acquire_gpu(st + kDone * n) < R.bounds[t + 1] - R.bounds[t]) return 0;
    long long cnt = 0;   // lane q < world, q != rank: rank q's logged entries of step t
    long long wrote = 0;  // ... and the rows its pairs wrote (statistics)
    bool ok = true;
    if (lane < R.world && lane != R.rank) {
        const unsigned long long v =
            ld_acquire_sys(R.mbox + ((long long)(R.tag & 1) * R.mbox_steps + t) * R.world + lane);
        ok = (unsigned)(v >> 48) == (R.tag & 0xffffu);
        cnt = (long long)(v & 0xffffffull);
        wrote = (long long)((v >> 24) & 0xffffffull);
    }
    if (!__all_sync(kFull, ok)) return 0;  // some peer's log of step t is not complete yet
    // 2. the peers' logged entries of step t for the rows this rank owns
    //    into the buffer (its own pairs added theirs directly)
    if (R.world > 1) {
        const long long cc = cnt < R.cap ? cnt : R.cap;
        long long incl = cc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        const long long E = __shfl_sync(kFull, incl, 31);
        const long long pre = incl - cc;
        if ((long long)ld_acquire_gpu(st + kAccDone * n) < E) {
            const long long i0 = persist_claim(R, st + kAccClaim * n, C, E, lane);
            if (i0 >= E) return 0;
            const long long ca = clock64();
            const int m = (int)(i0 + C < E ? C : E - i0);
            const int slot = persist_slot(R, t);
            // lane j < m: entry i0 + j of the union: rank q = the last rank
            // whose prefix is <= it, then its id and row address
            const long long x = i0 + lane;
            int q = 0;
            for (int r = 1; r < R.world; ++r)
                if (__shfl_sync(kFull, pre, r) <= x) q = r;
            const long long e = x - __shfl_sync(kFull, pre, q);
            int32_t id = 0;
            const float *row = nullptr;
            if (lane < m) {
                id = __ldcg(R.pids[slot][q] + e);
                row = R.prows[slot][q] + e * K;
            }
            for (int p0 = 0; p0 < m; p0 += 8) {  // 2 x 4 entries in flight
                float4 d[2][V];
                int32_t ids[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = p0 + 4 * h + g;
                    ids[h] = __shfl_sync(kFull, id, j & 31);
                    const float *rp = shfl_ptr(row, j & 31);
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        d[h][v] = j < m ? __ldcg(reinterpret_cast<const float4 *>(rp + 32 * v + 4 * c))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    persist_accumulate<K>(R, b, t, ids[h], c,
                                          p0 + 4 * h + g < m && ids[h] % R.world == R.rank, d[h]);
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) {
                atomicAdd(st + kAccDone * n, (unsigned long long)m);
                s_pw[10] += clock64() - ca;
                s_pw[12] += 1;
            }
            return 1;
        }
    }
    // 3. every touched row converted once
    const long long rows = (long long)ld_acquire_gpu(st + kRows * n);
    if ((long long)ld_acquire_gpu(st + kCvtDone * n) < rows) {
        constexpr long long CR = 16;  // rows per claim: 2 x (two groups of 4, loads in flight)
        const long long i0 = persist_claim(R, st + kCvtClaim * n, CR, rows, lane);
        if (i0 >= rows) return 0;
        const long long cv = clock64();
        const int m = (int)(i0 + CR < rows ? CR : rows - i0);
        // rows i0 .. i0 + m - 1 of the step's list
        int32_t myid = 0;
        if (lane < m) myid = __ldcg(R.touched[b] + i0 + lane);
        const uint64_t pef = acc_policy(R);
        for (int hb = 0; hb < m; hb += 8) {
        longlong2 q01[2][V], q23[2][V];
        float4 tv[2][V];
        int32_t ids[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = hb + 4 * h + g;
            ids[h] = __shfl_sync(kFull, myid, j & 31);
            if (j < m) {
                const long long *ac = R.acc[b] + (i0 + j) * K + 4 * c;
                const float *tr = R.T + (int64_t)ids[h] * K + 4 * c;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    q01[h][v] = ld_acc2(ac + 32 * v, pef);
                    q23[h][v] = ld_acc2(ac + 32 * v + 2, pef);
                    tv[h][v] = __ldcg(reinterpret_cast<const float4 *>(tr + 32 * v));
                }
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int j = hb + 4 * h + g;
            if (j < m) {
                long long *ac = R.acc[b] + (i0 + j) * K + 4 * c;
                float *tr = R.T + (int64_t)ids[h] * K + 4 * c;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    zero_acc2(ac + 32 * v, pef);
                    zero_acc2(ac + 32 * v + 2, pef);
                    float4 x = tv[h][v];
                    x.x += (float)((double)q01[h][v].x * (1.0 / kFix));
                    x.y += (float)((double)q01[h][v].y * (1.0 / kFix));
                    x.z += (float)((double)q23[h][v].x * (1.0 / kFix));
                    x.w += (float)((double)q23[h][v].y * (1.0 / kFix));
                    __stcg(reinterpret_cast<float4 *>(tr + 32 * v), x);
                    // the owner's new row into every peer's replica (NVLink)
                    for (int p = 0; p < R.world; ++p)
                        if (p != R.rank)
                            *reinterpret_cast<float4 *>(R.t_tab[p] + (int64_t)ids[h] * K + 4 * c + 32 * v) = x;
                }
                if (c == 0) R.map[b][ids[h]] = 0;
            }
        }
        }
        if (R.world > 1) __threadfence_system();  // the peers' replicas too
        __threadfence();
        __syncwarp();
        long long d = 0;
        if (lane == 0) {
            d = (long long)atomicAdd(st + kCvtDone * n, (unsigned long long)m) + m;
            s_pw[11] += clock64() - cv;
        }
        if (__shfl_sync(kFull, d, 0) == rows) persist_finish(R, t, wrote, lane);
        return 1;
    }
    if (rows == 0) {  // nothing touched: one warp finishes the step
        int win = 0;
        if (lane == 0) win = atomicCAS(st + kFin * n, 0ull, 1ull) == 0ull;
        if (__shfl_sync(kFull, win, 0)) {
            persist_finish(R, t, wrote, lane);
            return 1;
        }
    }
    return 0;  // the step's last chunks are in other warps' hands
}


// ---- the persistent kernel's per-warp bookkeeping ---------------------------
// What MODE 2/3 adds to a pair is a few loads and atomics at its start and
// end; the state it carries between them lives in shared memory, so the
// pair's streaming loop compiles as in the single-GPU kernel (it needs every
// register of the 12-warps-per-SM budget).  s_pw: [0] the highest global step
// whose gate this warp saw open, [1] start clock, clocks in [2] gate waits,
// [3] apply work after pairs (diagnostics), [5] apply units done, [6] the step
// of the last claimed pair (claims only grow), [7] the current pair's step.

__device__ __forceinline__ const PersistRank &persist_rank(const PersistRank *ctx, int nctx) {
    return ctx[nctx > 1 ? (int)(blockIdx.x % (unsigned)nctx) : 0];
}

__device__ __forceinline__ void persist_init(const PersistRank *ctx, int nctx, int lane) {
    const PersistRank &R = persist_rank(ctx, nctx);
    if (lane == 0) {
        s_pw[0] = -1;
        s_pw[1] = clock64();
        for (int i = 2; i < 16; ++i) s_pw[i] = 0;
        s_pw[13] = -1;  // start clock of a gate wait (-1: not waiting)
    }
    __syncwarp();
    // steps without local pairs have a complete (empty) log from the start
    for (int64_t s = blockIdx.x / nctx; s < R.nsteps; s += R.nblocks)
        if (R.bounds[s + 1] == R.bounds[s]) persist_publish(R, s, lane);
}

// MODE: 0 = host pair range, 1 = device range (captured step graphs),
// 2 = persistent sharded epoch of one rank (tables and pairs in `a`, the
// rank's exchange state in ctx[0]), 3 = persistent epoch of a loopback group
// (ctx: the ranks; block b serves rank b % nctx)
// PAIR2 (default): two rounds share one transposed butterfly (8 quantities
// over the row's 8 lanes: 8 shuffles instead of 10, and half the dependent
// shuffle depth per round — the per-round chain bounds this kernel; c4
// 33.5-33.8 M vs 31.9 M samples/s one round at a time)
// PH: phase profile (trainer.py:120-331 collect_phases): clocks of the
// pair's phases into a.phase.  The phases are fused here, so the marks split
// them by where the time goes: read_emb = the user row, the pair's ids and
// the first rounds' loads; similarity = the streaming rounds (the negative
// rows' reads and their dots, one pass); loss = the resolve (recorded rows
// re-read, binary64 decisions, hinge); gradient = row coefficients, item
// deltas and the user gradient; update = the row writes.
template <int K, int MINB, int MODE, bool PAIR2 = true, bool PH = false>
__global__ void __launch_bounds__(32, MINB)
    hogwild_stream(HogwildArgs a, FastMod fm, int snap_cap, float band_lo,
                   unsigned long long *claim, const PersistRank *__restrict__ ctx, int nctx,
                   int apply_warps, unsigned long long *prof) {
    constexpr bool DR = MODE == 1;
    constexpr bool PS = MODE >= 2;
    constexpr int V = K / 32;  // float4 per lane per row
    extern __shared__ __align__(16) unsigned char sm[];
    float *urow = reinterpret_cast<float *>(sm);  // K floats: the user row
    float *snap = urow + K;                       // snap_cap rows: the first written rows

    const int lane = threadIdx.x;
    const int g = lane >> 3;  // row slot of a group
    const int c = lane & 7;   // column chunk: columns 32j + 4c .. +3
    if constexpr (PH) {
        if (lane == 0) {
            for (int i = 0; i < 6; ++i) s_ph[i] = 0;
            s_ph[7] = clock64();
            s_ph[8] = globaltimer_ns();
        }
    }
    auto mark = [&](int i) {  // phase i ends here
        if constexpr (PH) {
            __syncwarp();
            if (lane == 0) {
                const long long t = clock64();
                s_ph[i] += t - s_ph[6];
                s_ph[6] = t;
            }
        }
    };
    int64_t k_start = a.start, k_stop = a.stop;
    uint64_t k_s0 = a.s0;
    if constexpr (DR) {
        k_start = a.range_dev[0];
        k_stop = a.range_dev[1];
        k_s0 = *a.s0_dev;
    }
    // the rank's tables, pairs and sink (PS: from its context)
    float *S = a.S, *T = a.T;
    const int32_t *users = a.users, *items = a.items;
    const int64_t *pidx = a.pair_index;
    heat_counters *ctr = a.ctr;
    // the context pointer is laundered through an asm move at every use, so
    // nothing derived from it (state words, buffer addresses) is hoisted out
    // of the worker loop and kept live across the streaming loop
    auto prank = [&]() -> const PersistRank & {
        const PersistRank *p = ctx + (MODE == 3 ? (int)(blockIdx.x % (unsigned)nctx) : 0);
        asm volatile("mov.b64 %0, %0;" : "+l"(p));
        return *p;
    };
    if constexpr (PS) {
        if constexpr (MODE == 3) {  // (MODE 2: the launcher put them in `a`)
            const PersistRank &R = persist_rank(ctx, nctx);
            S = R.S; T = R.T; users = R.users; items = R.items;
            pidx = R.pidx; ctr = R.ctr; claim = R.claim;
            k_start = 0;
            k_stop = R.bounds[R.nsteps];
        }
        persist_init(ctx, nctx, lane);
    }
    const int64_t npairs = k_stop - k_start;
    const int N = a.N;
    const int niter = (N + 1 + 31) >> 5;  // 4 rounds of 8 rows per iteration
    // (a launch parameter, not createpolicy's vector-register result: the
    // loads take it from a uniform register without a move per load)
    const uint64_t pol = a.l2_policy;
    // per-worker global area: written-row entries, rows past the snapshot
    unsigned char *mine_area = a.spill + (size_t)blockIdx.x * a.spill_stride;
    float *sp_rows = reinterpret_cast<float *>(mine_area);
    WriteEntry *ents = reinterpret_cast<WriteEntry *>(mine_area + (size_t)a.spill_cap * K * 4);
    // (id, flags) of each recorded row, written while streaming (one 8-byte
    // store); the full entries are filled by the resolve
    int2 *recs = reinterpret_cast<int2 *>(ents + a.spill_cap);
    auto slot_row = [&](int e) -> float * {
        return e < snap_cap ? snap + (size_t)e * K : sp_rows + (size_t)(e - snap_cap) * K;
    };

    double loss = 0.0;
    int degen = 0, active = 0, npairs_mine = 0;

    auto claim_next = [&]() -> int64_t {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(claim, 1ull);
        return (int64_t)__shfl_sync(kFull, t, 0);
    };

    // the next pair is claimed and its (user, item, RNG key) fetched one pair
    // ahead, so a pair starts without a chain of dependent global reads
    // (atomic -> ids -> rows).  Only read-only inputs are prefetched: table
    // rows are read when the pair starts.
    struct Next { int64_t t; int32_t u, pos; uint64_t pg; };
    auto fetch = [&](int64_t tt) -> Next {
        Next n{tt, 0, 0, 0};
        if (tt < npairs) {
            const int64_t pp = k_start + tt;
            n.u = users[pp];
            n.pos = items[pp];
            n.pg = pidx ? (uint64_t)pidx[pp] : (uint64_t)pp;
            if constexpr (PS) {  // the claimed pair's step (claims only grow)
                long long sc = s_pw[6];
                while (prank().bounds[sc + 1] <= tt) ++sc;
                __syncwarp();
                if (lane == 0) s_pw[6] = sc;
                __syncwarp();
            }
        }
        return n;
    };
    // PS: the rank's first `apply_warps` workers only apply (no pairs): they
    // start a step's apply the moment it becomes claimable
    const bool applier = PS && (int)(blockIdx.x / nctx) < apply_warps;
    Next nx = applier ? Next{npairs, 0, 0, 0} : fetch(claim_next());

    // PS: what the warp does next, so that every kind of apply work goes
    // through ONE inlined persist_help (a call to a user function would put
    // the whole kernel under the calling ABI and spill the streaming loop):
    // 0 = start pair nx, 1 = apply work after a pair, 2 = nx's gate is
    // closed, 3 = no pairs left
    // (hs = s_pw[14] and the waiting warps' backoff ns = s_pw[15] live in
    // shared memory: the streaming loop has no register to spare)
    if (lane == 0) {
        s_pw[14] = 0;
        s_pw[15] = 64;
    }
    __syncwarp();
    for (;;) {
        if constexpr (PS) {
            const PersistRank &R = prank();
            int hs = (int)s_pw[14];
            __syncwarp();
            if (hs == 0) {
                if (nx.t >= npairs) {
                    hs = 3;
                    if (lane == 0) s_pw[4] = clock64();
                } else {
                    const long long g = (long long)(R.gbase + (unsigned long long)s_pw[6]);
                    if (g > s_pw[0]) {  // (a gate open for g is open for every earlier step)
                        const bool open = persist_gate_open(R, g, lane);
                        __syncwarp();
                        if (lane == 0) {
                            if (open) {
                                s_pw[0] = g;
                                if (s_pw[13] >= 0) s_pw[2] += clock64() - s_pw[13];
                                s_pw[13] = -1;
                            } else if (s_pw[13] < 0) {
                                s_pw[13] = clock64();
                            }
                        }
                        if (!open) hs = 2;
                        __syncwarp();
                    }
                }
            }
            if (hs != 0) {
                const long long c0 = clock64();
                const int r = persist_help<K>(R, lane);
                if (hs == 1) {
                    if (r != 1) hs = 0;
                    if (lane == 0) s_pw[3] += clock64() - c0;
                } else if (hs == 2) {
                    const unsigned ns = (unsigned)s_pw[15];
                    if (r != 1) __nanosleep(ns);
                    __syncwarp();
                    if (lane == 0) s_pw[15] = r != 1 ? (ns < 2048 ? 2 * ns : ns) : 64;
                    hs = 0;  // look at the gate again
                    if (s_pw[13] >= 0) watchdog(s_pw[13], 2, R, s_pw[6]);
                } else {
                    if (r == 2) break;
                    if (r == 0) __nanosleep(500);
                    watchdog(s_pw[4], 3, R, (long long)R.rel[R.rank] - (long long)R.gbase);
                }
                if (lane == 0) {
                    if (r == 1) ++s_pw[5];
                    s_pw[14] = hs;
                }
                __syncwarp();
                continue;
            }
            if (lane == 0) s_pw[14] = hs;
            if (lane == 0) s_pw[7] = s_pw[6];  // the pair starts: its step
            __syncwarp();
        } else {
            if (nx.t >= npairs) break;
        }
        const int32_t u = nx.u;
        const int32_t pos = nx.pos;
        const uint64_t pg = nx.pg;
        if constexpr (PH) {
            if (lane == 0) s_ph[6] = clock64();
        }

        float4 uv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) uv[j] = ldcg4(S + (int64_t)u * K + 32 * j + 4 * c);

        // negative ids, 32 rows per draw block: lane l of block b holds the id
        // of row 32b + l; row r >= 1 is draw pg*N + r - 1 of the stream
        // (trainer.py:134-139): mix64(s0 + (pg*N + r) * GAMMA) mod rows.
        // Rows past N read row 0 (a harmless load) and are never recorded.
        uint64_t rstate = k_s0 + (pg * (uint64_t)N + (uint64_t)lane) * kGamma;
        auto draw = [&](int blk) -> int32_t {
            const int r = 32 * blk + lane;
            const int32_t id = (int32_t)fm.mod(mix64(rstate));
            return r == 0 ? pos : (r <= N ? id : 0);
        };
        int32_t idv = draw(0);

        // register ring: round rd (rows 8rd .. 8rd+7, two groups of 4) lives
        // in buffer rd & 1 and is loaded two rounds ahead
        float4 R[2][2][V];
        int32_t rid[2][2];
        // the row ids of round rd (rd & 3 selects them in idv) and the loads
        // of a round into buffer b, split so the id shuffles run ahead of the
        // arithmetic that frees the buffer
        auto round_ids = [&](int rd, int32_t (&ids)[2]) {
#pragma unroll
            for (int x = 0; x < 2; ++x)
                ids[x] = __shfl_sync(kFull, idv, ((rd & 3) << 3) + 4 * x + g);
        };
        auto load = [&](int b, const int32_t (&ids)[2], int32_t z) {
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                rid[b][x] = ids[x];
                const float *src = T + (int64_t)ids[x] * K + 4 * c + z;
#pragma unroll
                for (int j = 0; j < V; ++j) R[b][x][j] = ld_row4(src + 32 * j, pol);
            }
        };
        {
            int32_t ids[2];
            round_ids(0, ids);
            load(0, ids, 0);
            round_ids(1, ids);
            load(1, ids, 0);
        }
        nx = fetch(claim_next());

        // fp32 u.u for the screen; the exact binary64 ss (trainer.py:176-178)
        // is summed at the end of the pair, where the written rows are resolved
        float ssf;
        {
            float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                q0 = __ffma2_rn(make_float2(uv[j].x, uv[j].y), make_float2(uv[j].x, uv[j].y), q0);
                q1 = __ffma2_rn(make_float2(uv[j].z, uv[j].w), make_float2(uv[j].z, uv[j].w), q1);
            }
            ssf = (q0.x + q0.y) + (q1.x + q1.y);
            ssf += __shfl_xor_sync(kFull, ssf, 4);
            ssf += __shfl_xor_sync(kFull, ssf, 2);
            ssf += __shfl_xor_sync(kFull, ssf, 1);
        }
        // a query whose fp32 u.u is tiny or zero sends every row to the
        // binary64 resolve (the degenerate test of trainer.py:184, 203)
        const bool screen = ssf > 1e-30f;
        const float rss = screen ? rsqrt_approx(ssf) : 0.f;
        if (g == 0) {  // the user row: the rounds' u.v and the binary64 sums
#pragma unroll
            for (int j = 0; j < V; ++j) *reinterpret_cast<float4 *>(urow + 32 * j + 4 * c) = uv[j];
        }
        __syncwarp();
        // exact ss = u.u as trainer.py:176-178 sums it, while the first rows load
        const double ss = seq_dot<K>(urow, urow);
        const bool decay_all = a.l2 != 0.f;
        int cnt = 0;  // rows recorded for writing (same value in every lane)
        int32_t nidsA0 = 0, nidsA1 = 0, nidsB0 = 0, nidsB1 = 0;  // (PAIR2)
        mark(0);

        // one round: FFMA2 partials of its 8 rows, the buffer refilled two
        // rounds ahead as soon as they are consumed, then the reduction and
        // the fp32 screen.  Rows that may be written are only RECORDED here
        // (id + flags); the resolve below re-reads them, so no row data is
        // held past its FFMA2s.
        auto round = [&](int b, int rd, bool refill) {
            int32_t nids[2];
            if (refill) round_ids(rd + 2, nids);
            float2 tl[2], th[2], sl[2], sh[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) tl[x] = th[x] = sl[x] = sh[x] = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                // this lane's user columns, from shared memory (not held in
                // registers across the round: the ring needs them)
                const float4 w = *reinterpret_cast<const float4 *>(urow + 32 * j + 4 * c);
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const float2 vlo = make_float2(R[b][x][j].x, R[b][x][j].y);
                    const float2 vhi = make_float2(R[b][x][j].z, R[b][x][j].w);
                    tl[x] = __ffma2_rn(vlo, vlo, tl[x]);
                    th[x] = __ffma2_rn(vhi, vhi, th[x]);
                    sl[x] = __ffma2_rn(make_float2(w.x, w.y), vlo, sl[x]);
                    sh[x] = __ffma2_rn(make_float2(w.z, w.w), vhi, sh[x]);
                }
            }
            const int32_t id0 = rid[b][0], id1 = rid[b][1];
            // refill only after every FFMA2 of the round consumed the buffer
            if (refill) load(b, nids, opaque_zero(th[1].x) + opaque_zero(sh[1].y));
            float q[4];  // tt(x=0), st(x=0), tt(x=1), st(x=1)
#pragma unroll
            for (int x = 0; x < 2; ++x) {
                const float2 t2 = __fadd2_rn(tl[x], th[x]);
                const float2 s2 = __fadd2_rn(sl[x], sh[x]);
                q[2 * x] = t2.x + t2.y;
                q[2 * x + 1] = s2.x + s2.y;
            }
            // transposed butterfly over the row's 8 lanes: afterwards lane c
            // holds quantity (c >> 1) & 1 (tt, st) of group c >> 2
            const bool b2 = (c & 4) != 0, b1 = (c & 2) != 0;
            float k0 = b2 ? q[2] : q[0], k1 = b2 ? q[3] : q[1];
            const float s0 = b2 ? q[0] : q[2], s1 = b2 ? q[1] : q[3];
            k0 += __shfl_xor_sync(kFull, s0, 4);
            k1 += __shfl_xor_sync(kFull, s1, 4);
            float m = b1 ? k1 : k0;
            m += __shfl_xor_sync(kFull, b1 ? k0 : k1, 2);
            m += __shfl_xor_sync(kFull, m, 1);
            const float o = __shfl_xor_sync(kFull, m, 2);
            const float ttf = b1 ? o : m, stf = b1 ? m : o;
            // fp32 screen (lanes 0-3 decide for group 0, lanes 4-7 for group
            // 1).  Band rows — the positive, any row whose fp32 cosine is
            // within 1e-5 of theta or above (fp32 error < 1e-6 at K <= 128),
            // any row whose fp32 v.v underflows — are decided by the resolve
            // from binary64 sums; every other row cannot be active, so it is
            // written only as a decay row (l2 != 0).
            const int r = 8 * rd + (b2 ? 4 : 0) + g;
            const float sim32 = stf * rss * rsqrt_approx(ttf);
            const bool valid = r <= N;
            const bool band = valid & (!screen | (r == 0) | !(ttf > 1e-30f) | (sim32 > band_lo));
            const bool rec = band | (valid & decay_all);
            const unsigned mrec = __ballot_sync(kFull, rec & ((c & 3) == 0));
            if (rec & ((c & 3) == 0)) {
                const int idx = cnt + __popc(mrec & ((1u << lane) - 1u));
                recs[idx] = make_int2(b2 ? id1 : id0, band ? (r == 0 ? 3 : 1) : 0);
            }
            cnt += __popc(mrec);
        };

        // PAIR2: rounds rd (buffer 0) and rd + 1 (buffer 1) reduced together
        auto round2 = [&](int rd, bool refill) {
            float q[8];  // q[4 rb + 2 x + t]: t 0 = tt, 1 = st; rb 0 = round rd, 1 = rd + 1
#pragma unroll
            for (int rb = 0; rb < 2; ++rb) {
                int32_t nids[2];
                if (refill) round_ids(rd + rb + 2, nids);
                float2 tl[2], th[2], sl[2], sh[2];
#pragma unroll
                for (int x = 0; x < 2; ++x) tl[x] = th[x] = sl[x] = sh[x] = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const float4 w = *reinterpret_cast<const float4 *>(urow + 32 * j + 4 * c);
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        const float2 vlo = make_float2(R[rb][x][j].x, R[rb][x][j].y);
                        const float2 vhi = make_float2(R[rb][x][j].z, R[rb][x][j].w);
                        tl[x] = __ffma2_rn(vlo, vlo, tl[x]);
                        th[x] = __ffma2_rn(vhi, vhi, th[x]);
                        sl[x] = __ffma2_rn(make_float2(w.x, w.y), vlo, sl[x]);
                        sh[x] = __ffma2_rn(make_float2(w.z, w.w), vhi, sh[x]);
                    }
                }
                // the ids leave with the buffer: keep them for the recording
                if (rb == 0) {
                    nidsA0 = rid[0][0];
                    nidsA1 = rid[0][1];
                } else {
                    nidsB0 = rid[1][0];
                    nidsB1 = rid[1][1];
                }
                if (refill) load(rb, nids, opaque_zero(th[1].x) + opaque_zero(sh[1].y));
#pragma unroll
                for (int x = 0; x < 2; ++x) {
                    const float2 t2 = __fadd2_rn(tl[x], th[x]);
                    const float2 s2 = __fadd2_rn(sl[x], sh[x]);
                    q[4 * rb + 2 * x] = t2.x + t2.y;
                    q[4 * rb + 2 * x + 1] = s2.x + s2.y;
                }
            }
            // transposed butterfly: afterwards lane c holds quantity c
            const bool b2 = (c & 4) != 0, b1 = (c & 2) != 0, b0 = (c & 1) != 0;
            float k[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                k[i] = (b2 ? q[4 + i] : q[i]) + __shfl_xor_sync(kFull, b2 ? q[i] : q[4 + i], 4);
            float h0 = (b1 ? k[2] : k[0]) + __shfl_xor_sync(kFull, b1 ? k[0] : k[2], 2);
            float h1 = (b1 ? k[3] : k[1]) + __shfl_xor_sync(kFull, b1 ? k[1] : k[3], 2);
            const float mq = (b0 ? h1 : h0) + __shfl_xor_sync(kFull, b0 ? h0 : h1, 1);
            const float o = __shfl_xor_sync(kFull, mq, 1);
            const float ttf = b0 ? o : mq, stf = b0 ? mq : o;
            // lanes with even c screen row (round rd + (c >> 2), group (c >> 1) & 1, slot g)
            const int rb = b2 ? 1 : 0, x = b1 ? 1 : 0;
            const int r = 8 * (rd + rb) + 4 * x + g;
            const float sim32 = stf * rss * rsqrt_approx(ttf);
            const bool valid = r <= N;
            const bool band = valid & (!screen | (r == 0) | !(ttf > 1e-30f) | (sim32 > band_lo));
            const bool rec = band | (valid & decay_all);
            const bool me = rec & !b0;
            const unsigned mrec = __ballot_sync(kFull, me);
            if (me) {
                const int32_t id = rb ? (x ? nidsB1 : nidsB0) : (x ? nidsA1 : nidsA0);
                const int idx = cnt + __popc(mrec & ((1u << lane) - 1u));
                recs[idx] = make_int2(id, band ? (r == 0 ? 3 : 1) : 0);
            }
            cnt += __popc(mrec);
        };

#pragma unroll 1
        for (int it = 0; it < niter; ++it) {
            const int rd = 4 * it;
            const bool more = it + 1 < niter;
            if constexpr (PAIR2) {
                round2(rd, true);
                rstate += 32ull * kGamma;
                idv = draw(it + 1);
                round2(rd + 2, more);
            } else {
                round(0, rd, true);
                round(1, rd + 1, true);
                rstate += 32ull * kGamma;  // rounds rd+4, rd+5 need the next block
                idv = draw(it + 1);
                round(0, rd + 2, more);
                round(1, rd + 3, more);
            }
        }
        mark(1);

        // resolve: re-read every recorded row into its snapshot slot (shared
        // memory, then the worker's spill rows; four rows per pass, one per
        // row slot g), then decide each band row from binary64 v.v and u.v
        // (warp-cooperative, heat_row_update.cuh) with the reference's
        // cosine, degenerate test, hinge and weight (trainer.py:184-227).  A
        // band row that is not written becomes a hole (id -1).  Every read
        // of the pair precedes every write.
        __syncwarp();
        const float irs = ss > 0.0 ? rsqrtf((float)ss) : 0.f;
        const double wneg = a.mu * (1.0 / (double)N);
        double hinge = 0.0, sim_p = 0.0;
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 4) {
            const int e = e0 + g;
            if (e < cnt) {
                float *dst = slot_row(e) + 4 * c;
                const float *src = T + (int64_t)recs[e].x * K + 4 * c;
#pragma unroll
                for (int j = 0; j < V; ++j)
                    *reinterpret_cast<float4 *>(dst + 32 * j) = ldcg4(src + 32 * j);
            }
        }
        __syncwarp();
#pragma unroll 1
        for (int e = 0; e < cnt; ++e) {
            const int2 rec = recs[e];
            if (!(rec.y & 1)) {  // a decay-only row: w = 0
                if (lane == 0) ents[e] = WriteEntry{0.0, 0.0, 0.0, rec.x, 0};
                continue;
            }
            double unused, tt, st;
            warp_dots64<K>(urow, slot_row(e), ContiguousCols{}, false, unused, tt, st);
            if (lane == 0) {
                const bool degenerate = ss <= 0.0 || tt <= 0.0;
                const double sim = degenerate ? 0.0 : st / (sqrt(ss) * sqrt(tt));
                if (degenerate) ++degen;
                double w = 0.0;
                bool write;
                if (rec.y & 2) {  // the positive
                    sim_p = sim;
                    w = -1.0;
                    write = !degenerate || a.l2 != 0.f;
                } else {
                    if (sim - a.theta > 0.0) {
                        hinge += sim - a.theta;
                        w = wneg;
                        if (w != 0.0) ++active;
                    }
                    write = (w != 0.0 && !degenerate) || (w == 0.0 && a.l2 != 0.f);
                }
                ents[e] = WriteEntry{tt, st, w, write ? rec.x : -1, 0};
            }
        }
        __syncwarp();
        mark(2);

        float4 ug[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            ug[j] = make_float4(0.f, 0.f, 0.f, 0.f);
            uv[j] = *reinterpret_cast<const float4 *>(urow + 32 * j + 4 * c);
        }
        // the writes, four rows at a time (trainer.py:236-251 user gradient,
        // 259-290 item update, cached scalars; fp32 coefficients)
        const bool dmode = PS || a.delta_ids != nullptr;
#pragma unroll 1
        for (int e0 = 0; e0 < cnt; e0 += 4) {
            const int e = e0 + g;
            WriteEntry ent{};
            if (e < cnt) ent = ents[e];
            const bool ok = e < cnt && ent.id >= 0;
            float4 d[V];
            if (ok) {
                const RowCoef co = row_coef_f(ent, ss, irs, a.lr, a.l2, true);
                const float *row = slot_row(e);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const float4 v = *reinterpret_cast<const float4 *>(row + 32 * j + 4 * c);
                    row_apply(co, uv[j].x, v.x, d[j].x, ug[j].x);
                    row_apply(co, uv[j].y, v.y, d[j].y, ug[j].y);
                    row_apply(co, uv[j].z, v.z, d[j].z, ug[j].z);
                    row_apply(co, uv[j].w, v.w, d[j].w, ug[j].w);
                }
            }
            mark(3);
            if (!dmode) {
                if (ok) {
                    float *dst = T + (int64_t)ent.id * K + 4 * c;
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        red_add4(dst + 32 * j, d[j].x, d[j].y, d[j].z, d[j].w);
                }
            } else {  // logged (PS: into the step's log slot)
                int32_t *lids = a.delta_ids;
                float *lrows = a.delta_rows;
                unsigned long long *lcnt = reinterpret_cast<unsigned long long *>(a.delta_count);
                int64_t lcap = a.delta_capacity;
                bool log = true;
                bool mine = true;
                if constexpr (PS) {  // owned rows into the step's buffer; the others logged
                    const PersistRank &R = prank();
                    const long long stp = s_pw[7];
                    mine = ent.id % R.world == R.rank;
                    persist_accumulate<K>(R, persist_buf(R, stp), stp, ent.id, c, ok && mine, d);
                    if (ok && c == 0) atomicAdd(R.state + kWritten * R.nsteps + stp, 1ull);
                    const int slt = persist_slot(R, stp);
                    lids = R.log_ids[slt];
                    lrows = R.log_rows[slt];
                    lcnt = R.cnt + stp;
                    lcap = R.cap;
                    log = !mine;
                }
                long long sl = 0;
                if (ok && log && c == 0) sl = (long long)atomicAdd(lcnt, 1ull);
                sl = __shfl_sync(kFull, sl, g * 8);
                if (log && ok && sl < lcap) {
                    if (c == 0) lids[sl] = ent.id;
                    float *dst = lrows + sl * K + 4 * c;
#pragma unroll
                    for (int j = 0; j < V; ++j) *reinterpret_cast<float4 *>(dst + 32 * j) = d[j];
                }
            }
            mark(4);
        }
        // user row (trainer.py:291-293): S[u] -= lr * (ugrad + l2 * S[u]),
        // the four row slots' partial gradients summed first
#pragma unroll
        for (int j = 0; j < V; ++j) {
#pragma unroll
            for (int o = 8; o <= 16; o <<= 1) {
                ug[j].x += __shfl_xor_sync(kFull, ug[j].x, o);
                ug[j].y += __shfl_xor_sync(kFull, ug[j].y, o);
                ug[j].z += __shfl_xor_sync(kFull, ug[j].z, o);
                ug[j].w += __shfl_xor_sync(kFull, ug[j].w, o);
            }
        }
        mark(3);
        if (g == 0) {
#pragma unroll
            for (int j = 0; j < V; ++j)
                red_add4(S + (int64_t)u * K + 32 * j + 4 * c, -a.lr * (ug[j].x + a.l2 * uv[j].x),
                         -a.lr * (ug[j].y + a.l2 * uv[j].y), -a.lr * (ug[j].z + a.l2 * uv[j].z),
                         -a.lr * (ug[j].w + a.l2 * uv[j].w));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            hinge += __shfl_xor_sync(kFull, hinge, o);
            sim_p += __shfl_xor_sync(kFull, sim_p, o);  // one lane holds it
        }
        if (lane == 0) loss += (1.0 - sim_p) + wneg * hinge;
        ++npairs_mine;
        __syncwarp();
        mark(4);
        if constexpr (PS) {
            // the pair's log entries are written: count it into its step; the
            // step's last pair publishes the log; then apply work is helped
            const PersistRank &R = prank();
            __threadfence();
            __syncwarp();
            const long long step = s_pw[7];
            int last = 0;
            if (lane == 0)
                last = atomicAdd(R.state + kDone * R.nsteps + step, 1ull) + 1 ==
                       (unsigned long long)(R.bounds[step + 1] - R.bounds[step]);
            if (__shfl_sync(kFull, last, 0)) persist_publish(R, step, lane);
            if (lane == 0) s_pw[14] = 1;  // then apply work, while there is some
            __syncwarp();
        }
    }
    if constexpr (PS) {
        if (prof && lane == 0) {
            atomicAdd(prof + 0, (unsigned long long)(clock64() - s_pw[1]));
            atomicAdd(prof + 1, (unsigned long long)s_pw[2]);
            atomicAdd(prof + 2, (unsigned long long)s_pw[3]);
            atomicAdd(prof + 3, (unsigned long long)(clock64() - s_pw[4]));
            atomicAdd(prof + 4, (unsigned long long)s_pw[5]);
            atomicAdd(prof + 5, (unsigned long long)npairs_mine);
            atomicAdd(prof + 6, 1ull);
            atomicAdd(prof + 7, (unsigned long long)s_pw[8]);
            atomicAdd(prof + 8, (unsigned long long)s_pw[10]);
            atomicAdd(prof + 9, (unsigned long long)s_pw[11]);
            atomicAdd(prof + 10, (unsigned long long)s_pw[12]);
        }
    }
    if constexpr (PH) {
        if (lane == 0 && a.phase) {
            for (int i = 0; i < 6; ++i) atomicAdd(a.phase + i, (unsigned long long)s_ph[i]);
            atomicAdd(a.phase + 6, (unsigned long long)(clock64() - s_ph[7]));
            atomicAdd(a.phase + 7, (unsigned long long)(globaltimer_ns() - s_ph[8]));
            atomicAdd(a.phase + 8, 1ull);
            atomicAdd(a.phase + 9, (unsigned long long)npairs_mine);
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        degen += __shfl_xor_sync(kFull, degen, o);
        active += __shfl_xor_sync(kFull, active, o);
    }
    if (lane == 0) {
        atomicAdd(&ctr->loss, loss);
        if (degen) atomicAdd((unsigned long long *)&ctr->degenerate, (unsigned long long)degen);
        if (active) atomicAdd((unsigned long long *)&ctr->active, (unsigned long long)active);
        atomicAdd((unsigned long long *)&ctr->pairs, (unsigned long long)npairs_mine);
        // re-arm the claim counter once every warp has made its last claim
        __threadfence();
        const unsigned long long nb = PS ? (unsigned long long)persist_rank(ctx, nctx).nblocks : gridDim.x;
        if (atomicAdd(claim + 1, 1ull) == nb - 1) {
            claim[0] = 0;
            claim[1] = 0;
            __threadfence();
        }
    }
}

// the persistent epoch (and the stream-ordered DELTA launches, which keep its
// order) reduce two rounds per butterfly as well: c4 sharded at N = 1 28.9 M
// vs 26.4 M samples/s one round at a time (HEAT_PERSIST_PAIR2=0)
static bool persist_pair2() {
    static const bool on = [] {
        const char *e = getenv("HEAT_PERSIST_PAIR2");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

template <int K, int MINB>
static cudaError_t launch_stream_k(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    const int snap_cap = K <= 64 ? 16 : 8;
    const size_t smem = K * sizeof(float) + (size_t)snap_cap * K * sizeof(float);
    static const bool pair2 = [] {  // HEAT_STREAM_PAIR2=0: one round at a time (A/B)
        const char *e = getenv("HEAT_STREAM_PAIR2");
        return e ? atoi(e) != 0 : true;
    }();
    // DELTA launches (the stream-ordered shard steps) keep the persistent
    // epoch's round order, so the two runtimes record rows, and sum the user
    // gradient, in the same order (bit-identical at one pair in flight)
    const bool p2 = a.delta_ids ? persist_pair2() : pair2;
    auto kern = a.range_dev                   ? hogwild_stream<K, MINB, 1, false>
                : a.phase && !a.delta_ids     ? hogwild_stream<K, MINB, 0, true, true>
                : p2                          ? hogwild_stream<K, MINB, 0, true>
                                              : hogwild_stream<K, MINB, 0, false>;
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32, smem, &e);
    if (e != cudaSuccess) return e;
    int64_t nw = (int64_t)per_sm * sm_count();
    if (a.window > 0) nw = std::min<int64_t>(nw, a.window);
    nw = std::min<int64_t>(nw, a.stop - a.start);
    if (nw < 1) return cudaSuccess;
    if (workers_out) *workers_out = (int)nw;
    HogwildArgs b = a;
    b.l2_policy = stream_row_policy();
    if (!b.l2_policy) return cudaErrorNotSupported;  // (another kernel family takes the launch)
    // spill area: a pair writes at most N+1 rows (all of them when l2 != 0)
    b.spill_cap = a.N + 1;
    b.spill_stride = ((int64_t)b.spill_cap * (K * sizeof(float) + sizeof(WriteEntry) + sizeof(int2)) + 255) &
                     ~(int64_t)255;
    b.spill = static_cast<unsigned char *>(stream_scratch(1, (size_t)(b.spill_stride * nw), st));
    unsigned long long *claim = stream_claim(st);
    if (!b.spill || !claim) return cudaErrorMemoryAllocation;
    kern<<<(unsigned)nw, 32, smem, st>>>(b, FastMod::make((uint64_t)a.num_items), snap_cap,
                                         (float)a.theta - 1e-5f, claim, nullptr, 0, 0, nullptr);
    return cudaGetLastError();
}

// HEAT_PERSIST_PROF=1: a device buffer of clock totals the persistent kernel
// adds into (printed and cleared by persist_prof_report after an epoch)
static unsigned long long *g_prof = nullptr;
static unsigned long long *persist_prof(cudaStream_t st) {
    static const bool on = getenv("HEAT_PERSIST_PROF") && atoi(getenv("HEAT_PERSIST_PROF")) != 0;
    if (!on) return nullptr;
    if (!g_prof && cudaMalloc(&g_prof, 16 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemsetAsync(g_prof, 0, 16 * sizeof(unsigned long long), st);
    return g_prof;
}

// the persistent sharded epoch: every resident one-warp CTA is a worker (the
// steps, not a window, bound the staleness); nctx > 1 splits them over the
// ranks of a loopback group and launches cooperatively
template <int K, int MINB>
static cudaError_t launch_persist_k(const HogwildArgs &a, const PersistRank *ctx_host,
                                    PersistRank *ctx_dev, int nctx, cudaStream_t st) {
    const int snap_cap = K <= 64 ? 16 : 8;
    const size_t smem = K * sizeof(float) + (size_t)snap_cap * K * sizeof(float);
    const bool p2 = persist_pair2();
    auto kern = nctx == 1 ? (p2 ? hogwild_stream<K, MINB, 2, true> : hogwild_stream<K, MINB, 2, false>)
                          : (p2 ? hogwild_stream<K, MINB, 3, true> : hogwild_stream<K, MINB, 3, false>);
    cudaError_t e;
    const int per_sm = kernel_occupancy((const void *)kern, 32, smem, &e);
    if (e != cudaSuccess) return e;
    // every rank gets an equal share of the resident workers, at most
    // `window` (pairs in flight per rank) when one is set
    int64_t per_rank = (int64_t)per_sm * sm_count() / nctx;
    if (a.window > 0) per_rank = std::min<int64_t>(per_rank, a.window);
    if (const char *w = getenv("HEAT_PERSIST_WORKERS"))  // A/B knob: fewer workers
        if (atoi(w) > 0) per_rank = std::min<int64_t>(per_rank, atoi(w));
    if (per_rank < 1) return cudaErrorInvalidConfiguration;
    const int64_t nw = per_rank * nctx;
    std::vector<PersistRank> cx(ctx_host, ctx_host + nctx);
    for (int r = 0; r < nctx; ++r) cx[r].nblocks = (int)(nw / nctx + (r < nw % nctx ? 1 : 0));
    e = cudaMemcpyAsync(ctx_dev, cx.data(), nctx * sizeof(PersistRank), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    HogwildArgs b = a;
    b.l2_policy = stream_row_policy();
    if (!b.l2_policy) return cudaErrorNotSupported;  // (another kernel family takes the launch)
    if (nctx == 1) {  // the rank's tables and pairs as kernel parameters
        b.S = ctx_host->S; b.T = ctx_host->T; b.users = ctx_host->users;
        b.items = ctx_host->items; b.pair_index = ctx_host->pidx; b.ctr = ctx_host->ctr;
        b.start = 0;
    }
    b.spill_cap = a.N + 1;
    b.spill_stride = ((int64_t)b.spill_cap * (K * sizeof(float) + sizeof(WriteEntry) + sizeof(int2)) + 255) &
                     ~(int64_t)255;
    b.spill = static_cast<unsigned char *>(stream_scratch(1, (size_t)(b.spill_stride * nw), st));
    if (!b.spill) return cudaErrorMemoryAllocation;
    FastMod fm = FastMod::make((uint64_t)a.num_items);
    int snap = snap_cap;
    float band_lo = (float)a.theta - 1e-5f;
    unsigned long long *claim = nctx == 1 ? ctx_host->claim : nullptr;
    const PersistRank *cd = ctx_dev;
    int nc = nctx;
    int apply_warps = 0;  // per rank (A/B knob; the workers help between pairs anyway)
    if (const char *w = getenv("HEAT_PERSIST_APPLY_WARPS"))
        apply_warps = std::max(0, std::min(atoi(w), (int)per_rank - 1));
    unsigned long long *prof = persist_prof(st);
    if (nctx == 1) {
        kern<<<(unsigned)nw, 32, smem, st>>>(b, fm, snap, band_lo, claim, cd, nc, apply_warps, prof);
        return cudaGetLastError();
    }
    void *args[] = {&b, &fm, &snap, &band_lo, &claim, &cd, &nc, &apply_warps, &prof};
    return cudaLaunchCooperativeKernel((const void *)kern, dim3((unsigned)nw), dim3(32), args, smem,
                                       st);
}

void persist_watchdog_report() {
    unsigned long long v[4] = {0, 0, 0, 0};
    if (cudaMemcpyFromSymbol(v, g_watchdog, sizeof(v)) == cudaSuccess && v[0])
        fprintf(stderr, "[persist] watchdog: site %llu rank %llu value %llu block %llu\n", v[0], v[1],
                v[2], v[3]);
}

void persist_prof_report() {
    if (!g_prof) return;
    unsigned long long v[16];
    cudaMemcpy(v, g_prof, sizeof(v), cudaMemcpyDeviceToHost);
    cudaMemset(g_prof, 0, sizeof(v));
    const double tot = v[0] ? (double)v[0] : 1.0;
    fprintf(stderr,
            "[persist] warps %llu pairs %llu: gate %.1f%% help %.1f%% drain %.1f%% of warp clocks;"
            " apply units %llu (%.2f per pair); help calls %llu; clocks per accumulate unit %.0f"
            " (%llu units), per convert unit %.0f\n",
            v[6], v[5], 100.0 * v[1] / tot, 100.0 * v[2] / tot, 100.0 * v[3] / tot, v[4],
            v[5] ? (double)v[4] / v[5] : 0.0, v[7], v[10] ? (double)v[8] / v[10] : 0.0, v[10],
            (v[4] > v[10]) ? (double)v[9] / (v[4] - v[10]) : 0.0);
}

cudaError_t launch_shard_persist(const HogwildArgs &a, const PersistRank *ctx_host,
                                 PersistRank *ctx_dev, int nctx, cudaStream_t st) {
    if (!hogwild_stream_supported(a) || nctx < 1) return cudaErrorNotSupported;
    // launch bounds the persistent build is compiled for: K = 128 at 10 (the
    // registers still come out at 168, 12 warps per SM, and the codegen of the
    // pair loop is better: 28.9 M vs 27.1 M samples/s at 12 on c4), K = 64 at
    // 12; 8 / 11 / 12 / 14 for A/B runs
    int warps = a.K == 128 ? 10 : 12;
    if (const char *e = getenv("HEAT_PERSIST_WARPS")) warps = atoi(e) > 0 ? atoi(e) : warps;
    if (a.K == 128) {
        switch (warps) {
        case 8: return launch_persist_k<128, 8>(a, ctx_host, ctx_dev, nctx, st);
        case 11: return launch_persist_k<128, 11>(a, ctx_host, ctx_dev, nctx, st);
        case 12: return launch_persist_k<128, 12>(a, ctx_host, ctx_dev, nctx, st);
        default: return launch_persist_k<128, 10>(a, ctx_host, ctx_dev, nctx, st);
        }
    }
    switch (warps) {
    case 12: return launch_persist_k<64, 12>(a, ctx_host, ctx_dev, nctx, st);
    case 14: return launch_persist_k<64, 14>(a, ctx_host, ctx_dev, nctx, st);
    default: return launch_persist_k<64, 11>(a, ctx_host, ctx_dev, nctx, st);
    }
}

bool hogwild_stream_supported(const HogwildArgs &a) {
    return (a.K == 64 || a.K == 128) && !a.fp64 && a.cosine && !a.query &&
           ((uintptr_t)a.S % 16 == 0) && ((uintptr_t)a.T % 16 == 0);
}

cudaError_t launch_hogwild_stream(const HogwildArgs &a, cudaStream_t st, int *workers_out) {
    if (!hogwild_stream_supported(a)) return cudaErrorNotSupported;
    // resident warps per SM the register budget is compiled for
    int warps = 12;
    if (const char *e = getenv("HEAT_STREAM_WARPS")) warps = atoi(e) > 0 ? atoi(e) : warps;
    if (a.K == 128) {
        switch (warps) {
        case 8: return launch_stream_k<128, 8>(a, st, workers_out);
        case 10: return launch_stream_k<128, 10>(a, st, workers_out);
        case 16: return launch_stream_k<128, 16>(a, st, workers_out);
        default: return launch_stream_k<128, 12>(a, st, workers_out);
        }
    }
    switch (warps) {
    case 12: return launch_stream_k<64, 12>(a, st, workers_out);
    default: return launch_stream_k<64, 16>(a, st, workers_out);
    }
}

}  // namespace heat
