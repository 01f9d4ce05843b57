// heat_common.cuh — shared device helpers for the B200 CCL training path.
//
// Counter-form SplitMix64 (restates /root/reference/pkg/src/heatcf/rng.py:26-31
// and 63-76): draw n (0-based) of the stream whose state is s0 is
// mix64(s0 + (n + 1) * GAMMA).  The reference's single-thread epoch draws
// negative j of the pair at epoch position p as draw p*N + j
// (trainer.py:134-139), so a sampler keyed by the global pair index returns
// the reference's ids whatever the thread/warp/GPU decomposition.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace heat {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kMix1;
    z = (z ^ (z >> 27)) * kMix2;
    return z ^ (z >> 31);
}

// Exact z mod n for 64-bit z and 1 <= n < 2^31 without the slow 64-bit
// division routine: q0 = umulhi(z, floor((2^64-1)/n)) satisfies
// q - 2 <= q0 <= q, so at most two corrections.  (rng.py:76 takes
// `rng_next(state) % uint64(n)`; tests check this against % on device.)
struct FastMod {
    uint64_t n;
    uint64_t m;  // floor((2^64 - 1) / n)
    __host__ __device__ static FastMod make(uint64_t n) { return FastMod{n, ~0ull / n}; }
    __device__ __forceinline__ uint64_t mod(uint64_t z) const {
        uint64_t q = __umul64hi(z, m);
        uint64_t r = z - q * n;
        if (r >= n) r -= n;
        if (r >= n) r -= n;
        return r;
    }
};

// Negative j of the pair at global epoch position p.
__device__ __forceinline__ int32_t neg_id(uint64_t s0, int64_t p, int n_neg, int j,
                                          const FastMod &fm) {
    uint64_t n = (uint64_t)p * (uint64_t)n_neg + (uint64_t)j;
    return (int32_t)fm.mod(mix64(s0 + (n + 1ull) * kGamma));
}

__device__ __forceinline__ float4 ldcg4(const float *p) {
    return __ldcg(reinterpret_cast<const float4 *>(p));
}

// Vector atomic add (sm_90+: red.global.add.v4.f32), no return value.
__device__ __forceinline__ void red_add4(float *addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
}

}  // namespace heat

namespace heat {
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
}  // namespace heat

// ---- async-copy (TMA bulk) + mbarrier helpers (sm_90+ PTX) -----------------
namespace heat {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// try_wait with a suspend-time hint: the warp sleeps until the phase
// completes (or the hint elapses) instead of re-polling
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "HEAT_WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra HEAT_WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "HEAT_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra HEAT_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0,
// both addresses 16-byte aligned).  Lands in SASS as UBLKCP.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Same with an L2 eviction-priority policy (createpolicy).
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes,
                                              uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void red_add2(float *addr, float a, float b) {
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(addr), "f"(a), "f"(b) : "memory");
}

}  // namespace heat

// ---- Ampere-style async copies (LDGSTS), 16 bytes per lane -----------------
namespace heat {

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}

__device__ __forceinline__ void cp_async16_hint(void *dst, const void *src, uint64_t policy) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)),
                 "l"(src), "l"(policy)
                 : "memory");
}

__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace heat

// ---- binary64 row dots in the reference's order, loads batched ------------
// tt = sum_k v_k*v_k and st = sum_k u_k*v_k accumulated strictly in k order
// with separate round-to-nearest multiply and add (trainer.py:193-197), the
// row read in bursts of up to 64 floats (16 independent 16-byte loads) so a
// row costs one or two memory latencies instead of one per element.
namespace heat {

template <int K>
__device__ __forceinline__ void row_dots_f64(const float *__restrict__ row, const double *ubuf,
                                             double &tt, double &st) {
    constexpr int C4 = K / 4;
    constexpr int B4 = C4 < 16 ? C4 : 16;  // float4s per burst
    const float4 *r4 = reinterpret_cast<const float4 *>(row);
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int c0 = 0; c0 < C4; c0 += B4) {
        float4 v[B4];
#pragma unroll
        for (int c = 0; c < B4; ++c) v[c] = r4[c0 + c];
#pragma unroll
        for (int c = 0; c < B4; ++c) {
            const int k = 4 * (c0 + c);
            const double x0 = (double)v[c].x, x1 = (double)v[c].y, x2 = (double)v[c].z,
                         x3 = (double)v[c].w;
            a = __dadd_rn(a, __dmul_rn(x0, x0)); b = __dadd_rn(b, __dmul_rn(ubuf[k], x0));
            a = __dadd_rn(a, __dmul_rn(x1, x1)); b = __dadd_rn(b, __dmul_rn(ubuf[k + 1], x1));
            a = __dadd_rn(a, __dmul_rn(x2, x2)); b = __dadd_rn(b, __dmul_rn(ubuf[k + 2], x2));
            a = __dadd_rn(a, __dmul_rn(x3, x3)); b = __dadd_rn(b, __dmul_rn(ubuf[k + 3], x3));
        }
    }
    tt = a;
    st = b;
}

// runtime-K dispatch: templated bursts for K in {16,32,64,128,256} (16-byte
// aligned rows), a scalar sequential loop otherwise
__device__ __forceinline__ void row_dots_any(const float *__restrict__ row, const double *ubuf,
                                             int K, double &tt, double &st) {
    const bool al = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
    if (al) {
        switch (K) {
        case 16: row_dots_f64<16>(row, ubuf, tt, st); return;
        case 32: row_dots_f64<32>(row, ubuf, tt, st); return;
        case 64: row_dots_f64<64>(row, ubuf, tt, st); return;
        case 128: row_dots_f64<128>(row, ubuf, tt, st); return;
        case 256: row_dots_f64<256>(row, ubuf, tt, st); return;
        default: break;
        }
    }
    double a = 0.0, b = 0.0;
    for (int k = 0; k < K; ++k) {
        const double x = (double)row[k];
        a = __dadd_rn(a, __dmul_rn(x, x));
        b = __dadd_rn(b, __dmul_rn(ubuf[k], x));
    }
    tt = a;
    st = b;
}

}  // namespace heat
