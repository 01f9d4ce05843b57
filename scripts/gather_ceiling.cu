// gather_ceiling.cu — what random-row gathers from an L2-resident table can
// reach on this GPU, independent of the training math.  The SGD kernels are
// gathers of ~1000 random 512-byte rows per pair (c4: T is 47 MB, L2-resident);
// this measures the row rate of pure gathers under the data paths the kernels
// can use, so the kernels' fraction of the achievable is known.
//
//   ldg  <LPR, U>: lanes-per-row LPR (8: 128 B per lane group, 32: a row per
//                   instruction), U independent row loads in flight per lane
//                   group, consumed by an FADD chain (registers only)
//   sts  <D>     : LDGSTS (cp.async 16 B) of 16-row stages into a D-deep ring,
//                   then LDS.128 reads of every byte (the staged kernel's path)
//   tma4 <D>     : TMA tile::gather4 (4 rows per instruction, one lane issues,
//                   mbarrier completion) of 16-row stages into a D-deep ring,
//                   then LDS.128 reads of every byte (`./gather_ceiling tma`)
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_ceiling gather_ceiling.cu
// Run:   ./gather_ceiling   (prints one line per variant: rows/s, GB/s, pairs/s at 1002 rows)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int LPR, int U>
__global__ void __launch_bounds__(32) gather_ldg(const float4 *__restrict__ T, int rows,
                                                 int iters, float *sink) {
    constexpr int RPI = 32 / LPR;  // rows per instruction
    constexpr int V = 32 / LPR;    // float4 per lane per row (K = 128)
    const int lane = threadIdx.x, g = lane / LPR, c = lane % LPR;
    uint32_t seed = blockIdx.x * 7919u + 17u;
    float acc = 0.f;
    float4 buf[U][V];
    auto issue = [&](int u, int it) {
        const uint32_t r = hash32(seed + (uint32_t)(it * U + u) * RPI + g) % (uint32_t)rows;
        const float4 *src = T + (size_t)r * 32 + c;
#pragma unroll
        for (int j = 0; j < V; ++j) buf[u][j] = __ldcg(src + j * LPR);
    };
#pragma unroll
    for (int u = 0; u < U; ++u) issue(u, 0);
    for (int it = 1; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int j = 0; j < V; ++j) acc += buf[u][j].x + buf[u][j].y + buf[u][j].z + buf[u][j].w;
            issue(u, it);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < V; ++j) acc += buf[u][j].x;
    if (acc == 12345.f) sink[0] = acc;
}

__device__ __forceinline__ void cp16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}

// one warp, 16-row stages (LPR 2 reads: lane = row half), ring of D stages
template <int D>
__global__ void __launch_bounds__(32) gather_sts(const float4 *__restrict__ T, int rows,
                                                 int iters, float *sink) {
    extern __shared__ float4 ring[];  // D * 16 rows * 33 float4 (padded)
    const int lane = threadIdx.x;
    uint32_t seed = blockIdx.x * 7919u + 17u;
    float acc = 0.f;
    auto issue = [&](int stage, int it) {
        float4 *dst = ring + stage * 16 * 33;
        for (int rr = 0; rr < 16; ++rr) {
            const uint32_t r = hash32(seed + (uint32_t)it * 16 + rr) % (uint32_t)rows;
            cp16(dst + rr * 33 + lane, T + (size_t)r * 32 + lane);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int s = 0; s < D; ++s) issue(s, s);
    for (int it = 0; it < iters; ++it) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        __syncwarp();
        const float4 *src = ring + (it % D) * 16 * 33 + (lane >> 1) * 33 + (lane & 1) * 16;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const float4 v = src[k];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        issue(it % D, it + D);
    }
    if (acc == 12345.f) sink[0] = acc;
}

// ---- TMA tile::gather4 into shared memory ----------------------------------
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int D>
__global__ void __launch_bounds__(32) gather_tma4(const __grid_constant__ CUtensorMap tmap,
                                                  int rows, int iters, float *sink) {
    extern __shared__ __align__(128) float4 ring4[];  // D stages x 16 rows x 32 float4
    __shared__ __align__(8) uint64_t bar[D];
    const int lane = threadIdx.x;
    uint32_t seed = blockIdx.x * 7919u + 17u;
    if (lane == 0)
        for (int i = 0; i < D; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    float acc = 0.f;
    auto issue = [&](int stage, int it) {
        if (lane != 0) return;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[stage])),
                     "r"(16 * 512) : "memory");
        float4 *dst = ring4 + stage * 16 * 32;
        for (int q = 0; q < 4; ++q) {
            int r[4];
            for (int k = 0; k < 4; ++k) r[k] = (int)(hash32(seed + (uint32_t)it * 16 + q * 4 + k) % (uint32_t)rows);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(s32(dst + q * 4 * 32)),
                "l"(&tmap), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(s32(&bar[stage]))
                : "memory");
        }
    };
    for (int s = 0; s < D; ++s) issue(s, s);
    for (int it = 0; it < iters; ++it) {
        const int st = it % D;
        const uint32_t parity = (uint32_t)((it / D) & 1);
        asm volatile(
            "{\n.reg .pred P1;\nW_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
            "@!P1 bra W_%=;\n}\n" ::"r"(s32(&bar[st])), "r"(parity) : "memory");
        const float4 *src = ring4 + st * 16 * 32 + lane;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const float4 v = src[k * 32];
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        issue(st, it + D);
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <typename F>
static void run(const char *name, F kern, int warps_per_sm, size_t smem, const float4 *T,
                int rows, int iters, int rows_per_iter, float *sink) {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
    const int per_sm = std::min(occ, warps_per_sm);
    const int grid = per_sm * sms;
    kern<<<grid, 32, smem>>>(T, rows, 4, sink);  // warm
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<grid, 32, smem>>>(T, rows, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = std::min(best, ms);
    }
    const double nrows = (double)grid * iters * rows_per_iter;
    const double s = best * 1e-3;
    printf("%-18s warps/SM %2d (occ %2d)  %8.3f Grows/s  %8.1f GB/s  %6.2f M pairs/s (1002 rows)%s\n",
           name, per_sm, occ, nrows / s / 1e9, nrows * 512 / s / 1e9, nrows / 1002 / s / 1e6,
           cudaGetLastError() == cudaSuccess ? "" : "  ERROR");
}

int main(int argc, char **argv) {
    const int rows = 92000;  // c4's item table: 92k x 128 fp32 = 47 MB
    float4 *T;
    float *sink;
    cudaMalloc(&T, (size_t)rows * 512);
    cudaMalloc(&sink, 4);
    cudaMemset(T, 0, (size_t)rows * 512);
    const int iters = 2000;
    if (argc > 1 && argv[1][0] == 't') {  // TMA gather4 into shared memory
        PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&encode, cudaEnableDefault, &q);
        if (!encode) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
        CUtensorMap tmap;
        cuuint64_t gdim[2] = {128, (cuuint64_t)rows};
        cuuint64_t gstride[1] = {512};
        cuuint32_t box[2] = {128, 1};
        cuuint32_t estride[2] = {1, 1};
        CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)T, gdim, gstride, box,
                            estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        for (int w : {8, 12, 16}) {
            auto k2 = [&](const float4 *, int rws, int its, float *sk, int grid, size_t smem) {
                gather_tma4<2><<<grid, 32, smem>>>(tmap, rws, its, sk);
            };
            auto k4 = [&](const float4 *, int rws, int its, float *sk, int grid, size_t smem) {
                gather_tma4<4><<<grid, 32, smem>>>(tmap, rws, its, sk);
            };
            for (int d : {2, 4}) {
                const size_t smem = (size_t)d * 16 * 512;
                auto kern = d == 2 ? (const void *)gather_tma4<2> : (const void *)gather_tma4<4>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                int occ = 0, sms = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32, smem);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
                const int per_sm = std::min(occ, w), grid = per_sm * sms;
                auto launch = [&](int its) { if (d == 2) k2(T, rows, its, sink, grid, smem); else k4(T, rows, its, sink, grid, smem); };
                launch(4);
                cudaEvent_t a, b;
                cudaEventCreate(&a); cudaEventCreate(&b);
                float best = 1e30f;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a); launch(iters); cudaEventRecord(b); cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
                }
                const double nrows = (double)grid * iters * 16, sec = best * 1e-3;
                printf("tma4 D%d           warps/SM %2d (occ %2d)  %8.3f Grows/s  %8.1f GB/s  %6.2f M pairs/s (1002 rows)%s\n",
                       d, per_sm, occ, nrows / sec / 1e9, nrows * 512 / sec / 1e9, nrows / 1002 / sec / 1e6,
                       cudaGetLastError() == cudaSuccess ? "" : "  ERROR");
            }
        }
        return 0;
    }
    if (argc > 1) {  // lanes-per-row sweep at the wide kernel's 12 warps/SM
        for (int w : {12, 16}) {
            run("ldg LPR4 U1", gather_ldg<4, 1>, w, 0, T, rows, iters, 1 * 8, sink);
            run("ldg LPR4 U2", gather_ldg<4, 2>, w, 0, T, rows, iters, 2 * 8, sink);
            run("ldg LPR8 U2", gather_ldg<8, 2>, w, 0, T, rows, iters, 2 * 4, sink);
            run("ldg LPR8 U4", gather_ldg<8, 4>, w, 0, T, rows, iters, 4 * 4, sink);
            run("ldg LPR16 U4", gather_ldg<16, 4>, w, 0, T, rows, iters, 4 * 2, sink);
            run("ldg LPR16 U8", gather_ldg<16, 8>, w, 0, T, rows, iters, 8 * 2, sink);
        }
        return 0;
    }
    for (int w : {8, 12, 16, 24, 32}) {
        run("ldg LPR8 U2", gather_ldg<8, 2>, w, 0, T, rows, iters, 2 * 4, sink);
        run("ldg LPR8 U4", gather_ldg<8, 4>, w, 0, T, rows, iters, 4 * 4, sink);
        run("ldg LPR32 U4", gather_ldg<32, 4>, w, 0, T, rows, iters, 4, sink);
        run("ldg LPR32 U8", gather_ldg<32, 8>, w, 0, T, rows, iters, 8, sink);
        run("ldg LPR32 U16", gather_ldg<32, 16>, w, 0, T, rows, iters, 16, sink);
        run("sts D1", gather_sts<1>, w, 1 * 16 * 33 * 16, T, rows, iters, 16, sink);
        run("sts D2", gather_sts<2>, w, 2 * 16 * 33 * 16, T, rows, iters, 16, sink);
    }
    return 0;
}
