// heat_sample.cu — device negative sampler (trainer.py:135-139, rng.py:63-76).
// One thread per (pair, negative): the counter-form SplitMix64 draw
// p*N + j of the epoch stream, reduced mod num_items exactly.
#include "heat_common.cuh"
#include "heat_internal.h"

namespace heat {

__global__ void sample_kernel(uint64_t s0, int64_t first_pair, int64_t total, int N, FastMod fm,
                              int32_t *__restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < total; i += stride) {
        int64_t p = first_pair + i / N;
        int j = (int)(i % N);
        out[i] = neg_id(s0, p, N, j, fm);
    }
}

cudaError_t launch_sample(uint64_t s0, int64_t first_pair, int64_t npairs, int N,
                          int64_t num_items, int32_t *out, cudaStream_t stream) {
    int64_t total = npairs * (int64_t)N;
    if (total == 0) return cudaSuccess;
    int blocks = (int)((total + 255) / 256);
    int cap = sm_count() * 8;
    if (blocks > cap) blocks = cap;
    sample_kernel<<<blocks, 256, 0, stream>>>(s0, first_pair, total, N,
                                              FastMod::make((uint64_t)num_items), out);
    return cudaGetLastError();
}

}  // namespace heat
