// dmma_peak.cu — measured binary64 tensor-core ceiling of this GPU, the
// roofline denominator of the recall@K evaluator (heat_eval.cu scores with
// mma.sync m8n8k4 f64: tcgen05 has no binary64 kind).
//
// Every warp issues mma.sync.m8n8k4.f64 back to back on 8 independent
// accumulator chains (register operands only: no memory traffic), at 4..32
// warps per SM.  512 flops per instruction (8 x 8 x 4 multiply-adds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_peak scripts/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(int iters, double *sink) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[j][0]), "+d"(c[j][1])
                         : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    if (s == 1234.5) sink[0] = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *sink;
    cudaMalloc(&sink, 8);
    const int iters = 20000;
    double best = 0.0;
    for (int wps : {4, 8, 16, 32}) {
        const int grid = sms * wps / 4;  // 4 warps per CTA
        dmma_loop<<<grid, 128>>>(iters / 10, sink);  // warm-up
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms_best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            dmma_loop<<<grid, 128>>>(iters, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            ms_best = ms < ms_best ? ms : ms_best;
        }
        const double flops = (double)grid * 4 * iters * 8 * 512.0;
        const double tf = flops / (ms_best * 1e-3) / 1e12;
        best = tf > best ? tf : best;
        printf("{\"warps_per_sm\": %d, \"ms\": %.3f, \"fp64_tensor_tflops\": %.2f}\n", wps, ms_best, tf);
    }
    printf("{\"fp64_tensor_tflops_best\": %.2f, \"sms\": %d, \"error\": \"%s\"}\n", best, sms,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
