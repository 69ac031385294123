// tools/fp64_peak.cu — measured FP64 DFMA throughput of this B200 (the
// co-roofline of K1's blur): every thread runs 8 independent DFMA
// chains; grid = 8 CTAs x 256 threads per SM.  Prints one JSON line:
//   {"dfma_per_s": ..., "fp64_tflops": ..., "sm_count": ..., "ms": ...}
// Built by __graft_entry__.build(); run by bench.py (once, before the timed region).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = __fma_rn(x[j], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[0] = s;   // keeps the chains live
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double));
    const int grid = sms * 8, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) dfma_kernel<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        dfma_kernel<<<grid, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    if (cudaGetLastError() != cudaSuccess) {
        printf("{\"error\": \"launch failed\"}\n");
        return 1;
    }
    const double dfma = (double)grid * 256 * iters * 8;
    const double rate = dfma / (best / 1e3);
    printf("{\"dfma_per_s\": %.6e, \"fp64_tflops\": %.3f, \"sm_count\": %d, \"ms\": %.4f}\n", rate, 2 * rate / 1e12,
           sms, best);
    return 0;
}
