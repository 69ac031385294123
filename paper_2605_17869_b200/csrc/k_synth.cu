// k_synth.cu — on-device synthetic input: synth::value_noise_image
// (reference tests/support/synth.cpp:14-66) with the identical integer hash
// and FP64 arithmetic (this file is compiled with -fmad=false), so device
// images are bit-identical to the host generator.  Used by bench.py to make
// batches without a host-side bottleneck.
#include <cuda_runtime.h>
#include <float.h>

#include "dsift_common.cuh"

namespace dsift {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ double lattice(unsigned long long seed, long long gx, long long gy) {
    const unsigned long long h = mix64(seed ^ mix64((unsigned long long)gx * 0x9e3779b97f4a7c15ull ^
                                                    (unsigned long long)gy * 0xbf58476d1ce4e5b9ull));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double smooth_noise(unsigned long long seed, double x, double y) {
    const long long gx = (long long)floor(x), gy = (long long)floor(y);
    const double fx = x - gx, fy = y - gy;
    const double sx = fx * fx * (3.0 - 2.0 * fx);
    const double sy = fy * fy * (3.0 - 2.0 * fy);
    const double v00 = lattice(seed, gx, gy), v10 = lattice(seed, gx + 1, gy);
    const double v01 = lattice(seed, gx, gy + 1), v11 = lattice(seed, gx + 1, gy + 1);
    const double top = v00 + sx * (v10 - v00);
    const double bot = v01 + sx * (v11 - v01);
    return top + sy * (bot - top);
}

// pass 1: raw values (float) + per-block min/max of the double values
__global__ void value_noise_kernel(float* out, int w, int h, unsigned long long seed0, int octaves,
                                   int cells, double* part_lo, double* part_hi) {
    const int b = blockIdx.y;
    const unsigned long long seed = seed0 + (unsigned long long)b;
    float* img = out + (long long)b * w * h;
    double lo = 1e9, hi = -1e9;
    const long long npx = (long long)w * h;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx;
         p += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(p % w), y = (int)(p / w);
        double v = 0.0, amp = 1.0, cl = cells;
        for (int o = 0; o < octaves; ++o) {
            v += amp * smooth_noise(seed + (unsigned long long)o, x * cl / w, y * cl / h);
            amp *= 0.55;
            cl *= 2.0;
        }
        img[p] = (float)v;
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    __shared__ double slo[256], shi[256];
    slo[threadIdx.x] = lo;
    shi[threadIdx.x] = hi;
    __syncthreads();
    for (int d = blockDim.x / 2; d; d >>= 1) {
        if ((int)threadIdx.x < d) {
            slo[threadIdx.x] = fmin(slo[threadIdx.x], slo[threadIdx.x + d]);
            shi[threadIdx.x] = fmax(shi[threadIdx.x], shi[threadIdx.x + d]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_lo[b * gridDim.x + blockIdx.x] = slo[0];
        part_hi[b * gridDim.x + blockIdx.x] = shi[0];
    }
}

// pass 2: min-max normalise (synth.cpp:60-64); min/max are exact, order-free
__global__ void value_noise_norm_kernel(float* out, int w, int h, const double* part_lo,
                                        const double* part_hi, int nparts) {
    const int b = blockIdx.y;
    __shared__ double lo_s, span_s;
    if (threadIdx.x == 0) {
        double lo = 1e9, hi = -1e9;
        for (int i = 0; i < nparts; ++i) {
            lo = fmin(lo, part_lo[b * nparts + i]);
            hi = fmax(hi, part_hi[b * nparts + i]);
        }
        lo_s = lo;
        span_s = hi > lo ? hi - lo : 1.0;
    }
    __syncthreads();
    float* img = out + (long long)b * w * h;
    const long long npx = (long long)w * h;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npx;
         p += (long long)gridDim.x * blockDim.x)
        img[p] = (float)(((double)img[p] - lo_s) / span_s);
}

cudaError_t launch_value_noise(float* out, int n, int w, int h, unsigned long long seed0, int octaves,
                               int cells, double* scratch, int nparts, cudaStream_t st) {
    const dim3 grid(nparts, n);
    value_noise_kernel<<<grid, 256, 0, st>>>(out, w, h, seed0, octaves, cells, scratch,
                                             scratch + (long long)n * nparts);
    value_noise_norm_kernel<<<grid, 256, 0, st>>>(out, w, h, scratch, scratch + (long long)n * nparts,
                                                  nparts);
    return cudaGetLastError();
}

}  // namespace dsift

