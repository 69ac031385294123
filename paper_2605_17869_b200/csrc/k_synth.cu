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

// ---- test probe: the device libm restatements over caller arrays ----------------
#include "dsift_math.cuh"
namespace dsift {
__global__ void libm_probe_kernel(int mode, const void* in, long long n, void* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (mode == 0) {   // atan2f(y, x): in float2 (y, x) -> float
            const float2 yx = static_cast<const float2*>(in)[i];
            static_cast<float*>(out)[i] = dsift_atan2f(yx.x, yx.y);
        } else if (mode == 1) {   // exp(double) -> double
            static_cast<double*>(out)[i] = dsift_exp(static_cast<const double*>(in)[i]);
        } else if (mode == 3) {   // in-range fast division vs __fdiv_rn: in = uint64 seed,
                                  // out = [mismatches, first (y bits << 32 | x bits)]
            const unsigned long long seed = *static_cast<const unsigned long long*>(in);
            unsigned long long z = seed + 0x9E3779B97F4A7C15ull * (unsigned long long)(i + 1);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            z ^= z >> 31;
            // operands: random mantissas and signs, exponents in [-100, 62]; every
            // 4th pair puts y near a multiple of x (quotients near integers /
            // halfway points, where a one-ulp slip would show)
            const unsigned mx = (unsigned)(z & 0x7fffffu), my = (unsigned)((z >> 23) & 0x7fffffu);
            const int ex = (int)((z >> 46) % 163u) - 100;
            // atan2f only divides when the exponents differ by <= 60 (its gap test)
            const int ey = (i & 3) == 3 ? ex : max(-100, min(62, ex + (int)((z >> 54) % 121u) - 60));
            const unsigned sx = (unsigned)(z >> 62) & 1u, sy = (unsigned)(z >> 63) & 1u;
            const float x = __uint_as_float((sx << 31) | ((unsigned)(ex + 127) << 23) | mx);
            float y = __uint_as_float((sy << 31) | ((unsigned)(ey + 127) << 23) | my);
            if ((i & 3) == 3) y = __fmul_rn(x, (float)((int)(z >> 40) & 1023) * 0.5f + 0.5f);
            if (y != 0.0f && (fabsf(y) < 0x1p-100f || fabsf(y) > 0x1p62f)) y = x;
            const float a = ds_fdiv_inrange(y, x), b = __fdiv_rn(y, x);
            if (__float_as_uint(a) != __float_as_uint(b)) {
                unsigned long long* o = static_cast<unsigned long long*>(out);
                if (atomicAdd(o, 1ull) == 0ull)
                    o[1] = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
            }
        } else {   // sincos(double) -> double2 (sin, cos)
            double s, c;
            dsift_sincos(static_cast<const double*>(in)[i], &s, &c);
            static_cast<double2*>(out)[i] = make_double2(s, c);
        }
    }
}
cudaError_t launch_libm_probe(int mode, const void* in, long long n, void* out, cudaStream_t st) {
    libm_probe_kernel<<<mode == 3 ? 148 * 16 : 256, 256, 0, st>>>(mode, in, n, out);
    return cudaGetLastError();
}
}  // namespace dsift
