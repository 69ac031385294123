// tests/native/libm_probe.cu — TEST-ONLY library (tests/native/libdsift_probe.so):
// evaluates the product's device restatements of the host libm calls on the
// path (paper_2605_17869_b200/csrc/dsift_math.cuh: glibc atan2f, __exp_fma,
// correctly rounded sin/cos, the atan2f fast-path division) over caller
// arrays, so tests can compare them with the live glibc.  Not part of the
// product library.  Built by __graft_entry__.build() with the product's flags.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_2605_17869_b200/csrc/dsift_math.cuh"

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
}  // namespace dsift

// mode 0: atan2f, in = n x {y, x} float32, out = n float32; mode 1: exp,
// in/out = n float64; mode 2: sin/cos, in = n float64, out = n x {sin, cos};
// mode 3: in = uint64 seed, out = uint64[2] {mismatches, first failing pair}
// of the fast division over n random operand pairs.  Host buffers.
extern "C" int dsift_test_libm_probe(int mode, const void* in, long long n, void* out) {
    if (mode < 0 || mode > 3 || n < 0) return 1;
    const size_t isz = mode == 3 ? 8 : 8 * (size_t)(n > 0 ? n : 1);
    const size_t osz = mode == 3 ? 16 : (mode == 0 ? 4 : (mode == 1 ? 8 : 16)) * (size_t)(n > 0 ? n : 1);
    void *din = nullptr, *dout = nullptr;
    if (cudaMalloc(&din, isz) != cudaSuccess || cudaMalloc(&dout, osz) != cudaSuccess) return 2;
    cudaMemcpy(din, in, mode == 3 ? 8 : isz, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, osz);
    dsift::libm_probe_kernel<<<mode == 3 ? 148 * 16 : 256, 256>>>(mode, din, n, dout);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dout, osz, cudaMemcpyDeviceToHost);
    cudaFree(din);
    cudaFree(dout);
    return e == cudaSuccess ? 0 : 3;
}
