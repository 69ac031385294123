// k_ingest.cu — image ingest (reference: io.cpp:49-81 load_image).
//
// 8-bit P5/P6 payloads travel to the device as bytes (4x less H2D than the
// float GrayImage) and are converted there with the reference's arithmetic:
//   gray:  float(b * (1.0 / 255.0))                                  io.cpp:77-78
//   color: float(((0.299 r + 0.587 g) + 0.114 b) * (1.0 / 255.0))    io.cpp:71-75
// in double, left to right, no contraction (this file is built -fmad=false).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"

namespace dsift {

__global__ void ingest_u8_kernel(const unsigned char* __restrict__ in, long long n_px, int channels,
                                 float* __restrict__ out) {
    const double inv255 = 1.0 / 255.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_px;
         i += (long long)gridDim.x * blockDim.x) {
        double v;
        if (channels == 1) {
            v = __dmul_rn((double)in[i], inv255);
        } else {
            const double r = in[3 * i], g = in[3 * i + 1], b = in[3 * i + 2];
            v = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)), __dmul_rn(0.114, b)),
                          inv255);
        }
        out[i] = __double2float_rn(v);
    }
}

cudaError_t launch_ingest_u8(const unsigned char* in, long long n_px, int channels, float* out, cudaStream_t st) {
    if (n_px <= 0) return cudaSuccess;
    const int grid = (int)std::min<long long>((n_px + 255) / 256, 148LL * 16);
    ingest_u8_kernel<<<grid, 256, 0, st>>>(in, n_px, channels, out);
    return cudaGetLastError();
}

}  // namespace dsift
