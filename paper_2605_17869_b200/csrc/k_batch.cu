// k_batch.cu — result bookkeeping on the device.
//
// A batch may hold images of several sizes (the reference's extract takes any
// image size per call, io.cpp:111-142; C5 mixes ten resolutions).  The host
// groups same-size images and runs the pipeline once per group, each group
// writing canonical-order rows into its own staging slice.  These kernels
// fold each group's counters into the result and, at the end, concatenate
// the per-image row ranges in batch order — the reference's per-index slots
// concatenated in index order (io.cpp:118-139).  No host synchronisation:
// counts and offsets never leave the device.
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"

namespace dsift {

__global__ void fold_totals_kernel(const Counters* __restrict__ ctr, BatchTotals* __restrict__ tot) {
    tot->err |= ctr->err;
    tot->slow += (unsigned long long)ctr->n_slow + ctr->n_fixed;
    tot->lattice += ctr->lattice;
    tot->lattice_in += ctr->lattice_in;
}

cudaError_t launch_fold_totals(const Counters* ctr, BatchTotals* tot, cudaStream_t st) {
    fold_totals_kernel<<<1, 1, 0, st>>>(ctr, tot);
    return cudaGetLastError();
}

// offsets[i] = exclusive scan over images of count_i (one CTA, chunks of 1024)
__global__ void __launch_bounds__(1024)
ragged_offsets_kernel(const long long* __restrict__ map, const long long* __restrict__ stage_offs, int n,
                      long long* __restrict__ offsets) {
    __shared__ long long warp_sum[32];
    __shared__ long long carry_s;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
        const int i = base + threadIdx.x;
        long long cnt = 0;
        if (i < n) {
            const long long e = map[2 * i];
            cnt = stage_offs[e + 1] - stage_offs[e];
        }
        long long incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long nb = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += nb;
        }
        if (lane == 31) warp_sum[warp] = incl;
        __syncthreads();
        long long woff = 0, tot = 0;
        for (int q = 0; q < 32; ++q) {
            woff += q < warp ? warp_sum[q] : 0;
            tot += warp_sum[q];
        }
        const long long carry = carry_s;
        if (i < n) offsets[i] = carry + woff + incl - cnt;
        __syncthreads();
        if (threadIdx.x == 0) carry_s = carry + tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) offsets[n] = carry_s;
}

// grid (chunks, n): CTA row of image i copies its rows; 16-byte units
__global__ void __launch_bounds__(256)
ragged_copy_kernel(const long long* __restrict__ map, const long long* __restrict__ stage_offs,
                   const dsift_keypoint* __restrict__ skp, const float* __restrict__ sdesc,
                   const unsigned char* __restrict__ su8, const long long* __restrict__ offsets,
                   dsift_keypoint* __restrict__ kp, float* __restrict__ desc, unsigned char* __restrict__ u8) {
    const int i = blockIdx.y;
    const long long e = map[2 * i];
    const long long src0 = map[2 * i + 1] + stage_offs[e];
    const long long rows = stage_offs[e + 1] - stage_offs[e];
    const long long dst0 = offsets[i];
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // descriptors: 32 float4 per row; uint8: 8 uint4 per row
    const float4* ds = reinterpret_cast<const float4*>(sdesc + src0 * kDescDim);
    float4* dd = reinterpret_cast<float4*>(desc + dst0 * kDescDim);
    for (long long q = t0; q < rows * (kDescDim / 4); q += stride) dd[q] = ds[q];
    const uint4* us = reinterpret_cast<const uint4*>(su8 + src0 * kDescDim);
    uint4* ud = reinterpret_cast<uint4*>(u8 + dst0 * kDescDim);
    for (long long q = t0; q < rows * (kDescDim / 16); q += stride) ud[q] = us[q];
    for (long long q = t0; q < rows; q += stride) kp[dst0 + q] = skp[src0 + q];
}

cudaError_t launch_ragged_gather(const long long* map, const long long* stage_offs, int n,
                                 const dsift_keypoint* skp, const float* sdesc, const unsigned char* su8,
                                 long long* offsets, dsift_keypoint* kp, float* desc, unsigned char* u8,
                                 cudaStream_t st) {
    ragged_offsets_kernel<<<1, 1024, 0, st>>>(map, stage_offs, n, offsets);
    ragged_copy_kernel<<<dim3(16, n), 256, 0, st>>>(map, stage_offs, skp, sdesc, su8, offsets, kp, desc, u8);
    return cudaGetLastError();
}

}  // namespace dsift
