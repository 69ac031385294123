// k_sort.cu — K7: canonical order (reference: core.cpp:116-170
// keypoint_less / canonical_sort) and per-image segmentation.
//
// The reference's total order is (octave, interval, y, x, angle, sigma,
// response, descriptor bytes).  All keypoint floats are >= +0 (angle -0 is
// canonicalised, orient.cpp:99-100), so their IEEE bit patterns order like
// the values and the order is an LSD radix sort on three 64-bit keys:
//   k1 = sigma:response,  k2 = x:angle,  k3 = image:octave:interval:y.
// Descriptors are a pure function of the keypoint fields, so full-key ties
// are byte-identical rows and the descriptor tie-break never changes bytes;
// the CTA sort therefore runs BEFORE descriptors, which are then written
// directly in canonical order (no 512-byte row permutation).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"

namespace dsift {

__global__ void sort_keys_kernel(const DevKeypoint* __restrict__ kp, const unsigned long long* n_dev,
                                 long long cap, int which, const int* __restrict__ perm,
                                 unsigned long long* __restrict__ keys, int* __restrict__ idx) {
    const long long n = (long long)*n_dev;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cap;
         i += (long long)gridDim.x * blockDim.x) {
        const long long src = perm ? perm[i] : i;
        unsigned long long key;
        if (src >= n) {
            key = ~0ull;
        } else {
            const DevKeypoint k = kp[src];
            if (which == 0)
                key = ((unsigned long long)__float_as_uint(k.sigma) << 32) | __float_as_uint(k.response);
            else if (which == 1)
                key = ((unsigned long long)__float_as_uint(k.x) << 32) | __float_as_uint(k.angle);
            else
                key = ((unsigned long long)(unsigned)k.image << 42) |
                      ((unsigned long long)(unsigned)(k.octave & 31) << 37) |
                      ((unsigned long long)(unsigned)(k.interval & 31) << 32) | __float_as_uint(k.y);
        }
        keys[i] = key;
        if (!perm) idx[i] = (int)i;
    }
}

__global__ void gather_kernel(const DevKeypoint* __restrict__ in, const int* __restrict__ perm,
                              const unsigned long long* n_dev, DevKeypoint* __restrict__ out,
                              dsift_keypoint* __restrict__ out_pub) {
    const long long n = (long long)*n_dev;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const DevKeypoint k = in[perm[i]];
        out[i] = k;
        dsift_keypoint p;
        p.x = k.x;
        p.y = k.y;
        p.sigma = k.sigma;
        p.angle = k.angle;
        p.response = k.response;
        p.octave = k.octave;
        p.interval = k.interval;
        out_pub[i] = p;
    }
}

// offsets[b] = first index of image b in the sorted list (b in [0, batch]).
__global__ void image_offsets_kernel(const DevKeypoint* __restrict__ sorted, const unsigned long long* n_dev,
                                     int batch, long long* offsets) {
    const long long n = (long long)*n_dev;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b <= batch; b += gridDim.x * blockDim.x) {
        long long lo = 0, hi = n;
        while (lo < hi) {
            const long long mid = (lo + hi) >> 1;
            if (sorted[mid].image < b) lo = mid + 1; else hi = mid;
        }
        offsets[b] = lo;
    }
}

size_t sort_temp_bytes(long long cap) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr,
                                    (int)cap, 0, 64);
    return bytes;
}

// Sorts in[0..n) (n on device, capacity cap) into out / out_pub; returns the
// number of kernel launches issued through *launches.
cudaError_t launch_canonical_sort(const DevKeypoint* in, const unsigned long long* n_dev, long long cap,
                                  const SortBuffers& sb, DevKeypoint* out, dsift_keypoint* out_pub,
                                  int batch, long long* offsets, cudaStream_t st, long long* launches) {
    if (cap <= 0) return cudaSuccess;
    const int threads = 256;
    const int grid = (int)std::min<long long>((cap + threads - 1) / threads, 148 * 16);
    const int* perm = nullptr;
    int* cur_idx = sb.idx_a;
    for (int which = 0; which < 3; ++which) {
        sort_keys_kernel<<<grid, threads, 0, st>>>(in, n_dev, cap, which, perm, sb.keys_a,
                                                   which == 0 ? sb.idx_a : nullptr);
        ++*launches;
        size_t tb = sb.temp_bytes;
        const int* vin = (which == 0) ? sb.idx_a : perm;
        // keys_a/vin -> keys_b/idx_b ; then idx_b becomes the permutation
        int* vout = (vin == sb.idx_b) ? sb.idx_a : sb.idx_b;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(sb.temp, tb, sb.keys_a, sb.keys_b, vin, vout,
                                                        (int)cap, 0, 64, st);
        if (e != cudaSuccess) return e;
        *launches += 10;  // onesweep on 64-bit keys: histogram + exclusive sum + 8 digit passes
        perm = vout;
        cur_idx = vout;
    }
    (void)cur_idx;
    gather_kernel<<<grid, threads, 0, st>>>(in, perm, n_dev, out, out_pub);
    image_offsets_kernel<<<1, 256, 0, st>>>(out, n_dev, batch, offsets);
    *launches += 2;
    return cudaGetLastError();
}

}  // namespace dsift
