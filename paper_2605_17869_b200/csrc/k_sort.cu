// k_sort.cu — K7: canonical order (reference: core.cpp:116-170
// keypoint_less / canonical_sort) and per-image segmentation, plus the
// device-wide exclusive scan the detector's compaction uses.
//
// The reference's total order is (octave, interval, y, x, angle, sigma,
// response, descriptor bytes).  Descriptors are a pure function of the
// keypoint fields, so full-key ties are byte-identical rows: the sort runs
// BEFORE the descriptor stage, which then writes rows directly in canonical
// order (no 512-byte row permutation).
//
// Bucket sort over the actual count n (device-resident, never the capacity):
//   bucket(kp) = image * NBI + (octave * s + interval - 1) * H + floor(y)
// (H = input height; y is in input coordinates, y in [0, H)), which is
// monotone in the key's leading fields (image, octave, interval, y).  A
// C3 image has ~15k keypoints over 8*3*1200 = 28.8k buckets, so a bucket
// holds ~0.5 keypoints on average (orientation fan-out copies share one).
//   K7a count:   bucket id per keypoint + integer-atomic bucket counts;
//   K7b scan:    exclusive scan of the counts (decoupled look-back);
//   K7c scatter: slot = bucket start + atomic cursor (arbitrary order inside
//                a bucket ...);
//   K7d rank:    ... made canonical: each keypoint's final slot is its bucket
//                start + the number of bucket members with a smaller
//                (y, x, angle, sigma, response, original index) — a pure
//                function of the data, whatever order K7c produced;
//   K7e gather:  sorted DevKeypoint list, the public 28-byte keypoints and the
//                per-image offsets (= the start of each image's first bucket).
// All keypoint floats are >= +0 here (x, y > 0 by construction, sigma > 0,
// response = |D|, angle canonicalised to +0, orient.cpp:99-100), so their
// IEEE bit patterns order like the values.
#include <cuda_runtime.h>

#include <algorithm>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_scan.cuh"

namespace dsift {

// ---- device-wide exclusive scan of uint32 (single pass, decoupled look-back) ----
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads)
scan_u32_kernel(const unsigned* __restrict__ in, unsigned* __restrict__ out, long long n, ScanState st,
                unsigned n_tiles, unsigned* total_out) {
    __shared__ unsigned ticket_s;
    __shared__ unsigned long long off_s;
    __shared__ unsigned warp_sum[kScanThreads / 32];
    const unsigned t = scan_ticket(st, &ticket_s);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long base = (long long)t * kScanTile + (long long)threadIdx.x * kScanItems;
    unsigned v[kScanItems];
    unsigned sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < n ? __ldg(in + base + k) : 0u;
        sum += v[k];
    }
    unsigned incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned nb = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += nb;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    unsigned warp_off = 0, tile_total = 0;
#pragma unroll
    for (int q = 0; q < kScanThreads / 32; ++q) {
        warp_off += q < warp ? warp_sum[q] : 0u;
        tile_total += warp_sum[q];
    }
    const unsigned long long off = scan_exclusive(st, t, tile_total, n_tiles, &off_s);
    unsigned run = (unsigned)off + warp_off + incl - sum;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
    if (total_out && t == n_tiles - 1 && threadIdx.x == kScanThreads - 1) *total_out = run;
}

size_t scan_state_bytes(long long n) {
    const long long tiles = std::max<long long>(1, (n + kScanTile - 1) / kScanTile);
    return sizeof(unsigned long long) * (size_t)tiles + 256;
}

cudaError_t launch_scan_u32(const unsigned* in, unsigned* out, long long n, void* state, unsigned* total_out,
                            cudaStream_t st) {
    if (n <= 0) {
        if (total_out) return cudaMemsetAsync(total_out, 0, sizeof(unsigned), st);
        return cudaSuccess;
    }
    const unsigned tiles = (unsigned)((n + kScanTile - 1) / kScanTile);
    cudaError_t e = cudaMemsetAsync(state, 0, scan_state_bytes(n), st);
    if (e != cudaSuccess) return e;
    ScanState s;
    s.states = static_cast<unsigned long long*>(state);
    s.ticket = reinterpret_cast<unsigned*>(static_cast<char*>(state) + sizeof(unsigned long long) * tiles);
    s.total = reinterpret_cast<unsigned long long*>(static_cast<char*>(state) + sizeof(unsigned long long) * tiles + 64);
    s.cap = ~0ull;
    scan_u32_kernel<<<tiles, kScanThreads, 0, st>>>(in, out, n, s, tiles, total_out);
    return cudaGetLastError();
}

// ---- K7 ----------------------------------------------------------------------
__device__ __forceinline__ unsigned sort_bucket(const DevKeypoint& k, const SortGeom& g) {
    const int row = min(max((int)k.y, 0), g.rows - 1);   // (int) of y >= 0 = floor
    const int lvl = k.octave * g.s + (k.interval - 1);
    return (unsigned)k.image * g.per_image + (unsigned)(lvl * g.rows + row);
}

// strict "a before b" over the fields that can differ inside one bucket
__device__ __forceinline__ bool sort_less(const DevKeypoint& a, int ia, const DevKeypoint& b, int ib) {
    const unsigned a0 = __float_as_uint(a.y), b0 = __float_as_uint(b.y);
    if (a0 != b0) return a0 < b0;
    const unsigned a1 = __float_as_uint(a.x), b1 = __float_as_uint(b.x);
    if (a1 != b1) return a1 < b1;
    const unsigned a2 = __float_as_uint(a.angle), b2 = __float_as_uint(b.angle);
    if (a2 != b2) return a2 < b2;
    const unsigned a3 = __float_as_uint(a.sigma), b3 = __float_as_uint(b.sigma);
    if (a3 != b3) return a3 < b3;
    const unsigned a4 = __float_as_uint(a.response), b4 = __float_as_uint(b.response);
    if (a4 != b4) return a4 < b4;
    return ia < ib;   // full ties: identical bytes either way (descriptors are field-determined)
}

__global__ void sort_count_kernel(const DevKeypoint* __restrict__ kp, const unsigned long long* n_dev, SortGeom g,
                                  unsigned* __restrict__ bkt, unsigned* __restrict__ cnt) {
    const long long n = (long long)*n_dev;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned b = sort_bucket(kp[i], g);
        bkt[i] = b;
        atomicAdd(cnt + b, 1u);   // integer counts: order-free
    }
}

__global__ void sort_scatter_kernel(const unsigned long long* n_dev, const unsigned* __restrict__ bkt,
                                    const unsigned* __restrict__ start, unsigned* __restrict__ cnt,
                                    int* __restrict__ tmp) {
    const long long n = (long long)*n_dev;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned b = bkt[i];
        const unsigned pos = atomicSub(cnt + b, 1u) - 1u;   // any order; K7d fixes it
        tmp[start[b] + pos] = (int)i;
    }
}

__global__ void sort_rank_kernel(const DevKeypoint* __restrict__ kp, const unsigned long long* n_dev,
                                 const unsigned* __restrict__ bkt, const unsigned* __restrict__ start,
                                 const int* __restrict__ tmp, int* __restrict__ perm) {
    const long long n = (long long)*n_dev;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
        const int i = tmp[j];
        const unsigned b = bkt[i];
        const unsigned lo = start[b], hi = start[b + 1];
        unsigned rank = 0;
        if (hi - lo > 1) {
            const DevKeypoint me = kp[i];
            for (unsigned q = lo; q < hi; ++q) {
                const int m = tmp[q];
                if (m != i && sort_less(kp[m], m, me, i)) ++rank;
            }
        }
        perm[lo + rank] = i;
    }
}

__global__ void sort_gather_kernel(const DevKeypoint* __restrict__ in, const int* __restrict__ perm,
                                   const unsigned long long* n_dev, DevKeypoint* __restrict__ out,
                                   dsift_keypoint* __restrict__ out_pub, const unsigned* __restrict__ start,
                                   SortGeom g, int batch, long long* __restrict__ offsets) {
    const long long n = (long long)*n_dev;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (long long i = tid; i < n; i += (long long)gridDim.x * blockDim.x) {
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
    // offsets[b] = first slot of image b = start of its first bucket (b = batch: n)
    for (long long b = tid; b <= batch; b += (long long)gridDim.x * blockDim.x)
        offsets[b] = (long long)start[(size_t)b * g.per_image];
}

size_t sort_work_bytes(long long cap, const SortGeom& g, int batch) {
    const size_t nb = (size_t)batch * g.per_image + 1;
    const size_t a = (sizeof(unsigned) * (size_t)cap + 255) & ~size_t(255);          // bkt
    const size_t b = (sizeof(int) * 2 * (size_t)cap + 255) & ~size_t(255);           // tmp, perm
    const size_t c = (sizeof(unsigned) * 2 * nb + 255) & ~size_t(255);               // cnt, start
    return a + b + c + scan_state_bytes((long long)nb);
}

cudaError_t launch_canonical_sort(const DevKeypoint* in, const unsigned long long* n_dev, long long cap,
                                  const SortGeom& g, void* work, DevKeypoint* out, dsift_keypoint* out_pub,
                                  int batch, long long* offsets, cudaStream_t st, long long* launches) {
    const size_t nb = (size_t)batch * g.per_image;   // buckets; start[] has nb + 1 entries
    char* p = static_cast<char*>(work);
    unsigned* bkt = reinterpret_cast<unsigned*>(p);
    p += (sizeof(unsigned) * (size_t)cap + 255) & ~size_t(255);
    int* tmp = reinterpret_cast<int*>(p);
    int* perm = tmp + cap;
    p += (sizeof(int) * 2 * (size_t)cap + 255) & ~size_t(255);
    unsigned* cnt = reinterpret_cast<unsigned*>(p);
    unsigned* start = cnt + (nb + 1);
    p += (sizeof(unsigned) * 2 * (nb + 1) + 255) & ~size_t(255);
    void* scan_state = p;

    const int threads = 256;
    const int grid = (int)std::max<long long>(1, std::min<long long>((cap + threads - 1) / threads, 148 * 8));
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned) * (nb + 1), st);
    if (e != cudaSuccess) return e;
    sort_count_kernel<<<grid, threads, 0, st>>>(in, n_dev, g, bkt, cnt);
    e = launch_scan_u32(cnt, start, (long long)nb, scan_state, start + nb, st);
    if (e != cudaSuccess) return e;
    sort_scatter_kernel<<<grid, threads, 0, st>>>(n_dev, bkt, start, cnt, tmp);
    sort_rank_kernel<<<grid, threads, 0, st>>>(in, n_dev, bkt, start, tmp, perm);
    sort_gather_kernel<<<grid, threads, 0, st>>>(in, perm, n_dev, out, out_pub, start, g, batch, offsets);
    *launches += 5;
    return cudaGetLastError();
}

}  // namespace dsift
