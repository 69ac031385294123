// dsift_scan.cuh — deterministic single-pass compaction (decoupled look-back).
//
// Tiles take a dynamic ticket (so every predecessor of a running tile has
// already started), publish their element count, and derive their exclusive
// output offset from predecessors' published aggregates/prefixes.  The output
// order is the ticket -> region mapping, never the scheduling order, so the
// compacted arrays are bit-identical run to run with no atomics on order.
#pragma once
#include "dsift_common.cuh"

namespace dsift {

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Block-wide: obtain this CTA's ticket (all threads).
__device__ __forceinline__ unsigned scan_ticket(const ScanState& st, unsigned* slot) {
    if (threadIdx.x == 0) *slot = atomicAdd(st.ticket, 1u);
    __syncthreads();
    return *slot;
}

// Block-wide: given this tile's element count (valid in thread 0), return the
// exclusive offset of the tile (all threads).  n_tiles lets the last tile
// publish the grand total.  Warp 0 looks back 32 predecessors at a time: each
// lane waits for one predecessor's state, the nearest published prefix ends
// the walk, and the aggregates in front of it are warp-summed (integer sums:
// order-free, so the result is deterministic).
__device__ __forceinline__ unsigned long long scan_exclusive(const ScanState& st, unsigned ticket,
                                                             unsigned long long count,
                                                             unsigned n_tiles,
                                                             unsigned long long* slot) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        count = __shfl_sync(0xffffffffu, count, 0);
        unsigned long long excl = 0;
        if (ticket == 0) {
            if (lane == 0) st_release_u64(&st.states[0], kLbPrefix | count);
        } else {
            if (lane == 0) st_release_u64(&st.states[ticket], kLbAggregate | count);
            long long j0 = (long long)ticket - 1;
            while (true) {
                const long long j = j0 - lane;
                unsigned long long s = kLbPrefix;   // before tile 0: an empty prefix
                if (j >= 0) {
                    do {
                        s = ld_acquire_u64(&st.states[j]);
                    } while ((s >> 62) == 0);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                const int last = pm ? __ffs(pm) - 1 : 31;   // nearest prefix, or the whole window
                unsigned long long v = lane <= last ? (s & kLbValueMask) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
                excl += v;
                if (pm) break;
                j0 -= 32;
            }
            if (lane == 0) st_release_u64(&st.states[ticket], kLbPrefix | (excl + count));
        }
        if (lane == 0) {
            // downstream stages read this count: never let it exceed what was written
            if (ticket == n_tiles - 1) *st.total = min(excl + count, st.cap);
            *slot = excl;
        }
    }
    __syncthreads();
    return *slot;
}

}  // namespace dsift
