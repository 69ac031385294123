// dsift_tree.cuh — the reference's fixed reduction tree (detsum.cpp:13-71)
// as a streaming binary counter.
//
// detsum::tree_sum folds leaf pairs (2j, 2j+1) level by level in double,
// promoting an odd tail, in 1024-leaf blocks that compose into the same tree.
// That tree is exactly the one a binary counter builds while leaves arrive in
// order: slot j holds the pending sum of an aligned 2^j-leaf block, a new leaf
// merges with every full slot below its first zero bit, and the pending slots
// are folded smallest-first at the end.  Because the tree shape is a function
// of the leaf index only, any producer that feeds a bin's leaves in canonical
// order reproduces tree_accumulate_histogram (detsum.cpp:135-177) bit-exactly.
#pragma once

namespace dsift {

// Register-resident counter (slots statically indexed -> no local memory).
template <int DEPTH>
struct TreeCounter {
    double node[DEPTH];
    unsigned count;

    __device__ __forceinline__ void reset() { count = 0; }

    __device__ __forceinline__ void push(double x) {
        const unsigned c = count;
#pragma unroll
        for (int j = 0; j < DEPTH; ++j) {
            if ((c >> j) & 1u) {
                x = node[j] + x;
            } else {
                node[j] = x;
                break;
            }
        }
        count = c + 1;
    }

    __device__ __forceinline__ double result() const {
        double r = 0.0;
        bool have = false;
#pragma unroll
        for (int j = 0; j < DEPTH; ++j) {
            if ((count >> j) & 1u) {
                r = have ? node[j] + r : node[j];
                have = true;
            }
        }
        return r;
    }
};

// Shared-memory variant for counters indexed at run time.
__device__ __forceinline__ void tree_push_smem(double* node, unsigned* count, double x) {
    unsigned c = *count;
    int j = 0;
    while (c & 1u) {
        x = node[j] + x;
        c >>= 1;
        ++j;
    }
    node[j] = x;
    *count += 1;
}

__device__ __forceinline__ double tree_result_smem(const double* node, unsigned count) {
    double r = 0.0;
    bool have = false;
    for (int j = 0; count >> j; ++j) {
        if ((count >> j) & 1u) {
            r = have ? node[j] + r : node[j];
            have = true;
        }
    }
    return r;
}

}  // namespace dsift
