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

// Register-resident counter.  push() is a compile-time chain of nested
// branches (one per slot), so every slot index is static and the slots stay
// in registers (a runtime loop with `break` is not unrolled by ptxas and would
// spill the array to local memory).
template <int J, int DEPTH>
struct TreePushStep {
    __device__ __forceinline__ static void run(double (&node)[DEPTH], unsigned c, double x) {
        if (c & 1u) {
            TreePushStep<J + 1, DEPTH>::run(node, c >> 1, node[J] + x);
        } else {
            node[J] = x;
        }
    }
};
template <int DEPTH>
struct TreePushStep<DEPTH, DEPTH> {
    __device__ __forceinline__ static void run(double (&)[DEPTH], unsigned, double) {}
};
template <int J, int DEPTH>
struct TreeFoldStep {
    __device__ __forceinline__ static void run(const double (&node)[DEPTH], unsigned c, double& r, bool& have) {
        if (c & 1u) {
            r = have ? node[J] + r : node[J];
            have = true;
        }
        if (c >> 1) TreeFoldStep<J + 1, DEPTH>::run(node, c >> 1, r, have);
    }
};
template <int DEPTH>
struct TreeFoldStep<DEPTH, DEPTH> {
    __device__ __forceinline__ static void run(const double (&)[DEPTH], unsigned, double&, bool&) {}
};

template <int DEPTH>
struct TreeCounter {
    double node[DEPTH];
    unsigned count;

    __device__ __forceinline__ void reset() { count = 0; }
    __device__ __forceinline__ void push(double x) {
        TreePushStep<0, DEPTH>::run(node, count, x);
        ++count;
    }
    __device__ __forceinline__ double result() const {
        double r = 0.0;
        bool have = false;
        TreeFoldStep<0, DEPTH>::run(node, count, r, have);
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
