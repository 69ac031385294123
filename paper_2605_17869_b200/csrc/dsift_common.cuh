// dsift_common.cuh — device-side data layout shared by the kernels and the
// host orchestration (dsift_host.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dsift.h"

namespace dsift {

constexpr int kMaxOctaves = 24;
constexpr int kMaxLevels = 16;      // s + 3 <= kMaxLevels
constexpr int kMaxRadius = 64;      // largest Gaussian tap radius supported
constexpr int kDescCells = 4;       // describe.hpp:11
constexpr int kDescOrients = 8;     // describe.hpp:12
constexpr int kDescDim = 128;       // describe.hpp:13
constexpr int kMaxDsp = 16;         // dsp_scales entries
constexpr int kMaxOriBins = 64;     // orientation_bins supported on device
constexpr double kTwoPi = 6.283185307179586476925286766559;  // orient.cpp:37

// Test-only bounds checks (the DSIFT_BOUNDS_CHECK build, tests/native/
// libdsift_bounds.so; the product build compiles them away).  DSIFT_BOUND(c,
// site) counts a failed index condition in this translation unit's device
// counter and records the first failing site id; the host reads the counters
// through dsift_test_bounds_<unit>() (DSIFT_BOUNDS_UNIT).  The stand-in for
// compute-sanitizer memcheck, which the GPU pool refuses to run.
#ifdef DSIFT_BOUNDS_CHECK
#define DSIFT_BOUNDS_UNIT(unit)                                                           \
    static __device__ unsigned long long g_bounds[2];                                    \
    extern "C" int dsift_test_bounds_##unit(unsigned long long* out, int reset) {          \
        if (cudaMemcpyFromSymbol(out, g_bounds, sizeof(g_bounds)) != cudaSuccess) return -1; \
        if (reset) {                                                                      \
            const unsigned long long z[2] = {0ull, 0ull};                                 \
            if (cudaMemcpyToSymbol(g_bounds, z, sizeof(z)) != cudaSuccess) return -1;     \
        }                                                                                 \
        return 0;                                                                         \
    }
#define DSIFT_BOUND(cond, site)                                                           \
    do {                                                                                  \
        if (!(cond) && atomicAdd(&g_bounds[0], 1ull) == 0ull) g_bounds[1] = (site);       \
    } while (0)
#else
#define DSIFT_BOUNDS_UNIT(unit)
#define DSIFT_BOUND(cond, site) \
    do {                        \
    } while (0)
#endif

// Pyramid layout in HBM: for octave o, Gaussian levels are a dense array
// [batch][s+3][h_o][pitch_o] and DoG levels [batch][s+2][h_o][pitch_o]
// (pitch_o = w_o rounded up to 32 floats = 128 B so every row starts on a
// cache-line boundary).
struct OctaveDesc {
    int w, h, pitch;
    int tiles_x, tiles_y;      // extrema tiles
    long long level_stride;    // pitch * h
    float* gauss;              // [batch][s+3] levels
    float* dog;                // [batch][s+2] levels
};

struct PyramidDesc {
    int n_oct, s, batch, upsampled;
    float sigma0;
    OctaveDesc oct[kMaxOctaves];
    double level_sigma[kMaxLevels];   // sigma0 * 2^(i/s)   (scalespace.cpp:11-13)
    __host__ __device__ long long gauss_img_stride(int o) const { return (long long)(s + 3) * oct[o].level_stride; }
    __host__ __device__ long long dog_img_stride(int o) const { return (long long)(s + 2) * oct[o].level_stride; }
};

// Keypoint as it travels between device stages (32 B).  `image` is the batch
// index; `src` packs the originating candidate (octave, interval, row, col)
// so stage-level APIs can restore the reference's candidate order.
struct DevKeypoint {
    float x, y, sigma, angle, response;
    int32_t octave, interval;
    int32_t image;
};

struct DevCandidate {   // raw extremum (detect.hpp:12-18)
    int32_t image, octave, interval, row, col, is_max;
};

// Per-launch error word bits (OR-ed on device, checked at sync).
enum : unsigned {
    kErrKeypointCapacity = 1u,
    kErrOrientedCapacity = 2u,
    kErrCandidateCapacity = 4u,
    kErrDescriptorLattice = 8u,
    kErrHistogramRange = 16u,   // NaN gradient -> out-of-range bin (detsum.cpp:138-141 throws)
};

// Decoupled look-back scan state (per ticket): bit 63..62 = status.
constexpr unsigned long long kLbAggregate = 1ull << 62;
constexpr unsigned long long kLbPrefix = 2ull << 62;
constexpr unsigned long long kLbValueMask = (1ull << 62) - 1;

struct ScanState {
    unsigned long long* states;   // [n_tiles]
    unsigned int* ticket;         // dynamic tile ticket
    unsigned long long* total;    // inclusive total (written by the last tile), clamped to cap
    unsigned long long cap;       // capacity of the compacted output
};

struct Counters {          // one small device block, cleared per batch
    unsigned long long n_det;
    unsigned long long n_ori;
    unsigned err;
    unsigned det_ticket;
    unsigned ori_ticket;
    unsigned n_slow;      // keypoints the certified fast descriptor path handed to the exact kernel
    unsigned ref_ticket;
    unsigned n_fixed;     // (keypoint, scale) pairs the stream kernel recomputed exactly in place
    unsigned long long n_kp;   // refined keypoints (compacted)
    unsigned emit_ticket;      // orientation fan-out tiles
    unsigned desc_ticket;      // describe: dynamic keypoint claims
    unsigned long long lattice;     // describe: lattice points sum (2r+1)^2 (work unit)
    unsigned long long lattice_in;  // describe: of those, inside the (-1, 4)-bin square (visited)
};

// Per-result device totals: every size group's counters are folded in here
// (OR of the error words, sum of the exact-fallback counts).
struct BatchTotals {
    unsigned err;
    unsigned pad;
    unsigned long long slow;
    unsigned long long lattice;
    unsigned long long lattice_in;
};

}  // namespace dsift
