// dsift_kernels.cuh — launch-argument structs and launcher entry points of
// the device stages (one definition shared by k_*.cu and dsift_host.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "dsift_common.cuh"

namespace dsift {

enum BlurMode : int { kModeLevel = 0, kModeRaw = 1, kModeUpsample = 2, kModeDecimate = 3 };

struct BlurArgs {
    const float* src;
    long long src_img_stride;
    int src_pitch, src_w, src_h;
    float* dst;
    long long dst_img_stride;
    float* dog;
    long long dog_img_stride;
    float* seed;
    long long seed_img_stride;
    int w, h, pitch;
    double taps[2 * kMaxRadius + 1];
    // strip kernel: TMA map of the source level (3-D {w, h, batch}, box {kInW, 32, 1};
    // DECIMATE: element stride 2 over the previous octave's level), valid iff use_tma
    CUtensorMap src_map;
    int use_tma;
    const int* src_flag;   // nonzero: a source value is not a positive normal >= 2^-100 (null: unknown)
    int* dst_flag;         // producer: set nonzero when an output is not one
};
// TMA box width (floats) of the strip kernel's source map for radius R (host side)
int blur_strip_box_w(int R);
cudaError_t launch_blur(const BlurArgs& a, int mode, int R, int batch, cudaStream_t st);

// fused small octaves o_first..n_oct-1 (one CTA per image, levels in shared memory)
constexpr int kSmallMaxLevels = kMaxLevels;
struct SmallOctArgs {
    PyramidDesc pyr;
    int o_first;
    int cap_px;                                // w * h of octave o_first (the largest fused level)
    int radius[kSmallMaxLevels];               // incremental blur i+1: radius
    double taps[kSmallMaxLevels][33];          // and taps (radius <= 16)
};
size_t small_octaves_smem(int cap_px);
cudaError_t launch_small_octaves(const SmallOctArgs& a, cudaStream_t st);

struct DetectArgs {
    PyramidDesc pyr;
    int tiles_per_image;
    int oct_tile_base[kMaxOctaves + 1];
    unsigned n_tiles;
    float pre_gate;
    double contrast_gate;
    double edge_r;
    int max_iters;
    int raw_mode;
    DevKeypoint* out;
    DevCandidate* cand_out;
    long long cap;
    unsigned* err;
    ScanState scan;
    // count -> scan -> emit compaction of the extrema (no cross-tile waiting)
    unsigned* hit_masks;         // [n_tiles][256] per-thread (level, row) hit bits (s <= 8)
    unsigned* tile_counts;       // [n_tiles]
    unsigned* tile_offsets;      // [n_tiles] exclusive scan of tile_counts
    void* scan_state;            // launch_scan_u32 scratch
    // TMA: per-octave 3-D maps of the DoG stack {w, h, batch * (s+2)}, passed
    // by value in the __grid_constant__ parameter block (no global-memory
    // descriptor, so no tensormap proxy fence is needed); octave o is staged
    // by TMA iff bit o is set
    unsigned tma_mask;
    CUtensorMap dog_maps[kMaxOctaves];
};
cudaError_t launch_detect(const DetectArgs& a, cudaStream_t st);
cudaError_t launch_refine(const DetectArgs& a, const DevCandidate* cand, const unsigned long long* n_cand,
                          long long cap, int* keep, cudaStream_t st);

struct OrientArgs {
    PyramidDesc pyr;
    const DevKeypoint* kps;
    const unsigned long long* n_dev;
    long long n_host;
    int bins;
    float peak_ratio;
    int depth;
    DevKeypoint* out;
    long long cap;
    unsigned* err;
    float* hist_out;
    ScanState scan;        // K4a: work tickets only
    unsigned n_tiles;
    float* angles;         // [cap_kp][bins] peak angles per keypoint (K4a -> K4b)
    int* counts;           // [cap_kp] oriented copies per keypoint
    ScanState emit_scan;   // K4b: fan-out compaction in keypoint order
};
cudaError_t launch_orient(const OrientArgs& a, cudaStream_t st);
int orient_tile_size();

struct DescArgs {
    PyramidDesc pyr;
    const unsigned long long* gauss_tex;   // [image][kMaxOctaves] texture objects of the Gaussian levels (nullable)
    const DevKeypoint* kps;
    const unsigned long long* n_dev;
    long long n_host;
    double dsp[kMaxDsp];
    int n_dsp;
    float clip;
    int raw_mode;
    double raw_scale;
    int max_axis;
    int chunk_rows;
    int tree_depth;        // levels of the per-bin binary counter: 2^tree_depth > leaves per bin
    const double2* trig;   // [n] (cos, sin) of the angle
    const int* slow_list;  // exact kernel: process only these keypoints (nullable)
    const unsigned* n_slow;
    int* slow_out;         // fast kernel: keypoints it could not certify
    unsigned* slow_count;
    unsigned* fix_count;   // stream kernel: (keypoint, scale) pairs recomputed exactly in place
    unsigned* ticket;      // stream kernel: next keypoint to claim (zeroed before the launch)
    unsigned long long* lattice;   // stream kernel: += (2r+1)^2 lattice points per (keypoint, scale)
    unsigned long long* lattice_in;   // stream kernel: += of those in the (-1, 4)-bin square
    long long slow_cap;
    int force_slow;        // test hook (DSIFT_OPT_FORCE_EXACT): fail every certificate
    int max_span;          // stream kernel: table/ring width bound (in-range span + guards)
    int nondet;            // negative-control build only (DSIFT_NONDET_TEST_HOOK + env DSIFT_NONDET=1):
                           // order-fragile float atomics instead of the fixed trees
    float* desc;
    unsigned char* desc_u8;
    unsigned* err;
};
cudaError_t launch_describe(const DescArgs& a, int grid, cudaStream_t st);
size_t describe_smem_bytes(int max_axis, int chunk_rows, int n_dsp, int tree_depth);

// K7 bucket geometry: bucket = image * per_image + (octave * s + interval - 1) * rows + floor(y)
struct SortGeom {
    int s;              // intervals per octave
    int rows;           // input image height (keypoint y is in input coordinates)
    unsigned per_image; // n_oct * s * rows
};
size_t sort_work_bytes(long long cap, const SortGeom& g, int batch);
cudaError_t launch_canonical_sort(const DevKeypoint* in, const unsigned long long* n_dev, long long cap,
                                  const SortGeom& g, void* work, DevKeypoint* out, dsift_keypoint* out_pub,
                                  int batch, long long* offsets, cudaStream_t st, long long* launches);
// device-wide exclusive scan of n uint32 (single pass, decoupled look-back);
// state = scan_state_bytes(n) of scratch; *total_out (optional) = the sum
size_t scan_state_bytes(long long n);
cudaError_t launch_scan_u32(const unsigned* in, unsigned* out, long long n, void* state, unsigned* total_out,
                            cudaStream_t st);
cudaError_t launch_value_noise(float* out, int n, int w, int h, unsigned long long seed0, int octaves,
                               int cells, double* scratch, int nparts, cudaStream_t st);

size_t describe_stream_smem_bytes(int max_span, int n_dsp);
size_t describe_stream_exact_smem_bytes(int max_axis, int chunk_rows, int n_dsp, int tree_depth);
int describe_stream_blocks_per_sm(size_t smem);
cudaError_t launch_describe_stream(const DescArgs& a, int grid, cudaStream_t st);
cudaError_t launch_trig(const DevKeypoint* kps, const unsigned long long* n_dev, long long n_host, double2* trig,
                        long long cap, cudaStream_t st);

// k_batch.cu: result bookkeeping.  Folds a group's counters into the
// result's totals; gathers a ragged batch's per-group staged outputs into
// batch order (map = per image: staging-offsets entry, staging row base).
cudaError_t launch_fold_totals(const Counters* ctr, BatchTotals* tot, cudaStream_t st);
cudaError_t launch_ragged_gather(const long long* map, const long long* stage_offs, int n,
                                 const dsift_keypoint* skp, const float* sdesc, const unsigned char* su8,
                                 long long* offsets, dsift_keypoint* kp, float* desc, unsigned char* u8,
                                 cudaStream_t st);

size_t match_scratch_bytes(long long na, long long nb);
// k_geom.cu: m = n x 4 doubles (x1, y1, x2, y2)
size_t magsac_scratch_bytes(long long n, int iters);
cudaError_t launch_magsac(const double* m, long long n, const int4* samples, int iters, double tau_sq, void* scratch,
                          unsigned char* mask, int* out_i, double* out_d, cudaStream_t st);
size_t dlt_scratch_bytes(long long n);
cudaError_t launch_dlt(const double* m, const double* w, int n, void* scratch, int* status, double* out,
                       cudaStream_t st);
cudaError_t launch_ratio_match(const float* A, long long na, const float* B, long long nb, float ratio, void* scratch,
                               int* best_a, int* best_b, float* dist_a, cudaStream_t st);
cudaError_t launch_ingest_u8(const unsigned char* in, long long n_px, int channels, float* out, cudaStream_t st);

}  // namespace dsift
