/* include/dsift.h — C ABI of the B200-native SIFT extraction path.
 *
 * Drop-in boundary for detsift::extract (reference:
 * /root/reference/proj/include/detsift/io.hpp:17-19, src/io.cpp:111-142) and
 * for the stage-level functions the reference's tests and oracles call
 * directly (scalespace.hpp:30-47, detect.hpp:23-33, orient.hpp:12-25,
 * describe.hpp:19-30, core.hpp:83-91, detsum.hpp:22-48).
 *
 * Plain C: pointers, sizes and status codes only; no exceptions and no torch
 * types cross this boundary.  Every entry point returns DSIFT_OK (0) or a
 * positive DSIFT_E* code; dsift_last_error() then holds the message (for
 * DSIFT_EINVAL it is the reference's std::invalid_argument text).
 *
 * Threading: one dsift_ctx per (device, host thread); all device work of a
 * context is ordered on its CUDA stream (host inputs are copied on a second
 * stream so they overlap the previous batch).  Results stay on the device
 * until copied or exported; a result is owned by its dsift_result (the
 * context's own one by default) until the next extract into it.
 */
#ifndef DSIFT_H
#define DSIFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSIFT_ABI_VERSION 2

enum {
    DSIFT_OK = 0,
    DSIFT_EINVAL = 1,    /* std::invalid_argument in the reference            */
    DSIFT_ECAPACITY = 2, /* a device work list overflowed; nothing truncated  */
    DSIFT_ECUDA = 3,     /* CUDA runtime error / no device / extension absent */
    DSIFT_ENOMEM = 4,    /* device or host allocation failed                  */
    DSIFT_ESTATE = 5,    /* call order violated (e.g. no result yet)          */
    DSIFT_ERANGE = 6,    /* std::out_of_range in the reference (NaN input)   */
    DSIFT_EIO = 7,       /* std::runtime_error in the reference (image I/O)  */
    DSIFT_EGEOM = 8      /* std::runtime_error in the reference (geometry:
                            degenerate DLT, point at infinity)               */
};

/* detsift::SiftConfig (core.hpp:30-47).  dsp_scales is borrowed by the call. */
typedef struct dsift_config {
    float sigma0;
    int32_t intervals;           /* intervals_per_octave (s)     */
    float assumed_blur;          /* assumed_input_blur           */
    float contrast_threshold;
    float edge_ratio;
    int32_t max_refine_iters;
    int64_t upsample_pixel_limit;
    const double* dsp_scales;
    int32_t n_dsp_scales;
    float descriptor_clip;
    int32_t orientation_bins;
    float orientation_peak_ratio;
    int32_t num_octaves;         /* 0 = auto                      */
} dsift_config;

/* detsift::Keypoint (core.hpp:55-63), 28 bytes, identical layout. */
typedef struct dsift_keypoint {
    float x, y, sigma, angle, response;
    int32_t octave, interval;
} dsift_keypoint;

typedef struct dsift_ctx dsift_ctx;
/* A batch result (keypoints, descriptors, offsets) with its own completion
 * event.  Every context has a built-in one; dsift_result_create adds more so
 * several batches can be in flight on one context. */
typedef struct dsift_result dsift_result;

/* detsift::GrayImage (core.hpp:11-26) as a view: row-major float32
 * width x height, values in [0, 1], on the host or the device (per flags). */
typedef struct dsift_image {
    const float* data;
    int32_t width, height;
} dsift_image;

/* input flags */
#define DSIFT_INPUT_HOST 0
#define DSIFT_INPUT_DEVICE 1

/* ---- library ------------------------------------------------------------ */
int dsift_abi_version(void);
const char* dsift_strerror(int code);
const char* dsift_last_error(void);
/* Fills the reference defaults (core.hpp:31-43); dsp_scales points at a
 * static 5-entry array owned by the library. */
void dsift_config_default(dsift_config* cfg);
/* SiftConfig::validate (core.cpp:17-46): DSIFT_EINVAL + reference message. */
int dsift_config_validate(const dsift_config* cfg);

/* ---- context ------------------------------------------------------------ */
/* Creates a context on `device` (cudaSetDevice semantics).  The config is
 * validated and copied. */
int dsift_create(int device, const dsift_config* cfg, dsift_ctx** out);
void dsift_destroy(dsift_ctx* ctx);
/* Use the caller's cudaStream_t (NULL restores the context's own stream). */
int dsift_set_stream(dsift_ctx* ctx, void* cuda_stream);
/* Per-image capacity of the keypoint work lists.  0 = automatic: sized from
 * the image, grown x4 and the batch replayed inside dsift_result_sync if a
 * list overflows (so every keypoint is still returned).  A fixed capacity
 * reports an overflow as DSIFT_ECAPACITY, never truncated output. */
int dsift_set_capacity(dsift_ctx* ctx, int64_t max_keypoints_per_image);

/* ---- full pipeline: detsift::extract (io.cpp:111-142) --------------------- */
/* `n` same-size images, row-major float32 [n][h][w], values in [0,1], on the
 * host (DSIFT_INPUT_HOST, copied H2D inside the call) or the device.  Work is
 * enqueued on the context stream; dsift_result_sync waits for it.  Output is
 * per image in canonical order (core.cpp:116-170). */
int dsift_extract_batch(dsift_ctx* ctx, const float* images, int n, int w, int h, int flags);
int dsift_extract(dsift_ctx* ctx, const float* image, int w, int h, int flags);
/* Ragged batch: n images of any sizes (the reference's extract takes any size
 * per call, io.cpp:111-142).  Same-size images are processed together; the
 * output is in batch order, image i's features bit-identical to a
 * single-image extract of it.  Device inputs must stay valid until
 * dsift_result_sync returns (a capacity overflow replays the batch). */
int dsift_extract_images(dsift_ctx* ctx, const dsift_image* images, int n, int flags);
/* Result handles.  dsift_result_select(ctx, r) routes the following extract
 * and dsift_result_* calls of ctx to r (NULL = the context's own result), so
 * a serving loop keeps batch k+1 running while it reads batch k out.  A
 * result must be destroyed before its context. */
int dsift_result_create(dsift_ctx* ctx, dsift_result** out);
void dsift_result_destroy(dsift_result* result);
int dsift_result_select(dsift_ctx* ctx, dsift_result* result);
/* 8-bit ingest (replaces load_image's float conversion, io.cpp:49-81): n
 * images of w x h pixels with channels = 1 (P5 gray) or 3 (P6 RGB,
 * interleaved), host or device (flags).  The bytes are converted on the
 * device with the reference's double arithmetic, then extracted exactly like
 * dsift_extract_batch on the resulting GrayImages. */
int dsift_extract_batch_u8(dsift_ctx* ctx, const uint8_t* pixels, int n, int w, int h, int channels,
                           int flags);
/* ---- matching ---------------------------------------------- */
/* detsift::Match (match.hpp:14-18). */
typedef struct dsift_match {
    int32_t a, b;
    float distance;
} dsift_match;
/* detsift::ratio_match (match.hpp:34-38, match.cpp:77-119): symmetric ratio
 * test with mutual-consistency filtering over two descriptor sets (row-major
 * n x dim float32, host or device per flags), bit-identical distances (fixed
 * tree dot products).  Pairs come sorted by a; *n_pairs may exceed cap (then
 * only cap are written).  This build supports dim = 128. */
int dsift_ratio_match(dsift_ctx* ctx, const float* desc_a, int64_t n_a, const float* desc_b, int64_t n_b,
                      int dim_a, int dim_b, float ratio, int flags, dsift_match* out, int64_t cap,
                      int64_t* n_pairs, int64_t* putative_a, int64_t* putative_b);
/* ---- robust homography ------------------------------------ */
/* detsift::MagsacResult (geom.hpp:55-61) without the mask vector. */
typedef struct dsift_magsac_result {
    int32_t success;
    int32_t best_iteration; /* -1 when no hypothesis was valid            */
    double score;           /* winning hypothesis score (0 on failure)    */
    double h[9];            /* refit model, row-major (identity on failure) */
} dsift_magsac_result;
/* detsift::magsac_lite (geom.hpp:63-67, geom.cpp:181-320): seeded hypotheses
 * (host SplitMix64 stream, as the reference draws them), minimal-sample DLT,
 * soft truncated-quadratic scores (detsum tree) and the weighted refit on the
 * device; bit-identical to the reference.  matches: host n x 4 doubles
 * (x1, y1, x2, y2) = detsift::Correspondence.  inlier_mask (n bytes, may be
 * NULL) is all zero on failure.  DSIFT_EINVAL for the reference's
 * std::invalid_argument cases (n < 4, tau <= 0, iterations < 1). */
int dsift_magsac_lite(dsift_ctx* ctx, const double* matches, int64_t n, int32_t iterations, double tau,
                      uint64_t seed, dsift_magsac_result* result, uint8_t* inlier_mask);
/* detsift::dlt_homography (geom.hpp:47-52, geom.cpp:108-161): normalized DLT
 * on the device, optional per-correspondence weights (NULL = 1).  DSIFT_EGEOM
 * where the reference throws std::runtime_error (degenerate / non-finite). */
int dsift_dlt_homography(dsift_ctx* ctx, const double* matches, int64_t n, const double* weights, double* h_out);
/* detsift::corner_error (geom.hpp:69-71, geom.cpp:322-333); DSIFT_EGEOM if a
 * corner maps to infinity. */
int dsift_corner_error(const double* h_est, const double* h_gt, double width, double height, double* out);
/* Reads a binary PNM (P5/P6, maxval 255) like detsift::load_image
 * (io.cpp:49-81), with its error messages (DSIFT_EIO).  Pass pixels = NULL to
 * query w, h, channels; otherwise pixels must hold w*h*channels bytes
 * (capacity in bytes). */
int dsift_load_image(const char* path, int32_t* w, int32_t* h, int32_t* channels, uint8_t* pixels,
                     int64_t capacity);
/* The float GrayImage load_image returns: n_px pixels of the given channel
 * count converted on the device (dev_out must be a device pointer). */
int dsift_ingest_u8(dsift_ctx* ctx, const uint8_t* pixels, int64_t n_px, int channels, int flags,
                    float* dev_out);
/* dsift_result_* act on the selected result (dsift_result_select).
 * Waits for the last extract; *total = keypoints over all images. */
int dsift_result_sync(dsift_ctx* ctx, int64_t* total);
/* [begin, begin+count) of `image` inside the batch result (after sync). */
int dsift_result_range(dsift_ctx* ctx, int image, int64_t* begin, int64_t* count);
/* Host copies of the whole batch result (any pointer may be NULL):
 * kps [total], desc [total][128] float32, desc_u8 [total][128] (q(v) =
 * min(255, lround(v * 255.0))), offsets [n+1]. */
int dsift_result_copy(dsift_ctx* ctx, dsift_keypoint* kps, float* desc, uint8_t* desc_u8,
                      int64_t* offsets);
/* Device pointers (valid until the next extract / destroy), no copy. */
int dsift_result_device(dsift_ctx* ctx, const dsift_keypoint** kps, const float** desc,
                        const uint8_t** desc_u8, const int64_t** offsets);
/* Zero-copy DLPack export of the batch result: which = 0 keypoints (float32
 * [total][7] view, octave/interval reinterpreted), 1 desc f32 [total][128],
 * 2 desc u8 [total][128].  Returns a DLManagedTensor* (see dlpack.h); its
 * deleter keeps the context buffer alive until called. */
#define DSIFT_EXPORT_KEYPOINTS 0
#define DSIFT_EXPORT_DESC_F32 1
#define DSIFT_EXPORT_DESC_U8 2
int dsift_export_dlpack(dsift_ctx* ctx, int which, void** dl_managed_tensor);
/* SHA-256 of the DSF1 serialization of image `image` of the last result
 * (detsum.cpp:129-132, core.cpp:153-196), computed on the host. */
int dsift_result_sha256(dsift_ctx* ctx, int image, char hex65[65]);

/* ---- stage level (scalespace.hpp / detect.hpp / orient.hpp / describe.hpp) */
/* build_scale_space (scalespace.cpp:144-214) for one image, kept in ctx. */
int dsift_build_scale_space(dsift_ctx* ctx, const float* image, int w, int h, int flags);
/* Handcrafted scale space (as tests/test_detect.cpp:14-30 builds): gauss
 * [n_oct*(s+3)] and dog [n_oct*(s+2)] host planes of dims[2*o] x dims[2*o+1]. */
int dsift_load_scale_space(dsift_ctx* ctx, int n_oct, int upsampled, const int32_t* dims,
                           const float* const* gauss, const float* const* dog);
int dsift_scale_space_info(dsift_ctx* ctx, int32_t* n_oct, int32_t* upsampled, int32_t* dims);
/* kind 0 = gauss level, 1 = DoG level; copies [h][w] float32 to host. */
int dsift_scale_space_level(dsift_ctx* ctx, int octave, int kind, int level, float* out);
/* find_extrema (detect.cpp:32-71): n x 5 int32 (octave, interval, row, col,
 * is_max), in canonical (octave, interval, row, col) order. */
int dsift_find_extrema(dsift_ctx* ctx, int32_t* out5, int64_t cap, int64_t* n);
/* detect_keypoints (detect.cpp:158-172): refined keypoints in candidate order. */
int dsift_detect(dsift_ctx* ctx, dsift_keypoint* out, int64_t cap, int64_t* n);
/* orientation_histogram (orient.cpp:26-60) for n host keypoints: [n][bins]. */
int dsift_orientation_histograms(dsift_ctx* ctx, const dsift_keypoint* kps, int64_t n,
                                 float* out);
/* assign_orientations (orient.cpp:77-113), flattened in keypoint order. */
int dsift_assign_orientations(dsift_ctx* ctx, const dsift_keypoint* kps, int64_t n,
                              dsift_keypoint* out, int64_t cap, int64_t* n_out);
/* raw_descriptor (describe.cpp:33-127) at one support scale: [n][128]. */
int dsift_raw_descriptors(dsift_ctx* ctx, const dsift_keypoint* kps, int64_t n,
                          double scale_factor, float* out);
/* dsp_descriptor (describe.cpp:148-173): [n][128] float32 (+ optional u8). */
int dsift_dsp_descriptors(dsift_ctx* ctx, const dsift_keypoint* kps, int64_t n, float* out,
                          uint8_t* out_u8);

/* ---- synthetic input (tests/support/synth.cpp:14-66) on the device -------- */
/* n images of value noise, image i uses seed0 + i; writes device [n][h][w]. */
int dsift_synth_value_noise(dsift_ctx* ctx, float* dev_out, int n, int w, int h,
                            uint64_t seed0, int octaves, int base_cells);

/* ---- accounting -------------------------------------------------------------- */
/* Number of kernel launches the context has issued since creation. */
int64_t dsift_kernel_launches(dsift_ctx* ctx);
/* Stage timing with CUDA events on the context stream (bench/profiling):
 * ms5 = {input+pyramid, extrema+refine, orientation, canonical sort,
 * descriptors} of the last extract. */
int dsift_set_profiling(dsift_ctx* ctx, int on);
/* Options: DSIFT_OPT_FORCE_EXACT = 1 routes every descriptor through the
 * exact scan-order kernel (test hook for the certified fast path); 0 or 1. */
#define DSIFT_OPT_FORCE_EXACT 1
/* DSIFT_OPT_CAPACITY_SCALE: scale of the automatic work-list capacities in
 * 1/1000 (default 1000; an overflow multiplies it by 4 and replays). */
#define DSIFT_OPT_CAPACITY_SCALE 2
/* DSIFT_OPT_TEXTURE_GATHERS: 1 (default) reads the descriptor's bilinear
 * footprints with texture gathers, 0 with plain loads (the path used when a
 * level stack exceeds the texture limits); identical results either way. */
#define DSIFT_OPT_TEXTURE_GATHERS 3
int dsift_set_option(dsift_ctx* ctx, int key, int64_t value);
/* Statistics of the last synced result: DSIFT_STAT_EXACT_FALLBACKS = number
 * of keypoints whose descriptor the fast path could not certify. */
#define DSIFT_STAT_EXACT_FALLBACKS 1
/* DSIFT_STAT_REPLAYS = times the last result was replayed after an automatic
 * capacity overflow. */
#define DSIFT_STAT_REPLAYS 2
/* DSIFT_STAT_LATTICE_POINTS = descriptor lattice points of the last result,
 * sum over keypoints and DSP scales of (2r+1)^2 (the trip count of
 * describe.cpp:76-77), counted on the device; DSIFT_STAT_LATTICE_IN_RANGE =
 * those inside the (-1, 4)-bin square, the points that contribute. */
#define DSIFT_STAT_LATTICE_POINTS 3
#define DSIFT_STAT_LATTICE_IN_RANGE 4
int64_t dsift_stat(dsift_ctx* ctx, int key);
int dsift_stage_times(dsift_ctx* ctx, float* ms5);

#ifdef __cplusplus
}
#endif
#endif /* DSIFT_H */
