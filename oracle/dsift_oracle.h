/* oracle/dsift_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference extraction path
 * (detsift::extract, /root/reference/proj/src/io.cpp:111-142) used as the CPU
 * parity checker for the CUDA product.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * Parity pinning: every function is checked bit-for-bit against the unmodified
 * reference compiled into oracle/_ref/libdetsift_ref.so (tests/test_oracle.py)
 * and against committed golden vectors in tests/golden/.
 */
#ifndef DSIFT_ORACLE_H
#define DSIFT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same layout as dsift_config (include/dsift.h) and detsift::SiftConfig fields. */
typedef struct {
    float sigma0;
    int32_t intervals;
    float assumed_blur;
    float contrast_threshold;
    float edge_ratio;
    int32_t max_refine_iters;
    int64_t upsample_pixel_limit;
    const double* dsp_scales;
    int32_t n_dsp_scales;
    float descriptor_clip;
    int32_t orientation_bins;
    float orientation_peak_ratio;
    int32_t num_octaves;
} dor_config;

/* detsift::Keypoint (core.hpp:55-63), 28 bytes. */
typedef struct {
    float x, y, sigma, angle, response;
    int32_t octave, interval;
} dor_keypoint;

typedef struct {
    int n_oct, s, upsampled;
    float sigma0;
    int32_t* w;      /* [n_oct] */
    int32_t* h;      /* [n_oct] */
    float** gauss;   /* [n_oct * (s+3)] */
    float** dog;     /* [n_oct * (s+2)] */
} dor_scale_space;

const char* dor_last_error(void);
void dor_config_default(dor_config* c, double* scales5);
int dor_config_validate(const dor_config* c);

int dor_gaussian_kernel(double sigma, float* out, int cap);
int dor_convolve(const float* img, int w, int h, const float* k, int len, float* out);
void dor_upsample2x(const float* img, int w, int h, float* out);
void dor_decimate2x(const float* img, int w, int h, float* out);

int dor_build_scale_space(const float* img, int w, int h, const dor_config* c,
                          dor_scale_space** out);
void dor_ss_free(dor_scale_space* ss);
void dor_ss_info(const dor_scale_space* ss, int32_t* n_oct, int32_t* upsampled, int32_t* dims);
void dor_ss_level(const dor_scale_space* ss, int o, int kind, int i, float* out);
dor_scale_space* dor_ss_from_levels(int n_oct, int s, float sigma0, int upsampled,
                                    const int32_t* dims, const float* const* gauss,
                                    const float* const* dog);

int64_t dor_find_extrema(const dor_scale_space* ss, const dor_config* c, int32_t* out5,
                         int64_t cap);
int dor_refine(const dor_scale_space* ss, const int32_t* e5, const dor_config* c,
               dor_keypoint* out);
int64_t dor_detect(const dor_scale_space* ss, const dor_config* c, dor_keypoint* out,
                   int64_t cap);

int dor_nearest_gauss_level(const dor_scale_space* ss, double sigma_rel);
int dor_orientation_histogram(const dor_scale_space* ss, const dor_keypoint* kp,
                              const dor_config* c, float* out);
int dor_assign_orientations(const dor_scale_space* ss, const dor_keypoint* kp,
                            const dor_config* c, dor_keypoint* out);

int dor_raw_descriptor(const dor_scale_space* ss, const dor_keypoint* kp, double f,
                       const dor_config* c, float* out);
int dor_dsp_descriptor(const dor_scale_space* ss, const dor_keypoint* kp, const dor_config* c,
                       float* out);
int dor_root_sift(float* v, int n);

/* Full pipeline; *kps / *desc are malloc'd (free with dor_free). */
int dor_extract(const float* img, int w, int h, const dor_config* c, dor_keypoint** kps,
                float** desc, int64_t* n);
void dor_free(void* p);
/* load_image (io.cpp:49-81): 0, or -2 with the std::runtime_error message. */
int dor_load_image(const char* path, int* w, int* h, float* out);
void dor_canonical_sort(dor_keypoint* kps, float* desc, int64_t n);
int64_t dor_serialize(const dor_keypoint* kps, const float* desc, int64_t n, uint8_t* out,
                      int64_t cap);
void dor_sha256(const uint8_t* p, int64_t n, char* hex65);
void dor_hash_features(const dor_keypoint* kps, const float* desc, int64_t n, char* hex65);

float dor_tree_sum(const float* v, int64_t n);
double dor_tree_sum_f64(const double* v, int64_t n);
int dor_tree_hist(const int32_t* bins, const float* w, int64_t n, int bin_count, float* out);

void dor_value_noise(int w, int h, uint64_t seed, int octaves, int cells, float* out);

#ifdef __cplusplus
}
#endif
#endif
