// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile with the
// reference's own Release flags: -std=gnu++20 -O3 -DNDEBUG, no -march, no
// fast-math).  The output lands in oracle/_ref/libdetsift_ref.so and is used by
// tests/ (parity checker) and by bench.py's cpu_baseline / --impl reference leg.
//
// Nothing here re-implements reference math: every function forwards to the
// reference entry point cited beside it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <stdexcept>
#include <memory>
#include <string>
#include <vector>

#include "detsift/core.hpp"
#include "detsift/describe.hpp"
#include "detsift/detect.hpp"
#include "detsift/detsum.hpp"
#include "detsift/geom.hpp"
#include "detsift/io.hpp"
#include "detsift/match.hpp"
#include "detsift/orient.hpp"
#include "detsift/scalespace.hpp"
#include "support/oracles.hpp"
#include "support/synth.hpp"

using namespace detsift;

extern "C" {

// Layout-identical to dsift_config in include/dsift.h (checked by tests).
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
} oref_config;

}  // extern "C"

namespace {

thread_local std::string g_err;

SiftConfig to_cfg(const oref_config* c) {
    SiftConfig cfg;
    if (!c) return cfg;
    cfg.sigma0 = c->sigma0;
    cfg.intervals_per_octave = c->intervals;
    cfg.assumed_input_blur = c->assumed_blur;
    cfg.contrast_threshold = c->contrast_threshold;
    cfg.edge_ratio = c->edge_ratio;
    cfg.max_refine_iters = c->max_refine_iters;
    cfg.upsample_pixel_limit = c->upsample_pixel_limit;
    if (c->dsp_scales && c->n_dsp_scales > 0)
        cfg.dsp_scales.assign(c->dsp_scales, c->dsp_scales + c->n_dsp_scales);
    else
        cfg.dsp_scales.clear();
    cfg.descriptor_clip = c->descriptor_clip;
    cfg.orientation_bins = c->orientation_bins;
    cfg.orientation_peak_ratio = c->orientation_peak_ratio;
    cfg.num_octaves = c->num_octaves;
    return cfg;
}

GrayImage to_img(const float* p, int w, int h) {
    GrayImage img;
    img.width = w;
    img.height = h;
    if (w > 0 && h > 0) img.data.assign(p, p + size_t(w) * h);
    return img;
}

template <typename F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}

}  // namespace

extern "C" {

const char* oref_last_error() { return g_err.c_str(); }

void oref_config_default(oref_config* c, double* scales5) {
    SiftConfig d;
    c->sigma0 = d.sigma0;
    c->intervals = d.intervals_per_octave;
    c->assumed_blur = d.assumed_input_blur;
    c->contrast_threshold = d.contrast_threshold;
    c->edge_ratio = d.edge_ratio;
    c->max_refine_iters = d.max_refine_iters;
    c->upsample_pixel_limit = d.upsample_pixel_limit;
    for (size_t i = 0; i < d.dsp_scales.size() && i < 5; ++i) scales5[i] = d.dsp_scales[i];
    c->dsp_scales = scales5;
    c->n_dsp_scales = int32_t(d.dsp_scales.size());
    c->descriptor_clip = d.descriptor_clip;
    c->orientation_bins = d.orientation_bins;
    c->orientation_peak_ratio = d.orientation_peak_ratio;
    c->num_octaves = d.num_octaves;
}

int oref_config_validate(const oref_config* c) {
    return guard([&] { to_cfg(c).validate(); return 0; });
}

// ---- image ingest: io.cpp:49-81 (w, h first with out = NULL) ---------------
int oref_load_image(const char* path, int* w, int* h, float* out) {
    return guard([&] {
        const GrayImage img = load_image(path);
        *w = img.width;
        *h = img.height;
        if (out) std::memcpy(out, img.data.data(), img.data.size() * sizeof(float));
        return 0;
    });
}

// ---- matching: match.cpp:77-119 (ratio_match), :71-75 (descriptor_distance)
// out3 receives (a, b, distance-bits) triples; returns the pair count or < 0.
int64_t oref_ratio_match(const float* da, int64_t na, const float* db, int64_t nb, int dim, float ratio,
                         int workers, int32_t* out3, int64_t cap, int64_t* putative) {
    int64_t n = -1;
    const int rc = guard([&] {
        FeatureSet a, b;
        a.dim = b.dim = dim;
        a.keypoints.resize((size_t)na);
        b.keypoints.resize((size_t)nb);
        a.descriptors.assign(da, da + na * dim);
        b.descriptors.assign(db, db + nb * dim);
        const MatchSet m = ratio_match(a, b, ratio, workers);
        putative[0] = m.putative_a;
        putative[1] = m.putative_b;
        n = (int64_t)m.pairs.size();
        for (int64_t i = 0; i < n && i < cap; ++i) {
            out3[3 * i + 0] = m.pairs[i].a;
            out3[3 * i + 1] = m.pairs[i].b;
            std::memcpy(&out3[3 * i + 2], &m.pairs[i].distance, 4);
        }
        return 0;
    });
    return rc ? rc : n;
}
float oref_descriptor_distance(const float* a, const float* b, int dim) {
    return descriptor_distance(std::span<const float>(a, dim), std::span<const float>(b, dim));
}

// ---- geometry: geom.cpp:108-161 (dlt_homography), :181-320 (magsac_lite),
// :322-333 (corner_error).  m = n x 4 doubles (x1, y1, x2, y2).
// Returns 0, or 1 for std::invalid_argument, 2 for std::runtime_error.
static std::vector<Correspondence> to_corr(const double* m, int64_t n) {
    std::vector<Correspondence> v((size_t)n);
    for (int64_t i = 0; i < n; ++i) v[(size_t)i] = {m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]};
    return v;
}
static int geom_guard(const std::function<void()>& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
int oref_dlt_homography(const double* m, int64_t n, const double* w, double* h_out) {
    return geom_guard([&] {
        const auto c = to_corr(m, n);
        const Homography h = w ? dlt_homography(c, std::span<const double>(w, (size_t)n)) : dlt_homography(c);
        for (int i = 0; i < 9; ++i) h_out[i] = h.h[i];
    });
}
int oref_magsac_lite(const double* m, int64_t n, int iterations, double tau, uint64_t seed, int workers,
                     int32_t* success_best, double* score_h /*[10]*/, uint8_t* mask) {
    return geom_guard([&] {
        const auto c = to_corr(m, n);
        const MagsacResult r = magsac_lite(c, iterations, tau, seed, workers);
        success_best[0] = r.success ? 1 : 0;
        success_best[1] = r.best_iteration;
        score_h[0] = r.score;
        for (int i = 0; i < 9; ++i) score_h[1 + i] = r.h.h[i];
        for (int64_t i = 0; i < n; ++i) mask[i] = r.success ? r.inlier_mask[(size_t)i] : 0;
    });
}
int oref_corner_error(const double* he, const double* hg, double w, double h, double* out) {
    return geom_guard([&] {
        Homography a, b;
        for (int i = 0; i < 9; ++i) {
            a.h[i] = he[i];
            b.h[i] = hg[i];
        }
        *out = corner_error(a, b, w, h);
    });
}

// ---- full pipeline: io.cpp:111-142 -----------------------------------------
int oref_extract(const float* img, int w, int h, const oref_config* c, int workers,
                 void** out) {
    return guard([&] {
        auto* fs = new FeatureSet(extract(to_img(img, w, h), to_cfg(c), workers));
        *out = fs;
        return 0;
    });
}
int64_t oref_fs_size(void* fs) { return int64_t(static_cast<FeatureSet*>(fs)->size()); }
void oref_fs_copy(void* fsv, Keypoint* kps, float* desc) {
    auto* fs = static_cast<FeatureSet*>(fsv);
    if (kps && fs->size()) std::memcpy(kps, fs->keypoints.data(), fs->size() * sizeof(Keypoint));
    if (desc && !fs->descriptors.empty())
        std::memcpy(desc, fs->descriptors.data(), fs->descriptors.size() * sizeof(float));
}
void oref_fs_free(void* fs) { delete static_cast<FeatureSet*>(fs); }

// detsum.cpp:129-132 / core.cpp:153-196 on caller-provided features.
static FeatureSet make_fs(const Keypoint* kps, const float* desc, int64_t n) {
    FeatureSet fs;
    fs.dim = kDescriptorDim;
    fs.keypoints.assign(kps, kps + n);
    fs.descriptors.assign(desc, desc + n * kDescriptorDim);
    return fs;
}
int oref_hash_features(const Keypoint* kps, const float* desc, int64_t n, char* hex65) {
    return guard([&] {
        const std::string h = detsum::hash_features(make_fs(kps, desc, n));
        std::memcpy(hex65, h.c_str(), 65);
        return 0;
    });
}
int64_t oref_serialize(const Keypoint* kps, const float* desc, int64_t n, uint8_t* out,
                       int64_t cap) {
    const auto bytes = serialize_features(make_fs(kps, desc, n));
    if (out && int64_t(bytes.size()) <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return int64_t(bytes.size());
}
void oref_canonical_sort(Keypoint* kps, float* desc, int64_t n) {
    FeatureSet fs = make_fs(kps, desc, n);
    canonical_sort(fs);
    std::memcpy(kps, fs.keypoints.data(), n * sizeof(Keypoint));
    std::memcpy(desc, fs.descriptors.data(), n * kDescriptorDim * sizeof(float));
}
int oref_sha256(const uint8_t* p, int64_t n, char* hex65) {
    const std::string h = detsum::sha256_hex(std::span<const uint8_t>(p, size_t(n)));
    std::memcpy(hex65, h.c_str(), 65);
    return 0;
}

// ---- scale space: scalespace.cpp:144-214 ------------------------------------
int oref_ss_build(const float* img, int w, int h, const oref_config* c, int workers,
                  void** out) {
    return guard([&] {
        *out = new ScaleSpace(build_scale_space(to_img(img, w, h), to_cfg(c), workers));
        return 0;
    });
}
// Handcrafted scale space (test_detect.cpp:14-30 style): levels supplied by caller.
void* oref_ss_from_levels(int n_oct, int s, float sigma0, int upsampled, const int32_t* dims,
                          const float* const* gauss, const float* const* dog) {
    auto* ss = new ScaleSpace();
    ss->intervals = s;
    ss->sigma0 = sigma0;
    ss->upsampled = upsampled != 0;
    ss->octaves.resize(n_oct);
    for (int o = 0; o < n_oct; ++o) {
        const int w = dims[2 * o], h = dims[2 * o + 1];
        for (int i = 0; i < s + 3; ++i) ss->octaves[o].gauss.push_back(to_img(gauss[o * (s + 3) + i], w, h));
        for (int i = 0; i < s + 2; ++i) ss->octaves[o].dog.push_back(to_img(dog[o * (s + 2) + i], w, h));
    }
    return ss;
}
void oref_ss_info(void* ssv, int32_t* n_oct, int32_t* upsampled, int32_t* dims) {
    auto* ss = static_cast<ScaleSpace*>(ssv);
    *n_oct = int32_t(ss->octaves.size());
    *upsampled = ss->upsampled ? 1 : 0;
    if (dims)
        for (size_t o = 0; o < ss->octaves.size(); ++o) {
            dims[2 * o] = ss->octaves[o].gauss[0].width;
            dims[2 * o + 1] = ss->octaves[o].gauss[0].height;
        }
}
// kind 0 = gauss, 1 = dog
void oref_ss_level(void* ssv, int o, int kind, int i, float* out) {
    auto* ss = static_cast<ScaleSpace*>(ssv);
    const GrayImage& g = kind == 0 ? ss->octaves[o].gauss[i] : ss->octaves[o].dog[i];
    std::memcpy(out, g.data.data(), g.size() * sizeof(float));
}
void oref_ss_free(void* ss) { delete static_cast<ScaleSpace*>(ss); }

int oref_gaussian_kernel(double sigma, float* out, int cap) {
    return guard([&] {
        const auto k = gaussian_kernel(sigma);
        if (int(k.size()) <= cap) std::memcpy(out, k.data(), k.size() * 4);
        return int(k.size());
    });
}
int oref_convolve(const float* img, int w, int h, const float* k, int len, int workers,
                  float* out) {
    return guard([&] {
        const GrayImage r = convolve_separable(to_img(img, w, h),
                                               std::span<const float>(k, size_t(len)), workers);
        std::memcpy(out, r.data.data(), r.size() * 4);
        return 0;
    });
}
void oref_upsample2x(const float* img, int w, int h, float* out) {
    const GrayImage r = upsample2x(to_img(img, w, h));
    std::memcpy(out, r.data.data(), r.size() * 4);
}
void oref_decimate2x(const float* img, int w, int h, float* out) {
    const GrayImage r = decimate2x(to_img(img, w, h));
    std::memcpy(out, r.data.data(), r.size() * 4);
}

// ---- detection: detect.cpp:32-172 ---------------------------------------------
// extrema out: n x 5 int32 (octave, interval, row, col, is_max)
int64_t oref_find_extrema(void* ssv, const oref_config* c, int workers, int32_t* out,
                          int64_t cap) {
    const auto ex = find_extrema(*static_cast<ScaleSpace*>(ssv), to_cfg(c), workers);
    for (size_t k = 0; k < ex.size() && int64_t(k) < cap; ++k) {
        out[5 * k + 0] = ex[k].octave;
        out[5 * k + 1] = ex[k].interval;
        out[5 * k + 2] = ex[k].row;
        out[5 * k + 3] = ex[k].col;
        out[5 * k + 4] = ex[k].is_max ? 1 : 0;
    }
    return int64_t(ex.size());
}
int oref_refine(void* ssv, const int32_t* e5, const oref_config* c, Keypoint* out) {
    RawExtremum e{e5[0], e5[1], e5[2], e5[3], e5[4] != 0};
    const auto kp = refine_extremum(*static_cast<ScaleSpace*>(ssv), e, to_cfg(c));
    if (!kp) return 0;
    *out = *kp;
    return 1;
}
int64_t oref_detect(void* ssv, const oref_config* c, int workers, Keypoint* out, int64_t cap) {
    const auto kps = detect_keypoints(*static_cast<ScaleSpace*>(ssv), to_cfg(c), workers);
    for (size_t k = 0; k < kps.size() && int64_t(k) < cap; ++k) out[k] = kps[k];
    return int64_t(kps.size());
}

// ---- orientation: orient.cpp:13-113 -------------------------------------------
int oref_orientation_histogram(void* ssv, const Keypoint* kp, const oref_config* c,
                               float* out) {
    return guard([&] {
        const auto h = orientation_histogram(*static_cast<ScaleSpace*>(ssv), *kp, to_cfg(c));
        std::memcpy(out, h.data(), h.size() * 4);
        return int(h.size());
    });
}
int oref_assign_orientations(void* ssv, const Keypoint* kp, const oref_config* c,
                             Keypoint* out) {
    const auto v = assign_orientations(*static_cast<ScaleSpace*>(ssv), *kp, to_cfg(c));
    for (size_t k = 0; k < v.size(); ++k) out[k] = v[k];
    return int(v.size());
}
int oref_nearest_gauss_level(void* ssv, double sigma_rel) {
    return nearest_gauss_level(*static_cast<ScaleSpace*>(ssv), sigma_rel);
}

// ---- descriptor: describe.cpp:33-173 ------------------------------------------
int oref_raw_descriptor(void* ssv, const Keypoint* kp, double f, const oref_config* c,
                        float* out) {
    return guard([&] {
        const auto d = raw_descriptor(*static_cast<ScaleSpace*>(ssv), *kp, f, to_cfg(c));
        std::memcpy(out, d.data(), d.size() * 4);
        return 0;
    });
}
int oref_dsp_descriptor(void* ssv, const Keypoint* kp, const oref_config* c, float* out) {
    return guard([&] {
        const auto d = dsp_descriptor(*static_cast<ScaleSpace*>(ssv), *kp, to_cfg(c));
        std::memcpy(out, d.data(), d.size() * 4);
        return 0;
    });
}
int oref_root_sift(float* v, int n) {
    return guard([&] { root_sift(std::span<float>(v, size_t(n))); return 0; });
}

// ---- detsum: detsum.cpp:13-127 -------------------------------------------------
float oref_tree_sum(const float* v, int64_t n, int workers) {
    return detsum::tree_sum(std::span<const float>(v, size_t(n)), workers);
}
double oref_tree_sum_f64(const double* v, int64_t n, int workers) {
    return detsum::tree_sum(std::span<const double>(v, size_t(n)), workers);
}
int oref_tree_hist(const int32_t* bins, const float* w, int64_t n, int bin_count, int workers,
                   float* out) {
    return guard([&] {
        std::vector<detsum::Contribution> c(n);
        for (int64_t i = 0; i < n; ++i) c[i] = {bins[i], w[i]};
        const auto h = detsum::tree_accumulate_histogram(c, bin_count, workers);
        std::memcpy(out, h.data(), h.size() * 4);
        return 0;
    });
}

// ---- synthetic inputs: tests/support/synth.cpp ------------------------------------
void oref_value_noise(int w, int h, uint64_t seed, int octaves, int cells, float* out) {
    const GrayImage g = synth::value_noise_image(w, h, seed, octaves, cells);
    std::memcpy(out, g.data.data(), g.size() * 4);
}
void oref_blob_field(int w, int h, uint64_t seed, int count, float* out) {
    const GrayImage g = synth::blob_field(w, h, seed, count);
    std::memcpy(out, g.data.data(), g.size() * 4);
}
void oref_add_blob(float* img, int w, int h, double cx, double cy, double sigma, double amp) {
    GrayImage g = to_img(img, w, h);
    synth::add_blob(g, cx, cy, sigma, amp);
    std::memcpy(img, g.data.data(), g.size() * 4);
}
void oref_photometric(const float* img, int w, int h, double gamma, double gain, double bias,
                      float* out) {
    const GrayImage g = synth::photometric(to_img(img, w, h), gamma, gain, bias);
    std::memcpy(out, g.data.data(), g.size() * 4);
}
void oref_warp_similarity(const float* img, int w, int h, double angle, double scale, double cx,
                          double cy, int ow, int oh, float* out) {
    const GrayImage g =
        synth::warp_image(to_img(img, w, h), synth::similarity(angle, scale, cx, cy), ow, oh);
    std::memcpy(out, g.data.data(), g.size() * 4);
}
uint64_t oref_splitmix_next(uint64_t* state) {
    SplitMix64 r(*state);
    const uint64_t v = r.next();
    *state = r.state;
    return v;
}

// ---- independent brute-force oracles: tests/support/oracles.cpp ---------------------
// out: n x 6 doubles (x, y, sigma, octave, interval, response)
int64_t oref_brute_force_detect(void* ssv, const oref_config* c, double* out, int64_t cap) {
    const auto v = oracles::brute_force_detect(*static_cast<ScaleSpace*>(ssv), to_cfg(c));
    for (size_t k = 0; k < v.size() && int64_t(k) < cap; ++k) {
        out[6 * k + 0] = v[k].x;
        out[6 * k + 1] = v[k].y;
        out[6 * k + 2] = v[k].sigma;
        out[6 * k + 3] = v[k].octave;
        out[6 * k + 4] = v[k].interval;
        out[6 * k + 5] = v[k].response;
    }
    return int64_t(v.size());
}
void oref_naive_orientation_histogram(void* ssv, const Keypoint* kp, const oref_config* c,
                                      double* out) {
    const auto v = oracles::naive_orientation_histogram(*static_cast<ScaleSpace*>(ssv), *kp,
                                                        to_cfg(c));
    std::memcpy(out, v.data(), v.size() * 8);
}
void oref_naive_single_scale_descriptor(void* ssv, const Keypoint* kp, const oref_config* c,
                                        double* out) {
    const auto v = oracles::naive_single_scale_descriptor(*static_cast<ScaleSpace*>(ssv), *kp,
                                                          to_cfg(c));
    std::memcpy(out, v.data(), v.size() * 8);
}

}  // extern "C"
