// include/dsift.hpp — header-only C++ face of the C ABI, mirroring the
// reference's extraction API so existing C++ callers swap one include:
//
//   reference:  detsift::FeatureSet detsift::extract(const GrayImage&, const SiftConfig&, int workers = 1)
//               (/root/reference/proj/include/detsift/io.hpp:17-19)
//   here:       dsift::FeatureSet  dsift::extract(const GrayImage&, const SiftConfig&, int workers = 1)
//
// `workers` keeps its meaning (host threads, 0 = all; parallel.hpp:12-16) and,
// as in the reference, never changes the output.  The device is
// dsift::default_device() ($DSIFT_DEVICE, else 0); Extractor picks one
// explicitly.  Each host thread reuses one cached context per config.
//
// The types restate detsift's (core.hpp:11-78) field for field; Keypoint is
// layout-identical to the reference struct and to dsift_keypoint.  Errors
// surface as the same exception types the reference throws:
// std::invalid_argument for DSIFT_EINVAL, std::runtime_error otherwise.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdlib>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsift.h"

namespace dsift {

struct GrayImage {   // core.hpp:11-26
    int width = 0;
    int height = 0;
    std::vector<float> data;
    GrayImage() = default;
    GrayImage(int w, int h, float fill = 0.0f) : width(w), height(h), data(size_t(w) * h, fill) {}
    float& at(int x, int y) { return data[size_t(y) * width + x]; }
    float at(int x, int y) const { return data[size_t(y) * width + x]; }
    size_t size() const { return data.size(); }
    bool empty() const { return width <= 0 || height <= 0; }
};

struct SiftConfig {   // core.hpp:30-47
    float sigma0 = 1.6f;
    int intervals_per_octave = 3;
    float assumed_input_blur = 0.5f;
    float contrast_threshold = 0.04f;
    float edge_ratio = 10.0f;
    int max_refine_iters = 5;
    int64_t upsample_pixel_limit = 4'000'000;
    std::vector<double> dsp_scales = {0.5, 1.0 / 1.4142135623730951, 1.0, 1.4142135623730951, 2.0};
    float descriptor_clip = 0.2f;
    int orientation_bins = 36;
    float orientation_peak_ratio = 0.8f;
    int num_octaves = 0;

    dsift_config to_c() const {
        dsift_config c;
        c.sigma0 = sigma0;
        c.intervals = intervals_per_octave;
        c.assumed_blur = assumed_input_blur;
        c.contrast_threshold = contrast_threshold;
        c.edge_ratio = edge_ratio;
        c.max_refine_iters = max_refine_iters;
        c.upsample_pixel_limit = upsample_pixel_limit;
        c.dsp_scales = dsp_scales.data();
        c.n_dsp_scales = int32_t(dsp_scales.size());
        c.descriptor_clip = descriptor_clip;
        c.orientation_bins = orientation_bins;
        c.orientation_peak_ratio = orientation_peak_ratio;
        c.num_octaves = num_octaves;
        return c;
    }
    void validate() const;   // SiftConfig::validate (core.cpp:17-46)
    bool operator==(const SiftConfig&) const = default;
};

struct Keypoint {   // core.hpp:55-63
    float x = 0.0f, y = 0.0f, sigma = 0.0f, angle = 0.0f, response = 0.0f;
    int32_t octave = 0, interval = 0;
};
static_assert(sizeof(Keypoint) == sizeof(dsift_keypoint), "Keypoint must stay layout-identical");
static_assert(sizeof(Keypoint) == 28, "detsift::Keypoint is 7 x 4 bytes");

struct FeatureSet {   // core.hpp:66-78
    std::vector<Keypoint> keypoints;
    std::vector<float> descriptors;
    std::vector<uint8_t> descriptors_u8;   // q(v) = min(255, lround(v * 255))
    int dim = 128;
    size_t size() const { return keypoints.size(); }
    std::span<const float> row(size_t i) const { return {descriptors.data() + i * dim, size_t(dim)}; }
};

// detsift::Homography / Correspondence / MagsacResult (geom.hpp:14-61),
// layout-compatible with the C ABI's double arrays.
struct Homography {
    std::array<double, 9> h = {1, 0, 0, 0, 1, 0, 0, 0, 1};
};
struct Correspondence {
    double x1 = 0, y1 = 0, x2 = 0, y2 = 0;
};
struct MagsacResult {
    bool success = false;
    Homography h;
    std::vector<uint8_t> inlier_mask;
    double score = 0.0;
    int best_iteration = -1;
};

[[noreturn]] inline void throw_status(int rc) {
    const std::string msg = dsift_last_error();
    if (rc == DSIFT_EINVAL) throw std::invalid_argument(msg);
    if (rc == DSIFT_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(std::string(dsift_strerror(rc)) + ": " + msg);
}
inline void check(int rc) {
    if (rc != DSIFT_OK) throw_status(rc);
}

// detsift::corner_error (geom.cpp:322-333).
inline double corner_error(const Homography& est, const Homography& gt, double width, double height) {
    double out = 0.0;
    check(dsift_corner_error(est.h.data(), gt.h.data(), width, height, &out));
    return out;
}

inline void SiftConfig::validate() const {
    const dsift_config c = to_c();
    check(dsift_config_validate(&c));
}

// RAII context: one device, one stream, reusable across many images.
class Extractor {
   public:
    explicit Extractor(const SiftConfig& cfg = {}, int device = 0) : cfg_(cfg), device_(device) {
        const dsift_config c = cfg_.to_c();
        dsift_ctx* ctx = nullptr;
        check(dsift_create(device, &c, &ctx));
        ctx_.reset(ctx);
    }
    // detsift::extract (io.cpp:111-142) for one image.
    FeatureSet extract(const GrayImage& img) {
        return std::move(extract_batch(&img, 1)[0]);
    }
    // Any number of images of any sizes in one call (dsift_extract_images);
    // result i is bit-identical to extract(imgs[i]).
    std::vector<FeatureSet> extract_batch(const GrayImage* imgs, int n) {
        if (n <= 0) return {};
        std::vector<dsift_image> views(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) views[i] = dsift_image{imgs[i].data.data(), imgs[i].width, imgs[i].height};
        check(dsift_extract_images(ctx_.get(), views.data(), n, DSIFT_INPUT_HOST));
        int64_t total = 0;
        check(dsift_result_sync(ctx_.get(), &total));
        std::vector<Keypoint> kps(static_cast<size_t>(total));
        std::vector<float> desc(static_cast<size_t>(total) * 128);
        std::vector<uint8_t> desc8(static_cast<size_t>(total) * 128);
        std::vector<int64_t> offs(static_cast<size_t>(n) + 1);
        check(dsift_result_copy(ctx_.get(), reinterpret_cast<dsift_keypoint*>(kps.data()), desc.data(),
                                desc8.data(), offs.data()));
        std::vector<FeatureSet> out(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            const size_t b = size_t(offs[i]), e = size_t(offs[i + 1]);
            out[i].keypoints.assign(kps.begin() + b, kps.begin() + e);
            out[i].descriptors.assign(desc.begin() + b * 128, desc.begin() + e * 128);
            out[i].descriptors_u8.assign(desc8.begin() + b * 128, desc8.begin() + e * 128);
        }
        return out;
    }
    std::string sha256(int image = 0) {
        char hex[65];
        check(dsift_result_sha256(ctx_.get(), image, hex));
        return hex;
    }
    // detsift::magsac_lite (geom.cpp:181-320) on the device, bit-identical.
    MagsacResult magsac_lite(std::span<const Correspondence> matches, int iterations, double tau, uint64_t seed) {
        dsift_magsac_result r{};
        MagsacResult out;
        out.inlier_mask.assign(matches.size(), 0);
        check(dsift_magsac_lite(ctx_.get(), reinterpret_cast<const double*>(matches.data()),
                                static_cast<int64_t>(matches.size()), iterations, tau, seed, &r,
                                out.inlier_mask.data()));
        out.success = r.success != 0;
        std::copy(r.h, r.h + 9, out.h.h.begin());
        out.score = r.score;
        out.best_iteration = r.best_iteration;
        if (!out.success) out.inlier_mask.clear();
        return out;
    }
    // detsift::dlt_homography (geom.cpp:108-161) on the device.
    Homography dlt_homography(std::span<const Correspondence> pairs, std::span<const double> weights = {}) {
        if (!weights.empty() && weights.size() != pairs.size())
            throw std::invalid_argument("dlt: weight count mismatch");
        Homography h;
        check(dsift_dlt_homography(ctx_.get(), reinterpret_cast<const double*>(pairs.data()),
                                   static_cast<int64_t>(pairs.size()), weights.empty() ? nullptr : weights.data(),
                                   h.h.data()));
        return h;
    }
    dsift_ctx* handle() { return ctx_.get(); }
    int device() const { return device_; }
    const SiftConfig& config() const { return cfg_; }

   private:
    struct Deleter {
        void operator()(dsift_ctx* c) const { dsift_destroy(c); }
    };
    SiftConfig cfg_;
    int device_ = 0;
    std::unique_ptr<dsift_ctx, Deleter> ctx_;
};

// The device the drop-in extract() uses: $DSIFT_DEVICE, else 0.
inline int default_device() {
    const char* e = std::getenv("DSIFT_DEVICE");
    return e ? std::atoi(e) : 0;
}

// Drop-in for detsift::extract (io.hpp:17-19, io.cpp:111-142).  `workers`
// is accepted with the reference's meaning and, like there, does not change
// the output (io.hpp:17-18); the fan-out is the GPU's.  The context (stream,
// buffers) is cached per host thread and reused while config and device stay
// the same, so per-image calls pay no setup.
inline FeatureSet extract(const GrayImage& img, const SiftConfig& cfg = {}, int workers = 1) {
    (void)workers;
    thread_local std::unique_ptr<Extractor> cached;
    const int device = default_device();
    if (!cached || cached->device() != device || !(cached->config() == cfg)) {
        cached.reset();
        cached = std::make_unique<Extractor>(cfg, device);
    }
    return cached->extract(img);
}

}  // namespace dsift
