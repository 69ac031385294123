#include <cctype>
// dsift_host.cu — host orchestration and the C ABI (include/dsift.h).
//
// Replaces detsift::extract (io.cpp:111-142) and its parallel_for fan-out
// (parallel.hpp:21-54): a batch of same-size images is pushed through
// K1 (pyramid+DoG, per level, grid.z = image) -> K2/K3 (extrema+refine, one
// launch for all octaves) -> K4 (orientation + fan-out) -> K7 (canonical
// sort) -> K5/K6 (descriptors in canonical order), all on one stream, with a
// single host synchronisation when the caller asks for the result.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: stage ranges for ncu --nvtx / nsys
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dlpack_min.h"
#include "dsift_common.cuh"
#include "dsift_tma.cuh"
#include "dsift_kernels.cuh"

namespace dsift {


// ---- errors -------------------------------------------------------------------
thread_local std::string g_err;

struct Error {
    int code;
    std::string msg;
};

static void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error{e == cudaErrorMemoryAllocation ? DSIFT_ENOMEM : DSIFT_ECUDA,
                    std::string(what) + ": " + cudaGetErrorString(e)};
}

static void invalid(const std::string& m) { throw Error{DSIFT_EINVAL, m}; }

template <typename F>
static int guard(F&& f) {
    try {
        f();
        return DSIFT_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return DSIFT_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DSIFT_ECUDA;
    }
}

// ---- config (core.hpp:30-47, core.cpp:17-46) -----------------------------------
static const double kDefaultDsp[5] = {0.5, 1.0 / 1.4142135623730951, 1.0, 1.4142135623730951, 2.0};

struct Cfg {
    dsift_config c;
    std::vector<double> dsp;
};

static void validate(const dsift_config& c) {
    if (!(c.sigma0 > 0.0f) || !(c.assumed_blur >= 0.0f) || !(c.sigma0 > c.assumed_blur))
        invalid("config: require sigma0 > assumed_input_blur >= 0");
    if (c.intervals < 1) invalid("config: intervals_per_octave must be >= 1");
    if (!(c.contrast_threshold > 0.0f)) invalid("config: contrast_threshold must be > 0");
    if (!(c.edge_ratio > 1.0f)) invalid("config: edge_ratio must be > 1");
    if (c.max_refine_iters < 1) invalid("config: max_refine_iters must be >= 1");
    if (c.upsample_pixel_limit < 0) invalid("config: upsample_pixel_limit must be >= 0");
    if (c.n_dsp_scales <= 0 || !c.dsp_scales) invalid("config: dsp_scales must be nonempty");
    for (int i = 0; i < c.n_dsp_scales; ++i) {
        if (!(c.dsp_scales[i] > 0.0)) invalid("config: dsp_scales must all be > 0");
        if (i > 0 && !(c.dsp_scales[i] > c.dsp_scales[i - 1]))
            invalid("config: dsp_scales must be strictly increasing");
    }
    if (!(c.descriptor_clip > 0.0f)) invalid("config: descriptor_clip must be > 0");
    if (c.orientation_bins < 2) invalid("config: orientation_bins must be >= 2");
    if (!(c.orientation_peak_ratio > 0.0f) || c.orientation_peak_ratio > 1.0f)
        invalid("config: orientation_peak_ratio must be in (0,1]");
    if (c.num_octaves < 0) invalid("config: num_octaves must be >= 0 (0 = auto)");
    // device-implementation limits (explicit, never silent)
    if (c.intervals + 3 > kMaxLevels || c.intervals > 8)   // K2 packs 4 rows x s levels per thread in 32 bits
        invalid("config: intervals_per_octave too large for this build (max 8)");
    if (c.n_dsp_scales > kMaxDsp) invalid("config: too many dsp_scales for this build");
    if (c.orientation_bins > kMaxOriBins) invalid("config: orientation_bins too large for this build");
}

// ---- scale-space plan (scalespace.cpp:11-36, 144-214) --------------------------------
static std::vector<float> gaussian_taps(double sigma) {
    if (!(sigma > 0.0)) invalid("gaussian_kernel: sigma must be > 0");
    const int radius = (int)std::ceil(4.0 * sigma);
    std::vector<double> raw(2 * radius + 1);
    double sum = 0.0;
    for (int k = -radius; k <= radius; ++k) {
        raw[k + radius] = std::exp(-double(k) * k / (2.0 * sigma * sigma));
        sum += raw[k + radius];
    }
    std::vector<float> out(raw.size());
    for (size_t i = 0; i < raw.size(); ++i) out[i] = (float)(raw[i] / sum);
    return out;
}

struct Plan {
    int in_w = 0, in_h = 0, base_w = 0, base_h = 0;
    bool up = false;
    int s = 3, n_oct = 0;
    std::vector<int> ow, oh, pitch;
    std::vector<float> bridge;
    std::vector<std::vector<float>> inc;   // s+2 incremental kernels
    double level_sigma[kMaxLevels] = {};
    bool handcrafted = false;
};

static int round_pitch(int w) { return (w + 31) & ~31; }
// Rows per pyramid level: h, rounded up (by at most 3 for a 32-float pitch) so
// that a level is a multiple of 512 bytes.  With 512-byte aligned octave
// blocks every level and every image's level stack then starts 512-byte
// aligned, as a pitched 2D texture over the stack requires (K5's gathers).
static int level_rows(int pitch, int h) {
    int r = h;
    while (((long long)pitch * r) % 128 != 0) ++r;
    return r;
}

static Plan make_plan(const Cfg& cfg, int w, int h) {
    const dsift_config& c = cfg.c;
    if (w <= 0 || h <= 0) invalid("build_scale_space: empty image");
    Plan p;
    p.in_w = w;
    p.in_h = h;
    p.s = c.intervals;
    p.up = (int64_t)w * h <= c.upsample_pixel_limit;
    p.base_w = p.up ? 2 * w : w;
    p.base_h = p.up ? 2 * h : h;
    const double assumed = p.up ? 2.0 * c.assumed_blur : c.assumed_blur;
    if (!((double)c.sigma0 > assumed)) invalid("build_scale_space: effective input blur exceeds sigma0");
    if (std::min(p.base_w, p.base_h) < 8)
        invalid("build_scale_space: image smaller than 8x8 after upsampling policy");
    const int s = c.intervals;
    int auto_oct = -2;
    for (int d = std::min(p.base_w, p.base_h); d > 1; d /= 2) ++auto_oct;
    auto_oct = std::max(1, auto_oct);
    const double bridge = std::sqrt(double(c.sigma0) * c.sigma0 - assumed * assumed);
    std::vector<double> inc;
    for (int i = 1; i < s + 3; ++i)
        inc.push_back(c.sigma0 * std::pow(2.0, double(i - 1) / s) * std::sqrt(std::pow(2.0, 2.0 / s) - 1.0));
    int max_radius = (int)std::ceil(4.0 * bridge);
    for (double sg : inc) max_radius = std::max(max_radius, (int)std::ceil(4.0 * sg));
    if (std::max(p.base_w, p.base_h) < max_radius)
        invalid("build_scale_space: image too small for the blur ladder");
    if (max_radius > kMaxRadius) invalid("config: Gaussian radius exceeds this build's limit");
    int feasible = 1;
    for (int ww = p.base_w / 2, hh = p.base_h / 2; std::min(ww, hh) >= 8 && std::max(ww, hh) >= max_radius;
         ww /= 2, hh /= 2)
        ++feasible;
    int oct = c.num_octaves > 0 ? std::min(c.num_octaves, auto_oct) : auto_oct;
    oct = std::min(oct, feasible);
    if (oct > kMaxOctaves) oct = kMaxOctaves;
    p.n_oct = oct;
    int ww = p.base_w, hh = p.base_h;
    for (int o = 0; o < oct; ++o) {
        p.ow.push_back(ww);
        p.oh.push_back(hh);
        p.pitch.push_back(round_pitch(ww));
        ww /= 2;
        hh /= 2;
    }
    p.bridge = gaussian_taps(bridge);
    for (double sg : inc) p.inc.push_back(gaussian_taps(sg));
    for (int i = 0; i < s + 3; ++i) p.level_sigma[i] = c.sigma0 * std::pow(2.0, double(i) / s);
    return p;
}

// ---- device memory ---------------------------------------------------------------
struct DevBuf {
    std::shared_ptr<void> ptr;
    size_t bytes = 0;
    template <typename T>
    T* as() const { return static_cast<T*>(ptr.get()); }
    void ensure(size_t need) {
        if (need <= bytes && ptr && ptr.use_count() == 1) return;
        if (need < bytes) need = bytes;   // keep the larger size when forking an exported buffer
        ptr.reset();
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, std::max<size_t>(need, 256)), "cudaMalloc");
        ptr = std::shared_ptr<void>(p, [](void* q) { cudaFree(q); });
        bytes = std::max<size_t>(need, 256);
    }
};

// One size group of a (possibly ragged) batch: images of one size, packed
// contiguously on the device.
struct Group {
    int w = 0, h = 0;
    std::vector<int> idx;          // batch indices, ascending
    const float* dev = nullptr;    // [idx.size()][h][w] device images
    long long cap_det = 0, cap_ori = 0;
    long long stage_base = 0;      // first staging row (ragged batches)
    long long offs_base = 0;       // first entry in the staging offsets
};

}  // namespace dsift

using namespace dsift;

// A batch result: output buffers, its completion event and the replay record.
// A context owns a default result; dsift_result_create adds more so one
// context can keep several batches in flight (dsift_result_select).
struct dsift_result {
    dsift_ctx* owner = nullptr;
    DevBuf pub_kps, desc, desc_u8, offsets, totals, input, input_u8;
    DevBuf stage_kps, stage_desc, stage_u8, stage_offs, map;   // ragged batches only
    cudaEvent_t done = nullptr;        // the whole batch is written
    cudaEvent_t input_free = nullptr;  // input[] no longer read by the batch's kernels
    bool pending = false, ready = false;
    int batch = 0;
    int64_t total = 0;
    unsigned long long slow = 0;
    unsigned long long lattice = 0, lattice_in = 0;   // descriptor lattice points (DSIFT_STAT_LATTICE_*)
    std::vector<int64_t> h_offsets;
    std::vector<Group> groups;         // replayed on a capacity overflow (automatic capacity)
    std::vector<long long> h_map;      // ragged batches: image -> (staging offsets entry, row base)
    bool direct = true;                // one group in batch order: outputs written in place
    int retries = 0;
};

struct dsift_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;   // host -> device input copies (overlap the previous batch)
    Cfg cfg;
    long long cap_override = 0;
    double cap_scale = 1.0;   // automatic capacities grow x4 after an overflow (then the batch is replayed)
    Plan plan;
    int batch = 0;            // images in the current pyramid
    PyramidDesc pyr{};
    DevBuf det_aux, ori_aux, match_in, match_scratch, match_best, geom_in, geom_scratch, geom_out;
    DevBuf pyramid, blur_flags, counters, det_states, ori_states, det_kps, det_cand, ori_kps, sorted_kps, sort_work, scratch,
        stage_kps, stage_out, trig, slow, ref_states, keep, stage_in;
    long long cap_det = 0, cap_ori = 0;
    long long launches = 0;
    int sm_count = 148;
    bool profiling = false;
    int force_exact = 0;
    dsift_result def;
    dsift_result* cur = &def;
    cudaEvent_t stage_ev[6] = {};
    // K5's bilinear gathers: one pitched 2D texture per (image, octave) over
    // that image's Gaussian levels stacked vertically, rebuilt when the
    // pyramid's address or layout changes (gauss_tex_key)
    std::vector<cudaTextureObject_t> gauss_tex;
    std::vector<long long> gauss_tex_key;
    DevBuf gauss_tex_dev;
    bool gauss_tex_ok = false;
    bool tex_gathers = true;   // DSIFT_OPT_TEXTURE_GATHERS
};

namespace dsift {

static void set_device(dsift_ctx* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

static void build_pyramid_desc(dsift_ctx* c) {
    const Plan& p = c->plan;
    PyramidDesc d{};
    d.n_oct = p.n_oct;
    d.s = p.s;
    d.batch = c->batch;
    d.upsampled = p.up ? 1 : 0;
    d.sigma0 = c->cfg.c.sigma0;
    for (int i = 0; i < p.s + 3; ++i) d.level_sigma[i] = p.level_sigma[i];
    size_t off = 0;
    for (int o = 0; o < p.n_oct; ++o) {
        OctaveDesc& od = d.oct[o];
        od.w = p.ow[o];
        od.h = p.oh[o];
        od.pitch = p.pitch[o];
        od.level_stride = (long long)od.pitch * level_rows(od.pitch, od.h);
        od.tiles_x = od.w >= 3 ? (od.w - 2 + 31) / 32 : 0;
        od.tiles_y = od.h >= 3 ? (od.h - 2 + 31) / 32 : 0;
        if (od.tiles_x == 0 || od.tiles_y == 0) od.tiles_x = od.tiles_y = 0;
        const size_t g = sizeof(float) * (size_t)c->batch * (p.s + 3) * od.level_stride;
        const size_t dg = sizeof(float) * (size_t)c->batch * (p.s + 2) * od.level_stride;
        od.gauss = reinterpret_cast<float*>(off);
        off += (g + 511) & ~size_t(511);
        od.dog = reinterpret_cast<float*>(off);
        off += (dg + 511) & ~size_t(511);
    }
    c->pyramid.ensure(off);
    char* base = c->pyramid.as<char>();
    for (int o = 0; o < p.n_oct; ++o) {
        d.oct[o].gauss = reinterpret_cast<float*>(base + reinterpret_cast<size_t>(d.oct[o].gauss));
        d.oct[o].dog = reinterpret_cast<float*>(base + reinterpret_cast<size_t>(d.oct[o].dog));
    }
    c->pyr = d;
}

// octaves of at most this many pixels are fused into one launch, where the
// strip launches are pure latency (C3: from 50x37, C1: from 40x30); larger
// octaves are faster as strips (one CTA per image is conversion-bound there:
// C1 from 160x120 measured 0.91 ms of pyramid instead of 0.66)
constexpr long long kSmallOctavePx = 2500;

static void launch_pyramid(dsift_ctx* c, const float* dev_images) {
    const Plan& p = c->plan;
    const PyramidDesc& d = c->pyr;
    const int s = p.s;
    // per-level "every value a positive normal >= 2^-100" flags (0 = yes), set by
    // the producing kernel and read by the consumer (ALU widening); only levels
    // whose producer checks (radius <= 16) are handed on
    c->blur_flags.ensure(sizeof(int) * (size_t)p.n_oct * (s + 3));
    int* flags = c->blur_flags.as<int>();
    cuda_check(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)p.n_oct * (s + 3), c->stream), "memset flags");
    std::vector<char> checked((size_t)p.n_oct * (s + 3), 0);
    auto flag_of = [&](int o, int i) { return flags + o * (s + 3) + i; };
    // the strip kernel's source map: 3-D {w, h, batch}, box {kInW, 32, 1} (stride es)
    auto set_map = [&](BlurArgs& a, int R, uint32_t es) {
        const int bw = blur_strip_box_w(R);
        a.use_tma = bw > 0 && tma_encode_3d_f32(&a.src_map, a.src, (uint64_t)a.src_w, (uint64_t)a.src_h,
                                                  (uint64_t)c->batch, (uint64_t)a.src_pitch,
                                                  (uint64_t)a.src_img_stride, (uint32_t)bw * es, 32u * es, 1u, es)
                        ? 1 : 0;
    };
    // small octaves (two whole levels fit in shared memory, every incremental
    // radius <= 16) go to one fused launch, one CTA per image
    int o_small = p.n_oct;
    {
        bool radii_ok = true;
        for (int i = 0; i < s + 2; ++i) radii_ok = radii_ok && (int)p.inc[i].size() / 2 <= 16;
        for (int o = 1; radii_ok && o < p.n_oct; ++o)
            if ((long long)p.ow[o] * p.oh[o] <= kSmallOctavePx && small_octaves_smem(p.ow[o] * p.oh[o]) <= 200 * 1024) {
                o_small = o;
                break;
            }
    }
    for (int o = 0; o < o_small; ++o) {
        const OctaveDesc& od = d.oct[o];
        const long long gstride = d.gauss_img_stride(o), dstride = d.dog_img_stride(o);
        auto fill_taps = [](BlurArgs& a, const std::vector<float>& t) {
            for (size_t i = 0; i < t.size(); ++i) a.taps[i] = (double)t[i];
        };
        int first_level;
        if (o == 0) {
            BlurArgs a{};
            a.src = dev_images;
            a.src_img_stride = (long long)p.in_w * p.in_h;
            a.src_pitch = p.in_w;
            a.src_w = p.in_w;
            a.src_h = p.in_h;
            a.dst = od.gauss;
            a.dst_img_stride = gstride;
            a.w = od.w;
            a.h = od.h;
            a.pitch = od.pitch;
            fill_taps(a, p.bridge);
            const int R = (int)p.bridge.size() / 2;
            if (R <= 16) {
                a.dst_flag = flag_of(0, 0);
                checked[0] = 1;
            }
            if (!p.up) set_map(a, R, 1);
            cuda_check(launch_blur(a, p.up ? kModeUpsample : kModeRaw, R, c->batch, c->stream), "bridge blur");
            ++c->launches;
            first_level = 1;
        } else {
            const OctaveDesc& pd = d.oct[o - 1];
            BlurArgs a{};
            a.src = pd.gauss + (long long)s * pd.level_stride;
            a.src_img_stride = d.gauss_img_stride(o - 1);
            a.src_pitch = pd.pitch;
            a.src_w = pd.w;
            a.src_h = pd.h;
            a.seed = od.gauss;
            a.seed_img_stride = gstride;
            a.dst = od.gauss + od.level_stride;
            a.dst_img_stride = gstride;
            a.dog = od.dog;
            a.dog_img_stride = dstride;
            a.w = od.w;
            a.h = od.h;
            a.pitch = od.pitch;
            fill_taps(a, p.inc[0]);
            const int R = (int)p.inc[0].size() / 2;
            if (checked[(o - 1) * (s + 3) + s]) a.src_flag = flag_of(o - 1, s);
            if (R <= 16) {
                a.dst_flag = flag_of(o, 1);
                checked[o * (s + 3) + 1] = 1;
            }
            // (the decimated source is gathered: a stride-2 TMA box is not used)
            cuda_check(launch_blur(a, kModeDecimate, R, c->batch, c->stream), "decimate blur");
            ++c->launches;
            first_level = 2;
        }
        for (int i = first_level; i < s + 3; ++i) {
            BlurArgs a{};
            a.src = od.gauss + (long long)(i - 1) * od.level_stride;
            a.src_img_stride = gstride;
            a.src_pitch = od.pitch;
            a.src_w = od.w;
            a.src_h = od.h;
            a.dst = od.gauss + (long long)i * od.level_stride;
            a.dst_img_stride = gstride;
            a.dog = od.dog + (long long)(i - 1) * od.level_stride;
            a.dog_img_stride = dstride;
            a.w = od.w;
            a.h = od.h;
            a.pitch = od.pitch;
            fill_taps(a, p.inc[i - 1]);
            const int R = (int)p.inc[i - 1].size() / 2;
            if (checked[o * (s + 3) + i - 1]) a.src_flag = flag_of(o, i - 1);
            if (R <= 16) {
                a.dst_flag = flag_of(o, i);
                checked[o * (s + 3) + i] = 1;
            }
            set_map(a, R, 1);
            cuda_check(launch_blur(a, kModeLevel, R, c->batch, c->stream), "level blur");
            ++c->launches;
        }
    }
    if (o_small < p.n_oct) {
        SmallOctArgs a{};
        a.pyr = d;
        a.o_first = o_small;
        a.cap_px = p.ow[o_small] * p.oh[o_small];
        for (int i = 0; i < s + 2; ++i) {
            a.radius[i] = (int)p.inc[i].size() / 2;
            for (size_t t = 0; t < p.inc[i].size(); ++t) a.taps[i][t] = (double)p.inc[i][t];
        }
        cuda_check(launch_small_octaves(a, c->stream), "small octaves");
        ++c->launches;
    }
}

static Counters* counters(dsift_ctx* c) { return c->counters.as<Counters>(); }

// NVTX range around a stage's launches (host enqueue; `ncu --nvtx --nvtx-include
// "K5 describe/"` selects that stage's kernels).  Free when no tool is attached.
struct NvtxStage {
    explicit NvtxStage(const char* name) { nvtxRangePushA(name); }
    ~NvtxStage() { nvtxRangePop(); }
    NvtxStage(const NvtxStage&) = delete;
    NvtxStage& operator=(const NvtxStage&) = delete;
};

static unsigned detect_tiles(const PyramidDesc& d, int* base, int* per_image) {
    int acc = 0;
    for (int o = 0; o < d.n_oct; ++o) {
        base[o] = acc;
        acc += d.oct[o].tiles_x * d.oct[o].tiles_y;
    }
    base[d.n_oct] = acc;
    *per_image = acc;
    return (unsigned)acc * (unsigned)d.batch;
}

bool tma_encode_3d_f32(CUtensorMap* map, const float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                       uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, uint32_t es01) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<Fn>(p);
    }
    if (!fn) return false;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {s1 * sizeof(float), s2 * sizeof(float)};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t es[3] = {es01, es01, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K2's TMA maps: per octave, the DoG stack {w, h, batch * (s+2)}, box
// {36, 34, s+2} (detect tile + halo, all DoG levels of one image).  They go
// into the kernel's __grid_constant__ parameter block.
static unsigned build_dog_maps(const PyramidDesc& d, CUtensorMap* maps) {
    unsigned mask = 0;
    for (int o = 0; o < d.n_oct && o < 32; ++o) {
        const OctaveDesc& od = d.oct[o];
        if (od.tiles_x == 0) continue;
        if (tma_encode_3d_f32(&maps[o], od.dog, (uint64_t)od.w, (uint64_t)od.h,
                              (uint64_t)d.batch * (uint64_t)(d.s + 2), (uint64_t)od.pitch,
                              (uint64_t)od.level_stride, 36u, 34u, (uint32_t)(d.s + 2)))
            mask |= 1u << o;
    }
    return mask;
}

static void run_detect(dsift_ctx* c, int raw_mode, long long cap) {
    const dsift_config& cf = c->cfg.c;
    DetectArgs a{};
    a.pyr = c->pyr;
    a.n_tiles = detect_tiles(c->pyr, a.oct_tile_base, &a.tiles_per_image);
    a.pre_gate = 0.5f * cf.contrast_threshold / cf.intervals;
    a.tma_mask = build_dog_maps(a.pyr, a.dog_maps);
    a.contrast_gate = double(cf.contrast_threshold) / cf.intervals;
    a.edge_r = cf.edge_ratio;
    a.max_iters = cf.max_refine_iters;
    a.raw_mode = raw_mode;
    c->det_kps.ensure(sizeof(DevKeypoint) * (size_t)cap);
    a.out = c->det_kps.as<DevKeypoint>();
    a.cap = cap;
    Counters* ctr = counters(c);
    a.err = &ctr->err;
    a.scan.total = &ctr->n_det;
    a.scan.cap = (unsigned long long)cap;
    if (raw_mode) {
        c->det_cand.ensure(sizeof(DevCandidate) * (size_t)cap);
        a.cand_out = c->det_cand.as<DevCandidate>();
    } else {
        a.cand_out = nullptr;
    }
    {   // count -> scan -> emit scratch: masks, counts, offsets, scan state
        const size_t nt = std::max(1u, a.n_tiles);
        const size_t masks = (sizeof(unsigned) * 256 * nt + 255) & ~size_t(255);
        const size_t cnts = (sizeof(unsigned) * nt + 255) & ~size_t(255);
        c->det_aux.ensure(masks + 2 * cnts + scan_state_bytes((long long)nt) + 256);
        char* base = c->det_aux.as<char>();
        a.hit_masks = reinterpret_cast<unsigned*>(base);
        a.tile_counts = reinterpret_cast<unsigned*>(base + masks);
        a.tile_offsets = reinterpret_cast<unsigned*>(base + masks + cnts);
        a.scan_state = base + masks + 2 * cnts;
    }
    cuda_check(launch_detect(a, c->stream), "detect");
    c->launches += 3;
}

// K3: refine the compacted candidates (count n_det) into compacted keypoints
// (count n_kp), candidate order kept.
static void run_refine(dsift_ctx* c, long long cap, int* keep = nullptr) {
    const dsift_config& cf = c->cfg.c;
    DetectArgs a{};
    a.pyr = c->pyr;
    a.contrast_gate = double(cf.contrast_threshold) / cf.intervals;
    a.edge_r = cf.edge_ratio;
    a.max_iters = cf.max_refine_iters;
    c->det_kps.ensure(sizeof(DevKeypoint) * (size_t)cap);
    a.out = c->det_kps.as<DevKeypoint>();
    a.cap = cap;
    Counters* ctr = counters(c);
    a.err = &ctr->err;
    const unsigned max_tiles = (unsigned)((cap + 255) / 256);
    c->ref_states.ensure(sizeof(unsigned long long) * (size_t)std::max(1u, max_tiles));
    cuda_check(cudaMemsetAsync(c->ref_states.as<void>(), 0, sizeof(unsigned long long) * std::max(1u, max_tiles),
                               c->stream), "memset");
    a.scan.states = c->ref_states.as<unsigned long long>();
    a.scan.ticket = &ctr->ref_ticket;
    a.scan.total = &ctr->n_kp;
    a.scan.cap = (unsigned long long)cap;
    cuda_check(launch_refine(a, c->det_cand.as<DevCandidate>(), &ctr->n_det, cap, keep, c->stream), "refine");
    ++c->launches;
}

static int orient_depth(const dsift_config& cf, const std::vector<dsift_keypoint>* kps, const Plan& p) {
    // window <= (2R+1)^2 with R = lround(4.5 sigma_rel); sigma_rel <= sigma0 * 2^((s+0.5)/s)
    double smax = cf.sigma0 * std::pow(2.0, (cf.intervals + 0.5) / cf.intervals) * 1.001;
    if (kps)
        for (const auto& k : *kps) {
            const double to_input = std::ldexp(1.0, k.octave) * (p.up ? 0.5 : 1.0);
            smax = std::max(smax, k.sigma / to_input);
        }
    const long long r = std::llround(4.5 * smax) + 1;
    const long long n = (2 * r + 1) * (2 * r + 1);
    int depth = 1;
    while ((1ll << depth) <= n) ++depth;
    return depth + 1;
}

static void run_orient(dsift_ctx* c, const DevKeypoint* kps, long long n_host, long long cap_kp,
                       DevKeypoint* out, long long cap_out, float* hist_out, int depth) {
    const dsift_config& cf = c->cfg.c;
    OrientArgs a{};
    a.pyr = c->pyr;
    a.kps = kps;
    Counters* ctr = counters(c);
    a.n_dev = &ctr->n_kp;
    a.n_host = n_host;
    a.bins = cf.orientation_bins;
    a.peak_ratio = cf.orientation_peak_ratio;
    a.depth = depth;
    a.out = out;
    a.cap = cap_out;
    a.err = &ctr->err;
    a.hist_out = hist_out;
    const long long nk = n_host >= 0 ? n_host : cap_kp;
    a.n_tiles = (unsigned)((nk + orient_tile_size() - 1) / orient_tile_size());
    a.scan.ticket = &ctr->ori_ticket;
    // K4b fan-out: per-keypoint peak angles and counts, then a look-back over
    // tiles of 256 keypoints
    const size_t nkp = (size_t)std::max<long long>(1, nk);
    const size_t ang_bytes = (sizeof(float) * nkp * (size_t)a.bins + 255) & ~size_t(255);
    const size_t cnt_bytes = (sizeof(int) * nkp + 255) & ~size_t(255);
    c->ori_aux.ensure(ang_bytes + cnt_bytes);
    a.angles = c->ori_aux.as<float>();
    a.counts = reinterpret_cast<int*>(c->ori_aux.as<char>() + ang_bytes);
    const unsigned emit_tiles = (unsigned)((nkp + 255) / 256);
    c->ori_states.ensure(sizeof(unsigned long long) * (size_t)emit_tiles);
    cuda_check(cudaMemsetAsync(c->ori_states.as<void>(), 0, sizeof(unsigned long long) * emit_tiles, c->stream),
               "memset");
    a.emit_scan.states = c->ori_states.as<unsigned long long>();
    a.emit_scan.ticket = &ctr->emit_ticket;
    a.emit_scan.total = &ctr->n_ori;
    a.emit_scan.cap = (unsigned long long)cap_out;
    cuda_check(cudaMemsetAsync(a.scan.ticket, 0, sizeof(unsigned), c->stream), "memset ticket");
    cuda_check(launch_orient(a, c->stream), "orient");
    c->launches += 2;
}

static int describe_axis(const dsift_config& cf, const std::vector<double>& dsp, double smax) {
    double fmax = 0.0;
    for (double f : dsp) fmax = std::max(fmax, f);
    const double bw = 3.0 * fmax * smax;
    const long long r = std::llround(bw * 5.0 * 0.5 * 1.4142135623730951) + 2;
    (void)cf;
    return (int)(2 * r + 3);
}

// Texture objects for K5's 2x2 gathers (tld4): [image][kMaxOctaves] handles
// on the device.  Per (image, octave) the s + 3 levels are one pitched 2D
// array of (s + 3) * level_rows rows (level_stride = pitch * level_rows); the
// pitch is a multiple of 128 bytes and every image's block 512-byte aligned.
// Returns nullptr (the kernel then gathers with plain loads) when a level
// stack exceeds the device's pitched-texture limits.
static const unsigned long long* ensure_gauss_textures(dsift_ctx* c) {
    if (!c->tex_gathers) return nullptr;
    const PyramidDesc& d = c->pyr;
    std::vector<long long> key{(long long)(uintptr_t)c->pyramid.as<void>(), d.batch, d.n_oct, d.s};
    for (int o = 0; o < d.n_oct; ++o) {
        key.push_back(d.oct[o].w);
        key.push_back(d.oct[o].h);
        key.push_back(d.oct[o].pitch);
    }
    if (key == c->gauss_tex_key) return c->gauss_tex_ok ? c->gauss_tex_dev.as<unsigned long long>() : nullptr;
    cuda_check(cudaStreamSynchronize(c->stream), "sync before texture rebuild");   // no launch still reads the old ones
    for (cudaTextureObject_t t : c->gauss_tex) cudaDestroyTextureObject(t);
    c->gauss_tex.clear();
    c->gauss_tex_key = key;
    c->gauss_tex_ok = false;
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, c->device), "cudaGetDeviceProperties");
    for (int o = 0; o < d.n_oct; ++o) {
        const OctaveDesc& od = d.oct[o];
        const size_t pitch_b = sizeof(float) * (size_t)od.pitch;
        if (od.w > prop.maxTexture2DLinear[0] || (d.s + 3) * (od.level_stride / od.pitch) > prop.maxTexture2DLinear[1] ||
            (long long)pitch_b > prop.maxTexture2DLinear[2] || pitch_b % prop.texturePitchAlignment != 0)
            return nullptr;
        const size_t align = std::max<size_t>(prop.textureAlignment, prop.texturePitchAlignment);
        for (int i = 0; i < d.batch; ++i)
            if ((uintptr_t)(od.gauss + (long long)i * d.gauss_img_stride(o)) % align != 0) return nullptr;
    }
    std::vector<unsigned long long> h((size_t)d.batch * kMaxOctaves, 0ull);
    for (int i = 0; i < d.batch; ++i)
        for (int o = 0; o < d.n_oct; ++o) {
            const OctaveDesc& od = d.oct[o];
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypePitch2D;
            rd.res.pitch2D.devPtr = od.gauss + (long long)i * d.gauss_img_stride(o);
            rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
            rd.res.pitch2D.width = (size_t)od.w;
            rd.res.pitch2D.height = (size_t)(d.s + 3) * (od.level_stride / od.pitch);
            rd.res.pitch2D.pitchInBytes = sizeof(float) * (size_t)od.pitch;
            cudaTextureDesc td{};
            td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
            td.filterMode = cudaFilterModePoint;
            td.readMode = cudaReadModeElementType;
            td.normalizedCoords = 0;
            cudaTextureObject_t t = 0;
            if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess || t == 0) {
                // out of texture resources: the kernels gather with plain loads
                (void)cudaGetLastError();
                for (cudaTextureObject_t u : c->gauss_tex) cudaDestroyTextureObject(u);
                c->gauss_tex.clear();
                return nullptr;
            }
            c->gauss_tex.push_back(t);
            h[(size_t)i * kMaxOctaves + o] = (unsigned long long)t;
        }
    c->gauss_tex_dev.ensure(sizeof(unsigned long long) * h.size());
    cuda_check(cudaMemcpyAsync(c->gauss_tex_dev.as<void>(), h.data(), sizeof(unsigned long long) * h.size(),
                               cudaMemcpyHostToDevice, c->stream),   // pageable: staged before returning
               "texture handles");
    c->gauss_tex_ok = true;
    return c->gauss_tex_dev.as<unsigned long long>();
}

static void run_describe(dsift_ctx* c, const DevKeypoint* kps, long long n_host, float* desc,
                         unsigned char* desc_u8, int raw_mode, double raw_scale, double smax,
                         const unsigned long long* n_dev) {
    const dsift_config& cf = c->cfg.c;
    DescArgs a{};
    a.pyr = c->pyr;
    a.gauss_tex = ensure_gauss_textures(c);
    a.kps = kps;
    a.n_dev = n_dev;
    a.n_host = n_host;
    a.n_dsp = (int)c->cfg.dsp.size();
    for (int i = 0; i < a.n_dsp; ++i) a.dsp[i] = c->cfg.dsp[i];
    a.clip = cf.descriptor_clip;
    a.raw_mode = raw_mode;
    a.raw_scale = raw_scale;
    std::vector<double> fs = raw_mode ? std::vector<double>{raw_scale} : c->cfg.dsp;
    a.max_axis = describe_axis(cf, fs, smax);
    {
        double fmax = 0.0;
        for (double f : fs) fmax = std::max(fmax, f);
        const double bw = 3.0 * fmax * smax;
        // a bin's leaves come from its 2x2 cells: < (2 bw + 2)^2 points; the exact
        // path's binary counter needs 2^depth above that (13 covers the defaults)
        const double leaves = (2.0 * bw + 2.0) * (2.0 * bw + 2.0);
        a.tree_depth = 13;
        while (a.tree_depth < 24 && std::ldexp(1.0, a.tree_depth) <= leaves) ++a.tree_depth;
        if (std::ldexp(1.0, a.tree_depth) <= leaves)
            invalid("descriptor: support window exceeds the per-bin tree capacity of this build");
    }
    a.chunk_rows = 8;
    {
        const long long cap_n = n_host >= 0 ? n_host : c->cap_ori;
        c->trig.ensure(sizeof(double2) * (size_t)std::max<long long>(1, cap_n));
        cuda_check(launch_trig(kps, n_dev, n_host, c->trig.as<double2>(), cap_n, c->stream), "trig");
        ++c->launches;
        a.trig = c->trig.as<double2>();
    }
    a.desc = desc;
    a.desc_u8 = desc_u8;
    a.err = &counters(c)->err;
    if (raw_mode) {
        const size_t smem = describe_smem_bytes(a.max_axis, a.chunk_rows, 1, a.tree_depth);
        if (smem > 200 * 1024) invalid("descriptor: lattice too large for shared memory");
        int grid = c->sm_count * 4;
        if (n_host >= 0) grid = (int)std::max<long long>(1, std::min<long long>(grid, n_host));
        cuda_check(launch_describe(a, grid, c->stream), "describe exact");
        ++c->launches;
        return;
    }
    // certified stream kernel over every keypoint, then the exact kernel over
    // the (rare) keypoints whose certificate failed
    const long long cap_n = n_host >= 0 ? n_host : c->cap_ori;
    c->slow.ensure(sizeof(int) * (size_t)std::max<long long>(1, cap_n));
    Counters* ctr = counters(c);
    a.slow_out = c->slow.as<int>();
    a.slow_count = &ctr->n_slow;
    a.fix_count = &ctr->n_fixed;
    a.ticket = &ctr->desc_ticket;
    a.lattice = &ctr->lattice;
    a.lattice_in = &ctr->lattice_in;
    a.slow_cap = cap_n;
    a.force_slow = c->force_exact;
#ifdef DSIFT_NONDET_TEST_HOOK
    // the reference's negative control (detsum.cpp:73-109): a test-only build
    // whose histogram sums depend on scheduling when DSIFT_NONDET=1
    {
        const char* v = std::getenv("DSIFT_NONDET");
        a.nondet = v != nullptr && v[0] == '1';
    }
#endif
    DescArgs af = a;
    af.chunk_rows = 6;   // the stream kernel's in-place exact recompute works in 6-row chunks
    {
        double fmax = 0.0;
        for (double f : fs) fmax = std::max(fmax, f);
        af.max_span = 2 * (int)std::ceil(2.5 * 3.0 * fmax * smax) + 8;
    }
    const size_t smem_exact = describe_smem_bytes(a.max_axis, a.chunk_rows, a.n_dsp, a.tree_depth);
    if (smem_exact > 200 * 1024) invalid("descriptor: lattice too large for shared memory");
    const size_t smem_s = std::max(describe_stream_smem_bytes(af.max_span, a.n_dsp),
                                   describe_stream_exact_smem_bytes(af.max_axis, af.chunk_rows, a.n_dsp, a.tree_depth));
    if (smem_s > 200 * 1024) invalid("descriptor: lattice too large for shared memory");
    const int per_sm = std::max(1, describe_stream_blocks_per_sm(smem_s));
    int grid = c->sm_count * per_sm;
    if (n_host >= 0) grid = (int)std::max<long long>(1, std::min<long long>(grid, n_host));
    cuda_check(cudaMemsetAsync(af.ticket, 0, sizeof(unsigned), c->stream), "memset ticket");
    cuda_check(launch_describe_stream(af, grid, c->stream), "describe stream");
    DescArgs b = a;
    b.slow_list = c->slow.as<int>();
    b.n_slow = &ctr->n_slow;
    int grid2 = c->sm_count * 4;
    if (n_host >= 0) grid2 = (int)std::max<long long>(1, std::min<long long>(grid2, n_host));
    cuda_check(launch_describe(b, grid2, c->stream), "describe exact");
    c->launches += 2;
}

static void ensure_counters(dsift_ctx* c) {
    c->counters.ensure(sizeof(Counters));
}

static void reset_counters(dsift_ctx* c) {
    cuda_check(cudaMemsetAsync(c->counters.as<void>(), 0, sizeof(Counters), c->stream), "memset");
}

// Stage-level input (one image): host images go through the context's own
// staging buffer.
static const float* stage_input(dsift_ctx* c, const float* images, int n, int w, int h, int flags) {
    if (flags & DSIFT_INPUT_DEVICE) return images;
    const size_t bytes = sizeof(float) * (size_t)n * w * h;
    c->stage_in.ensure(bytes);
    cuda_check(cudaMemcpyAsync(c->stage_in.as<void>(), images, bytes, cudaMemcpyHostToDevice, c->stream), "H2D");
    return c->stage_in.as<float>();
}

static void ensure_events(dsift_result* r) {
    if (!r->done) cuda_check(cudaEventCreateWithFlags(&r->done, cudaEventDisableTiming), "event");
    if (!r->input_free) cuda_check(cudaEventCreateWithFlags(&r->input_free, cudaEventDisableTiming), "event");
}

// Per-group capacities (automatic: from the input size, x cap_scale after an
// overflow; or the caller's dsift_set_capacity).
static void group_caps(dsift_ctx* c, Group& g) {
    const long long n = (long long)g.idx.size();
    auto cap = [&](double factor) -> long long {
        if (c->cap_override > 0) return c->cap_override;
        const double px = (double)g.w * g.h * c->cap_scale;
        return std::max<long long>((long long)(4096 * c->cap_scale), (long long)(px * factor));
    };
    g.cap_det = n * cap(1.0 / 12.0);   // candidates (extrema)
    g.cap_ori = n * cap(1.0 / 16.0);   // oriented keypoints
}

// The pipeline for one size group: K1 pyramid -> K2/K3 detect + refine -> K4
// orientation + fan-out -> K7 canonical sort -> K5/K6 descriptors, all on the
// context stream.  Keypoints / descriptors / per-image offsets go to the given
// output pointers.
static void run_group(dsift_ctx* c, dsift_result* r, const Group& g, dsift_keypoint* out_kps, float* out_desc,
                      unsigned char* out_u8, long long* out_offs) {
    const int n = (int)g.idx.size();
    c->plan = make_plan(c->cfg, g.w, g.h);
    c->batch = n;
    build_pyramid_desc(c);
    reset_counters(c);
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[0], c->stream), "event");
    {
        NvtxStage r("K1 pyramid");
        launch_pyramid(c, g.dev);
    }
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[1], c->stream), "event");
    c->cap_det = g.cap_det;
    c->cap_ori = g.cap_ori;
    {
        NvtxStage r("K2-K3 detect");
        run_detect(c, 1, c->cap_det);   // K2: compacted extrema
        run_refine(c, c->cap_det);      // K3: one thread per candidate
    }
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[2], c->stream), "event");
    c->ori_kps.ensure(sizeof(DevKeypoint) * (size_t)c->cap_ori);
    {
        NvtxStage r("K4 orient");
        run_orient(c, c->det_kps.as<DevKeypoint>(), -1, c->cap_det, c->ori_kps.as<DevKeypoint>(), c->cap_ori, nullptr,
                   orient_depth(c->cfg.c, nullptr, c->plan));
    }
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[3], c->stream), "event");
    // canonical order (K7, hand-written bucket sort over the actual count)
    const long long cap = c->cap_ori;
    SortGeom sg;
    sg.s = c->plan.s;
    sg.rows = c->plan.in_h;
    sg.per_image = (unsigned)(c->plan.n_oct * c->plan.s * c->plan.in_h);
    c->sort_work.ensure(sort_work_bytes(cap, sg, n));
    c->sorted_kps.ensure(sizeof(DevKeypoint) * (size_t)cap);
    Counters* ctr = counters(c);
    {
        NvtxStage r("K7 sort");
        cuda_check(launch_canonical_sort(c->ori_kps.as<DevKeypoint>(), &ctr->n_ori, cap, sg, c->sort_work.as<void>(),
                                         c->sorted_kps.as<DevKeypoint>(), out_kps, n, out_offs, c->stream,
                                         &c->launches),
                   "sort");
    }
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[4], c->stream), "event");
    const double smax = c->cfg.c.sigma0 * std::pow(2.0, (c->cfg.c.intervals + 0.5) / c->cfg.c.intervals) * 1.001;
    {
        NvtxStage r("K5 describe");
        run_describe(c, c->sorted_kps.as<DevKeypoint>(), -1, out_desc, out_u8, 0, 0.0, smax, &ctr->n_ori);
    }
    if (c->profiling) cuda_check(cudaEventRecord(c->stage_ev[5], c->stream), "event");
    cuda_check(launch_fold_totals(ctr, r->totals.as<BatchTotals>(), c->stream), "fold");
    ++c->launches;
}

// Runs every group of r (first run or a capacity replay) and, for a ragged
// batch, gathers the groups' staged outputs into batch order.
static void run_batch(dsift_ctx* c, dsift_result* r) {
    set_device(c);
    ensure_counters(c);
    r->pending = r->ready = false;
    r->total = 0;
    long long rows = 0, offs = 0;
    size_t pyr_max = 0;
    for (Group& g : r->groups) {
        group_caps(c, g);
        g.stage_base = rows;
        g.offs_base = offs;
        rows += g.cap_ori;
        offs += (long long)g.idx.size() + 1;
        const Plan p = make_plan(c->cfg, g.w, g.h);
        size_t bytes = 0;
        for (int o = 0; o < p.n_oct; ++o) {
            const size_t lv = sizeof(float) * (size_t)p.pitch[o] * level_rows(p.pitch[o], p.oh[o]) * g.idx.size();
            bytes += ((lv * (p.s + 3) + 511) & ~size_t(511)) + ((lv * (p.s + 2) + 511) & ~size_t(511));
        }
        pyr_max = std::max(pyr_max, bytes);
    }
    c->pyramid.ensure(pyr_max);   // one allocation for every group of the batch
    r->totals.ensure(sizeof(BatchTotals));
    cuda_check(cudaMemsetAsync(r->totals.as<void>(), 0, sizeof(BatchTotals), c->stream), "memset");
    r->offsets.ensure(sizeof(long long) * (size_t)(r->batch + 1));
    if (r->direct) {
        const Group& g = r->groups[0];
        r->pub_kps.ensure(sizeof(dsift_keypoint) * (size_t)g.cap_ori);
        r->desc.ensure(sizeof(float) * kDescDim * (size_t)g.cap_ori);
        r->desc_u8.ensure((size_t)kDescDim * (size_t)g.cap_ori);
        run_group(c, r, g, r->pub_kps.as<dsift_keypoint>(), r->desc.as<float>(), r->desc_u8.as<unsigned char>(),
                  r->offsets.as<long long>());
        cuda_check(cudaEventRecord(r->input_free, c->stream), "event");
    } else {
        r->stage_kps.ensure(sizeof(dsift_keypoint) * (size_t)rows);
        r->stage_desc.ensure(sizeof(float) * kDescDim * (size_t)rows);
        r->stage_u8.ensure((size_t)kDescDim * (size_t)rows);
        r->stage_offs.ensure(sizeof(long long) * (size_t)offs);
        for (const Group& g : r->groups)
            run_group(c, r, g, r->stage_kps.as<dsift_keypoint>() + g.stage_base,
                      r->stage_desc.as<float>() + g.stage_base * kDescDim,
                      r->stage_u8.as<unsigned char>() + g.stage_base * kDescDim,
                      r->stage_offs.as<long long>() + g.offs_base);
        cuda_check(cudaEventRecord(r->input_free, c->stream), "event");
        // batch index -> (staging offsets entry, staging row base)
        std::vector<long long>& map = r->h_map;
        map.assign(2 * (size_t)r->batch, 0);
        for (const Group& g : r->groups)
            for (size_t j = 0; j < g.idx.size(); ++j) {
                map[2 * (size_t)g.idx[j]] = g.offs_base + (long long)j;
                map[2 * (size_t)g.idx[j] + 1] = g.stage_base;
            }
        r->map.ensure(sizeof(long long) * map.size());
        cuda_check(cudaMemcpyAsync(r->map.as<void>(), map.data(), sizeof(long long) * map.size(),
                                   cudaMemcpyHostToDevice, c->stream), "H2D");
        r->pub_kps.ensure(sizeof(dsift_keypoint) * (size_t)rows);
        r->desc.ensure(sizeof(float) * kDescDim * (size_t)rows);
        r->desc_u8.ensure((size_t)kDescDim * (size_t)rows);
        cuda_check(launch_ragged_gather(r->map.as<long long>(), r->stage_offs.as<long long>(), r->batch,
                                        r->stage_kps.as<dsift_keypoint>(), r->stage_desc.as<float>(),
                                        r->stage_u8.as<unsigned char>(), r->offsets.as<long long>(),
                                        r->pub_kps.as<dsift_keypoint>(), r->desc.as<float>(),
                                        r->desc_u8.as<unsigned char>(), c->stream),
                   "ragged gather");
        c->launches += 2;
    }
    cuda_check(cudaEventRecord(r->done, c->stream), "event");
    r->pending = true;
}

// Extraction entry: validates every image (reference messages, before any
// work is enqueued), groups the batch by image size (first-occurrence
// order), stages host / scattered inputs contiguously per group and runs it.
static void extract_images(dsift_ctx* c, const dsift_image* imgs, int n, int flags, dsift_result* r) {
    if (!r) r = c->cur;
    r->pending = r->ready = false;   // a failed submit leaves no stale result behind
    r->total = 0;
    r->batch = 0;
    r->groups.clear();
    if (n <= 0) invalid("extract: batch must contain at least one image");
    if (!imgs) invalid("extract: null image pointer");
    set_device(c);
    ensure_events(r);
    std::vector<Group> groups;
    for (int i = 0; i < n; ++i) {
        if (!imgs[i].data) invalid("extract: null image pointer");
        (void)make_plan(c->cfg, imgs[i].width, imgs[i].height);   // throws the reference's message
        auto it = std::find_if(groups.begin(), groups.end(),
                               [&](const Group& g) { return g.w == imgs[i].width && g.h == imgs[i].height; });
        if (it == groups.end()) {
            groups.emplace_back();
            groups.back().w = imgs[i].width;
            groups.back().h = imgs[i].height;
            it = groups.end() - 1;
        }
        it->idx.push_back(i);
    }
    const bool device = (flags & DSIFT_INPUT_DEVICE) != 0;
    bool contiguous = groups.size() == 1;
    if (contiguous) {
        const size_t px = (size_t)groups[0].w * groups[0].h;
        for (int i = 1; i < n && contiguous; ++i) contiguous = imgs[i].data == imgs[0].data + (size_t)i * px;
    }
    r->direct = groups.size() == 1;
    if (device && contiguous) {
        groups[0].dev = imgs[0].data;   // zero-copy: the caller's batch (kept valid until result_sync)
    } else {
        size_t total_px = 0;
        for (const Group& g : groups) total_px += (size_t)g.w * g.h * g.idx.size();
        r->input.ensure(sizeof(float) * total_px);
        cudaStream_t cs = device ? c->stream : c->copy_stream;
        if (!device) cuda_check(cudaStreamWaitEvent(cs, r->input_free, 0), "wait");   // previous batch done with input[]
        float* dst = r->input.as<float>();
        for (Group& g : groups) {
            g.dev = dst;
            const size_t px = (size_t)g.w * g.h;
            for (int i : g.idx) {
                cuda_check(cudaMemcpyAsync(dst, imgs[i].data, sizeof(float) * px,
                                           device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, cs),
                           "copy input");
                dst += px;
            }
        }
        if (!device) {
            cuda_check(cudaEventRecord(r->input_free, cs), "event");   // reused as "input staged"
            cuda_check(cudaStreamWaitEvent(c->stream, r->input_free, 0), "wait");
        }
    }
    r->batch = n;
    r->retries = 0;
    r->groups = std::move(groups);
    run_batch(c, r);
}

static void extract_batch(dsift_ctx* c, const float* images, int n, int w, int h, int flags) {
    if (n <= 0) invalid("extract: batch must contain at least one image");
    if (!images) invalid("extract: null image pointer");
    std::vector<dsift_image> v((size_t)n);
    for (int i = 0; i < n; ++i) v[(size_t)i] = dsift_image{images + (size_t)i * (size_t)std::max(0, w) * std::max(0, h), w, h};
    extract_images(c, v.data(), n, flags, nullptr);
}

static void result_sync(dsift_ctx* c, dsift_result* r) {
    if (!r->pending && !r->ready) throw Error{DSIFT_ESTATE, "result: no extract issued"};
    if (r->ready) return;
    set_device(c);
    for (;;) {
        cuda_check(cudaEventSynchronize(r->done), "sync");
        cuda_check(cudaGetLastError(), "async kernel error");
        BatchTotals t{};
        cuda_check(cudaMemcpy(&t, r->totals.as<void>(), sizeof(t), cudaMemcpyDeviceToHost), "D2H");
        r->pending = false;
        if (t.err & kErrHistogramRange)   // same text as detsum.cpp:140 (std::out_of_range)
            throw Error{DSIFT_ERANGE, "histogram: bin index out of range"};
        const unsigned list_err = kErrKeypointCapacity | kErrOrientedCapacity | kErrCandidateCapacity;
        if ((t.err & list_err) && c->cap_override == 0 && r->retries < 4) {
            // automatic capacity overflowed: grow it and replay the batch (the
            // inputs are still on the device), so the caller still gets every keypoint
            c->cap_scale *= 4.0;
            ++r->retries;
            run_batch(c, r);
            continue;
        }
        if (t.err) {
            std::string m = "device work list overflow:";
            if (t.err & kErrKeypointCapacity) m += " keypoints";
            if (t.err & kErrOrientedCapacity) m += " oriented keypoints";
            if (t.err & kErrCandidateCapacity) m += " candidates";
            if (t.err & kErrDescriptorLattice) m += " descriptor lattice";
            m += " (raise dsift_set_capacity)";
            throw Error{DSIFT_ECAPACITY, m};
        }
        r->slow = t.slow;
        r->lattice = t.lattice;
        r->lattice_in = t.lattice_in;
        break;
    }
    r->h_offsets.assign((size_t)r->batch + 1, 0);
    cuda_check(cudaMemcpy(r->h_offsets.data(), r->offsets.as<void>(), sizeof(long long) * (r->batch + 1),
                          cudaMemcpyDeviceToHost), "D2H");
    r->total = r->h_offsets[(size_t)r->batch];
    r->ready = true;
}

static void result_sync(dsift_ctx* c) { result_sync(c, c->cur); }

// ---- SHA-256 / DSF1 (sha256.cpp, core.cpp:153-196), host side -------------------------
static void sha256(const uint8_t* data, size_t n, char* hex) {
    static const uint32_t K[64] = {
        0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
        0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
        0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
        0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
        0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
        0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
        0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
        0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};
    uint32_t st[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    auto rot = [](uint32_t x, int r) { return (x >> r) | (x << (32 - r)); };
    auto block = [&](const uint8_t* p) {
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
        for (int i = 16; i < 64; ++i)
            w[i] = w[i - 16] + (rot(w[i - 15], 7) ^ rot(w[i - 15], 18) ^ (w[i - 15] >> 3)) + w[i - 7] +
                   (rot(w[i - 2], 17) ^ rot(w[i - 2], 19) ^ (w[i - 2] >> 10));
        uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
        for (int i = 0; i < 64; ++i) {
            const uint32_t t1 = h + (rot(e, 6) ^ rot(e, 11) ^ rot(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + w[i];
            const uint32_t t2 = (rot(a, 2) ^ rot(a, 13) ^ rot(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
    };
    size_t i = 0;
    for (; i + 64 <= n; i += 64) block(data + i);
    uint8_t tail[128] = {0};
    const size_t rem = n - i;
    std::memcpy(tail, data + i, rem);
    tail[rem] = 0x80;
    const size_t tl = rem + 9 <= 64 ? 64 : 128;
    const uint64_t bits = (uint64_t)n * 8u;
    for (int k = 0; k < 8; ++k) tail[tl - 1 - k] = (uint8_t)(bits >> (8 * k));
    block(tail);
    if (tl == 128) block(tail + 64);
    for (int k = 0; k < 8; ++k) std::snprintf(hex + 8 * k, 9, "%08x", st[k]);
    hex[64] = 0;
}

}  // namespace dsift

// ================================ C ABI =========================================
extern "C" {

int dsift_abi_version(void) { return DSIFT_ABI_VERSION; }

const char* dsift_strerror(int code) {
    switch (code) {
        case DSIFT_OK: return "ok";
        case DSIFT_EINVAL: return "invalid argument";
        case DSIFT_ECAPACITY: return "device capacity exceeded";
        case DSIFT_ECUDA: return "CUDA error";
        case DSIFT_ENOMEM: return "out of memory";
        case DSIFT_ESTATE: return "invalid call order";
        case DSIFT_ERANGE: return "out of range";
        case DSIFT_EIO: return "image I/O error";
        case DSIFT_EGEOM: return "degenerate geometry";
        default: return "unknown error";
    }
}

const char* dsift_last_error(void) { return g_err.c_str(); }

void dsift_config_default(dsift_config* c) {
    c->sigma0 = 1.6f;
    c->intervals = 3;
    c->assumed_blur = 0.5f;
    c->contrast_threshold = 0.04f;
    c->edge_ratio = 10.0f;
    c->max_refine_iters = 5;
    c->upsample_pixel_limit = 4000000;
    c->dsp_scales = kDefaultDsp;
    c->n_dsp_scales = 5;
    c->descriptor_clip = 0.2f;
    c->orientation_bins = 36;
    c->orientation_peak_ratio = 0.8f;
    c->num_octaves = 0;
}

int dsift_config_validate(const dsift_config* c) {
    return guard([&] {
        if (!c) invalid("config: null");
        validate(*c);
    });
}

int dsift_create(int device, const dsift_config* cfg, dsift_ctx** out) {
    return guard([&] {
        if (!out) invalid("create: null output");
        dsift_config c;
        if (cfg) c = *cfg; else dsift_config_default(&c);
        validate(c);
        auto ctx = std::make_unique<dsift_ctx>();
        ctx->device = device;
        ctx->cfg.c = c;
        ctx->cfg.dsp.assign(c.dsp_scales, c.dsp_scales + c.n_dsp_scales);
        ctx->cfg.c.dsp_scales = ctx->cfg.dsp.data();
        int ndev = 0;
        cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) throw Error{DSIFT_ECUDA, "create: no such CUDA device"};
        set_device(ctx.get());
        cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
        cuda_check(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "stream");
        ctx->stream = ctx->own_stream;
        ctx->def.owner = ctx.get();
        ensure_events(&ctx->def);
        cuda_check(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device), "attr");
        ensure_counters(ctx.get());
        *out = ctx.release();
    });
}

void dsift_destroy(dsift_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaStreamSynchronize(c->copy_stream);
    if (c->def.done) cudaEventDestroy(c->def.done);
    if (c->def.input_free) cudaEventDestroy(c->def.input_free);
    for (auto& e : c->stage_ev)
        if (e) cudaEventDestroy(e);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    for (cudaTextureObject_t t : c->gauss_tex) cudaDestroyTextureObject(t);
    delete c;
}

int dsift_set_stream(dsift_ctx* c, void* s) {
    return guard([&] {
        if (!c) invalid("null context");
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    });
}

int dsift_set_capacity(dsift_ctx* c, int64_t cap) {
    return guard([&] {
        if (!c) invalid("null context");
        if (cap < 0) invalid("capacity must be >= 0");
        c->cap_override = cap;
    });
}

int dsift_extract_batch(dsift_ctx* c, const float* images, int n, int w, int h, int flags) {
    return guard([&] {
        if (!c) invalid("null context");
        extract_batch(c, images, n, w, h, flags);
    });
}

int dsift_extract(dsift_ctx* c, const float* image, int w, int h, int flags) {
    return dsift_extract_batch(c, image, 1, w, h, flags);
}

int dsift_extract_images(dsift_ctx* c, const dsift_image* images, int n, int flags) {
    return guard([&] {
        if (!c) invalid("null context");
        if (n > 65535) invalid("extract: at most 65535 images per call");
        extract_images(c, images, n, flags, nullptr);
    });
}

int dsift_result_create(dsift_ctx* c, dsift_result** out) {
    return guard([&] {
        if (!c || !out) invalid("null argument");
        set_device(c);
        auto r = std::make_unique<dsift_result>();
        r->owner = c;
        ensure_events(r.get());
        *out = r.release();
    });
}

void dsift_result_destroy(dsift_result* r) {
    if (!r) return;
    dsift_ctx* c = r->owner;
    if (c && r == &c->def) return;   // the context's own result lives with the context
    if (c) {
        cudaSetDevice(c->device);
        if (c->cur == r) c->cur = &c->def;
    }
    if (r->done) {
        cudaEventSynchronize(r->done);
        cudaEventDestroy(r->done);
    }
    if (r->input_free) {
        cudaEventSynchronize(r->input_free);
        cudaEventDestroy(r->input_free);
    }
    delete r;
}

int dsift_result_select(dsift_ctx* c, dsift_result* r) {
    return guard([&] {
        if (!c) invalid("null context");
        if (r && r->owner != c) invalid("result: belongs to another context");
        c->cur = r ? r : &c->def;
    });
}

// ---- matching (match.cpp:77-119) --------------------------------------------
int dsift_ratio_match(dsift_ctx* c, const float* desc_a, int64_t n_a, const float* desc_b, int64_t n_b, int dim_a,
                      int dim_b, float ratio, int flags, dsift_match* out, int64_t cap, int64_t* n_pairs,
                      int64_t* putative_a, int64_t* putative_b) {
    return guard([&] {
        if (!c) invalid("null context");
        if (dim_a != dim_b) invalid("ratio_match: dimension mismatch");
        if (!(ratio > 0.0f) || ratio > 1.0f) invalid("ratio_match: ratio must be in (0,1]");
        if (dim_a != kDescDim) invalid("ratio_match: this build matches 128-d descriptors");
        if (n_a < 0 || n_b < 0) invalid("ratio_match: negative size");
        if (n_pairs) *n_pairs = 0;
        if (putative_a) *putative_a = 0;
        if (putative_b) *putative_b = 0;
        if (n_a < 2 || n_b < 2) return;   // match.cpp:85
        if ((!desc_a || !desc_b)) invalid("ratio_match: null descriptors");
        set_device(c);
        const float* A = desc_a;
        const float* B = desc_b;
        const size_t ba = sizeof(float) * kDescDim * (size_t)n_a, bb = sizeof(float) * kDescDim * (size_t)n_b;
        if (!(flags & DSIFT_INPUT_DEVICE)) {
            c->match_in.ensure(ba + bb + 256);
            char* p = c->match_in.as<char>();
            cuda_check(cudaMemcpyAsync(p, desc_a, ba, cudaMemcpyHostToDevice, c->stream), "H2D");
            cuda_check(cudaMemcpyAsync(p + ((ba + 255) & ~size_t(255)), desc_b, bb, cudaMemcpyHostToDevice, c->stream),
                       "H2D");
            A = reinterpret_cast<const float*>(p);
            B = reinterpret_cast<const float*>(p + ((ba + 255) & ~size_t(255)));
        }
        c->match_scratch.ensure(match_scratch_bytes(n_a, n_b));
        c->match_best.ensure(sizeof(int) * (size_t)(n_a + n_b) + sizeof(float) * (size_t)n_a + 512);
        int* best_a = c->match_best.as<int>();
        int* best_b = best_a + n_a;
        float* dist_a = reinterpret_cast<float*>(best_b + n_b);
        cuda_check(launch_ratio_match(A, n_a, B, n_b, ratio, c->match_scratch.as<void>(), best_a, best_b, dist_a,
                                      c->stream),
                   "ratio_match");
        c->launches += 5;
        std::vector<int> ha((size_t)n_a), hb((size_t)n_b);
        std::vector<float> hd((size_t)n_a);
        cuda_check(cudaMemcpyAsync(ha.data(), best_a, sizeof(int) * n_a, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hb.data(), best_b, sizeof(int) * n_b, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hd.data(), dist_a, sizeof(float) * n_a, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        // putative counts and the mutual filter in index order (match.cpp:109-117)
        int64_t pa = 0, pb = 0, np = 0;
        for (int64_t i = 0; i < n_a; ++i) pa += ha[i] >= 0;
        for (int64_t j = 0; j < n_b; ++j) pb += hb[j] >= 0;
        for (int64_t i = 0; i < n_a; ++i) {
            const int j = ha[i];
            if (j >= 0 && hb[j] == (int)i) {
                if (out && np < cap) out[np] = dsift_match{(int32_t)i, (int32_t)j, hd[i]};
                ++np;
            }
        }
        if (n_pairs) *n_pairs = np;
        if (putative_a) *putative_a = pa;
        if (putative_b) *putative_b = pb;
    });
}

// ---- robust homography (geom.cpp:104-320) ------------------------
// Hypothesis samples: the reference's sequential seeded stream (geom.cpp:193-232),
// drawn here on the host exactly as the reference draws them.
namespace {
struct SplitMix64 {
    uint64_t state;
    uint64_t next() {
        uint64_t z = (state += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
};

std::vector<int4> magsac_samples(const double* m, int64_t n, int iterations, uint64_t seed) {
    SplitMix64 rng{seed};
    std::vector<int4> out;
    out.reserve((size_t)iterations);
    for (int it = 0; it < iterations; ++it) {
        int sample[4] = {-1, -1, -1, -1};
        bool ok = false;
        for (int attempt = 0; attempt < 64 && !ok; ++attempt) {
            int filled = 0, guard = 0;
            while (filled < 4 && guard < 256) {
                ++guard;
                const int idx = static_cast<int>(rng.next() % (uint64_t)n);
                bool dup = false;
                for (int k = 0; k < filled; ++k) dup |= (sample[k] == idx);
                if (!dup) sample[filled++] = idx;
            }
            if (filled < 4) break;
            double xs[4], ys[4], xd[4], yd[4];
            for (int k = 0; k < 4; ++k) {
                xs[k] = m[4 * sample[k]];
                ys[k] = m[4 * sample[k] + 1];
                xd[k] = m[4 * sample[k] + 2];
                yd[k] = m[4 * sample[k] + 3];
            }
            double span = 1e-12;
            for (int p = 0; p < 4; ++p)
                for (int q = p + 1; q < 4; ++q)
                    span = std::max({span, std::fabs(xs[p] - xs[q]), std::fabs(ys[p] - ys[q])});
            bool degenerate = false;
            for (int p = 0; p < 4 && !degenerate; ++p)
                for (int q = p + 1; q < 4 && !degenerate; ++q)
                    for (int r = q + 1; r < 4 && !degenerate; ++r) {
                        const double area = (xs[q] - xs[p]) * (ys[r] - ys[p]) - (xs[r] - xs[p]) * (ys[q] - ys[p]);
                        const double area_d = (xd[q] - xd[p]) * (yd[r] - yd[p]) - (xd[r] - xd[p]) * (yd[q] - yd[p]);
                        if (std::fabs(area) < 1e-8 * span * span || std::fabs(area_d) < 1e-8 * span * span)
                            degenerate = true;
                    }
            ok = !degenerate;
        }
        out.push_back(ok ? make_int4(sample[0], sample[1], sample[2], sample[3]) : make_int4(-1, -1, -1, -1));
    }
    return out;
}
}  // namespace

int dsift_magsac_lite(dsift_ctx* c, const double* matches, int64_t n, int32_t iterations, double tau, uint64_t seed,
                      dsift_magsac_result* res, uint8_t* inlier_mask) {
    return guard([&] {
        if (!c) invalid("null context");
        if (n < 4) invalid("magsac_lite: need at least 4 correspondences");
        if (!(tau > 0.0)) invalid("magsac_lite: tau must be > 0");
        if (iterations < 1) invalid("magsac_lite: iterations must be >= 1");
        if (!matches || !res) invalid("magsac_lite: null argument");
        if (n > (int64_t)INT32_MAX) invalid("magsac_lite: too many correspondences");
        set_device(c);
        const std::vector<int4> samples = magsac_samples(matches, n, iterations, seed);
        const size_t bm = sizeof(double) * 4 * (size_t)n, bs = sizeof(int4) * (size_t)iterations;
        c->geom_in.ensure(bm + bs + (size_t)n + 1024);
        char* p = c->geom_in.as<char>();
        double* dm = reinterpret_cast<double*>(p);
        int4* ds = reinterpret_cast<int4*>(p + ((bm + 255) & ~size_t(255)));
        unsigned char* dmask = reinterpret_cast<unsigned char*>(p + ((bm + 255) & ~size_t(255)) + ((bs + 255) & ~size_t(255)));
        c->geom_scratch.ensure(magsac_scratch_bytes(n, iterations));
        c->geom_out.ensure(256);
        int* out_i = c->geom_out.as<int>();
        double* out_d = reinterpret_cast<double*>(c->geom_out.as<char>() + 64);
        cuda_check(cudaMemcpyAsync(dm, matches, bm, cudaMemcpyHostToDevice, c->stream), "H2D");
        cuda_check(cudaMemcpyAsync(ds, samples.data(), bs, cudaMemcpyHostToDevice, c->stream), "H2D");
        cuda_check(launch_magsac(dm, n, ds, iterations, tau * tau, c->geom_scratch.as<void>(), dmask, out_i, out_d,
                                 c->stream),
                   "magsac");
        c->launches += 3;
        int hi[2];
        double hd[10];
        cuda_check(cudaMemcpyAsync(hi, out_i, sizeof(hi), cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaMemcpyAsync(hd, out_d, sizeof(hd), cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (inlier_mask)
            cuda_check(cudaMemcpyAsync(inlier_mask, dmask, (size_t)n, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        res->success = hi[0];
        res->best_iteration = hi[1];
        res->score = hi[0] ? hd[0] : 0.0;
        const double ident[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
        for (int i = 0; i < 9; ++i) res->h[i] = hi[0] ? hd[1 + i] : ident[i];
        if (!hi[0]) res->best_iteration = hi[1] >= 0 ? hi[1] : -1;
    });
}

int dsift_dlt_homography(dsift_ctx* c, const double* matches, int64_t n, const double* weights, double* h_out) {
    return guard([&] {
        if (!c) invalid("null context");
        if (n < 4) invalid("dlt: need at least 4 correspondences");
        if (!matches || !h_out) invalid("dlt: null argument");
        if (n > (int64_t)INT32_MAX) invalid("dlt: too many correspondences");
        set_device(c);
        const size_t bm = sizeof(double) * 4 * (size_t)n, bw = weights ? sizeof(double) * (size_t)n : 0;
        c->geom_in.ensure(bm + bw + 1024);
        char* p = c->geom_in.as<char>();
        double* dm = reinterpret_cast<double*>(p);
        double* dw = weights ? reinterpret_cast<double*>(p + ((bm + 255) & ~size_t(255))) : nullptr;
        c->geom_scratch.ensure(dlt_scratch_bytes(n));
        c->geom_out.ensure(256);
        int* st = c->geom_out.as<int>();
        double* out = reinterpret_cast<double*>(c->geom_out.as<char>() + 64);
        cuda_check(cudaMemcpyAsync(dm, matches, bm, cudaMemcpyHostToDevice, c->stream), "H2D");
        if (dw) cuda_check(cudaMemcpyAsync(dw, weights, bw, cudaMemcpyHostToDevice, c->stream), "H2D");
        cuda_check(launch_dlt(dm, dw, (int)n, c->geom_scratch.as<void>(), st, out, c->stream), "dlt");
        c->launches += 1;
        int status = 0;
        cuda_check(cudaMemcpyAsync(&status, st, sizeof(int), cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaMemcpyAsync(h_out, out, sizeof(double) * 9, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        if (!status) throw Error{DSIFT_EGEOM, "dlt: degenerate or non-finite solution"};
    });
}

// corner_error (geom.cpp:322-333): four corners, host arithmetic (std::hypot).
int dsift_corner_error(const double* h_est, const double* h_gt, double width, double height, double* out) {
    return guard([&] {
        if (!h_est || !h_gt || !out) invalid("corner_error: null argument");
        const double corners[4][2] = {{0, 0}, {width, 0}, {width, height}, {0, height}};
        auto apply = [](const double* h, double x, double y, double& ox, double& oy) {
            const double w = h[6] * x + h[7] * y + h[8];
            if (std::fabs(w) < 1e-12) throw Error{DSIFT_EGEOM, "homography: point maps to infinity"};
            ox = (h[0] * x + h[1] * y + h[2]) / w;
            oy = (h[3] * x + h[4] * y + h[5]) / w;
        };
        double sum = 0.0;
        for (const auto& cn : corners) {
            double ex, ey, gx, gy;
            apply(h_est, cn[0], cn[1], ex, ey);
            apply(h_gt, cn[0], cn[1], gx, gy);
            sum += std::hypot(ex - gx, ey - gy);
        }
        *out = sum / 4.0;
    });
}

// ---- image ingest (io.cpp:49-81) ---------------------------------------------
static void ingest(dsift_ctx* c, const uint8_t* pixels, long long n_px, int channels, int flags, DevBuf& bytes_buf,
                   float* dev_out) {
    if (channels != 1 && channels != 3) invalid("ingest: channels must be 1 (P5) or 3 (P6)");
    if (!pixels) invalid("extract: null image pointer");
    const size_t bytes = (size_t)n_px * channels;
    const unsigned char* dev_bytes = reinterpret_cast<const unsigned char*>(pixels);
    if (!(flags & DSIFT_INPUT_DEVICE)) {
        bytes_buf.ensure(bytes);
        cuda_check(cudaMemcpyAsync(bytes_buf.as<void>(), pixels, bytes, cudaMemcpyHostToDevice, c->stream), "H2D");
        dev_bytes = bytes_buf.as<unsigned char>();
    }
    cuda_check(launch_ingest_u8(dev_bytes, n_px, channels, dev_out, c->stream), "ingest");
    ++c->launches;
}

int dsift_extract_batch_u8(dsift_ctx* c, const uint8_t* pixels, int n, int w, int h, int channels, int flags) {
    return guard([&] {
        if (!c) invalid("null context");
        if (n <= 0) invalid("extract: batch must contain at least one image");
        if (w <= 0 || h <= 0) invalid("build_scale_space: empty image");
        set_device(c);
        dsift_result* r = c->cur;
        r->pending = r->ready = false;
        const long long n_px = (long long)n * w * h;
        ensure_events(r);
        cuda_check(cudaStreamWaitEvent(c->stream, r->input_free, 0), "wait");
        r->input.ensure(sizeof(float) * (size_t)n_px);
        ingest(c, pixels, n_px, channels, flags, r->input_u8, r->input.as<float>());
        extract_batch(c, r->input.as<float>(), n, w, h, DSIFT_INPUT_DEVICE);
    });
}

int dsift_ingest_u8(dsift_ctx* c, const uint8_t* pixels, int64_t n_px, int channels, int flags, float* dev_out) {
    return guard([&] {
        if (!c) invalid("null context");
        if (!dev_out) invalid("ingest: null output");
        set_device(c);
        ingest(c, pixels, n_px, channels, flags, c->scratch, dev_out);
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
    });
}

namespace {
// next_token / parse_dim (io.cpp:17-45): whitespace-separated tokens, '#'
// comments to end of line; std::stoi semantics (optional sign, leading
// digits, trailing junk ignored), value must be > 0.
std::string pnm_token(FILE* f) {
    std::string tok;
    int ch;
    while ((ch = std::fgetc(f)) != EOF) {
        if (ch == '#') {
            while ((ch = std::fgetc(f)) != EOF && ch != '\n') {
            }
            continue;
        }
        if (std::isspace(ch)) {
            if (!tok.empty()) return tok;
            continue;
        }
        tok.push_back((char)ch);
    }
    return tok;
}
int pnm_dim(const std::string& tok, const char* what) {
    const char* p = tok.c_str();
    bool ok = false;
    long long v = 0;
    int sign = 1;
    if (*p == '+' || *p == '-') sign = (*p++ == '-') ? -1 : 1;
    while (*p >= '0' && *p <= '9') {
        v = v * 10 + (*p++ - '0');
        ok = true;
        if (v > 2147483647LL) {
            ok = false;
            break;
        }
    }
    v *= sign;
    if (!ok || v <= 0) throw Error{DSIFT_EIO, std::string("image: bad ") + what};
    return (int)v;
}
}  // namespace

int dsift_load_image(const char* path, int32_t* w, int32_t* h, int32_t* channels, uint8_t* pixels, int64_t capacity) {
    return guard([&] {
        if (!path) invalid("load_image: null path");
        FILE* f = std::fopen(path, "rb");
        if (!f) throw Error{DSIFT_EIO, std::string("cannot open: ") + path};
        struct Closer {
            FILE* f;
            ~Closer() { std::fclose(f); }
        } closer{f};
        const std::string magic = pnm_token(f);
        if (magic != "P5" && magic != "P6")
            throw Error{DSIFT_EIO, "image: unsupported format '" + magic + "' (want P5/P6)"};
        const int ch = magic == "P6" ? 3 : 1;
        const int ww = pnm_dim(pnm_token(f), "width");
        const int hh = pnm_dim(pnm_token(f), "height");
        const int maxval = pnm_dim(pnm_token(f), "maxval");
        if (maxval != 255) throw Error{DSIFT_EIO, "image: maxval must be 255"};
        if (w) *w = ww;
        if (h) *h = hh;
        if (channels) *channels = ch;
        if (!pixels) return;
        const size_t payload = (size_t)ww * hh * ch;
        if ((int64_t)payload > capacity) invalid("load_image: pixel buffer too small");
        if (std::fread(pixels, 1, payload, f) != payload) throw Error{DSIFT_EIO, "image: truncated payload"};
    });
}

int dsift_result_sync(dsift_ctx* c, int64_t* total) {
    return guard([&] {
        if (!c) invalid("null context");
        result_sync(c);
        if (total) *total = c->cur->total;
    });
}

int dsift_result_range(dsift_ctx* c, int image, int64_t* begin, int64_t* count) {
    return guard([&] {
        if (!c) invalid("null context");
        result_sync(c);
        const dsift_result* r = c->cur;
        if (image < 0 || image >= r->batch) invalid("result: image index out of range");
        if (begin) *begin = r->h_offsets[image];
        if (count) *count = r->h_offsets[image + 1] - r->h_offsets[image];
    });
}

int dsift_result_copy(dsift_ctx* c, dsift_keypoint* kps, float* desc, uint8_t* desc_u8, int64_t* offsets) {
    return guard([&] {
        if (!c) invalid("null context");
        result_sync(c);
        const dsift_result* r = c->cur;
        const size_t n = (size_t)r->total;
        if (kps && n)
            cuda_check(cudaMemcpy(kps, r->pub_kps.as<void>(), n * sizeof(dsift_keypoint), cudaMemcpyDeviceToHost), "D2H");
        if (desc && n)
            cuda_check(cudaMemcpy(desc, r->desc.as<void>(), n * kDescDim * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
        if (desc_u8 && n)
            cuda_check(cudaMemcpy(desc_u8, r->desc_u8.as<void>(), n * kDescDim, cudaMemcpyDeviceToHost), "D2H");
        if (offsets) std::memcpy(offsets, r->h_offsets.data(), sizeof(int64_t) * (r->batch + 1));
    });
}

int dsift_result_device(dsift_ctx* c, const dsift_keypoint** kps, const float** desc, const uint8_t** desc_u8,
                        const int64_t** offsets) {
    return guard([&] {
        if (!c) invalid("null context");
        const dsift_result* r = c->cur;
        if (!r->pending && !r->ready) throw Error{DSIFT_ESTATE, "result: no extract issued"};
        if (kps) *kps = r->pub_kps.as<dsift_keypoint>();
        if (desc) *desc = r->desc.as<float>();
        if (desc_u8) *desc_u8 = r->desc_u8.as<uint8_t>();
        if (offsets) *offsets = reinterpret_cast<const int64_t*>(r->offsets.as<long long>());
    });
}

struct DlHolder {
    std::shared_ptr<void> keep;
    int64_t shape[2];
    DLManagedTensor t;
};

int dsift_export_dlpack(dsift_ctx* c, int which, void** out) {
    return guard([&] {
        if (!c || !out) invalid("null argument");
        result_sync(c);
        dsift_result* r = c->cur;
        auto* h = new DlHolder();
        DLTensor& t = h->t.dl_tensor;
        t.device = {kDLCUDA, c->device};
        t.ndim = 2;
        t.strides = nullptr;
        t.byte_offset = 0;
        h->shape[0] = r->total;
        if (which == DSIFT_EXPORT_KEYPOINTS) {
            h->keep = r->pub_kps.ptr;
            h->shape[1] = 7;
            t.dtype = {kDLFloat, 32, 1};
        } else if (which == DSIFT_EXPORT_DESC_F32) {
            h->keep = r->desc.ptr;
            h->shape[1] = kDescDim;
            t.dtype = {kDLFloat, 32, 1};
        } else if (which == DSIFT_EXPORT_DESC_U8) {
            h->keep = r->desc_u8.ptr;
            h->shape[1] = kDescDim;
            t.dtype = {kDLUInt, 8, 1};
        } else {
            delete h;
            invalid("export: unknown tensor");
        }
        t.data = h->keep.get();
        t.shape = h->shape;
        h->t.manager_ctx = h;
        h->t.deleter = [](DLManagedTensor* self) { delete static_cast<DlHolder*>(self->manager_ctx); };
        *out = &h->t;
    });
}

int dsift_result_sha256(dsift_ctx* c, int image, char hex65[65]) {
    return guard([&] {
        if (!c) invalid("null context");
        result_sync(c);
        const dsift_result* r = c->cur;
        if (image < 0 || image >= r->batch) invalid("result: image index out of range");
        const int64_t b = r->h_offsets[image], n = r->h_offsets[image + 1] - b;
        std::vector<uint8_t> buf(16 + (size_t)n * (28 + kDescDim * 4));
        const uint32_t hdr[3] = {1u, (uint32_t)n, (uint32_t)kDescDim};
        std::memcpy(buf.data(), "DSF1", 4);
        std::memcpy(buf.data() + 4, hdr, 12);
        if (n) {
            cuda_check(cudaMemcpy(buf.data() + 16, r->pub_kps.as<dsift_keypoint>() + b, (size_t)n * 28,
                                  cudaMemcpyDeviceToHost), "D2H");
            cuda_check(cudaMemcpy(buf.data() + 16 + (size_t)n * 28, r->desc.as<float>() + b * kDescDim,
                                  (size_t)n * kDescDim * 4, cudaMemcpyDeviceToHost), "D2H");
        }
        sha256(buf.data(), buf.size(), hex65);
    });
}

// ---- stage level -------------------------------------------------------------------
int dsift_build_scale_space(dsift_ctx* c, const float* image, int w, int h, int flags) {
    return guard([&] {
        if (!c) invalid("null context");
        if (!image) invalid("build_scale_space: null image");
        set_device(c);
        c->plan = make_plan(c->cfg, w, h);
        c->batch = 1;
        build_pyramid_desc(c);
        ensure_counters(c);
        const float* dev_in = stage_input(c, image, 1, w, h, flags);
        launch_pyramid(c, dev_in);
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
    });
}

int dsift_load_scale_space(dsift_ctx* c, int n_oct, int upsampled, const int32_t* dims, const float* const* gauss,
                           const float* const* dog) {
    return guard([&] {
        if (!c) invalid("null context");
        if (n_oct <= 0 || n_oct > kMaxOctaves) invalid("load_scale_space: bad octave count");
        set_device(c);
        Plan p;
        p.s = c->cfg.c.intervals;
        p.up = upsampled != 0;
        p.n_oct = n_oct;
        p.handcrafted = true;
        for (int o = 0; o < n_oct; ++o) {
            p.ow.push_back(dims[2 * o]);
            p.oh.push_back(dims[2 * o + 1]);
            p.pitch.push_back(round_pitch(dims[2 * o]));
        }
        p.in_w = dims[0];
        p.in_h = dims[1];
        for (int i = 0; i < p.s + 3; ++i) p.level_sigma[i] = c->cfg.c.sigma0 * std::pow(2.0, double(i) / p.s);
        c->plan = p;
        c->batch = 1;
        build_pyramid_desc(c);
        ensure_counters(c);
        const int s = p.s;
        for (int o = 0; o < n_oct; ++o) {
            const OctaveDesc& od = c->pyr.oct[o];
            for (int i = 0; i < s + 3; ++i)
                cuda_check(cudaMemcpy2D(od.gauss + i * od.level_stride, sizeof(float) * od.pitch, gauss[o * (s + 3) + i],
                                        sizeof(float) * od.w, sizeof(float) * od.w, od.h, cudaMemcpyHostToDevice), "H2D");
            for (int i = 0; i < s + 2; ++i)
                cuda_check(cudaMemcpy2D(od.dog + i * od.level_stride, sizeof(float) * od.pitch, dog[o * (s + 2) + i],
                                        sizeof(float) * od.w, sizeof(float) * od.w, od.h, cudaMemcpyHostToDevice), "H2D");
        }
    });
}

int dsift_scale_space_info(dsift_ctx* c, int32_t* n_oct, int32_t* upsampled, int32_t* dims) {
    return guard([&] {
        if (!c || c->plan.n_oct == 0) throw Error{DSIFT_ESTATE, "scale space: none built"};
        if (n_oct) *n_oct = c->plan.n_oct;
        if (upsampled) *upsampled = c->plan.up ? 1 : 0;
        if (dims)
            for (int o = 0; o < c->plan.n_oct; ++o) {
                dims[2 * o] = c->plan.ow[o];
                dims[2 * o + 1] = c->plan.oh[o];
            }
    });
}

int dsift_scale_space_level(dsift_ctx* c, int octave, int kind, int level, float* out) {
    return guard([&] {
        if (!c || c->plan.n_oct == 0) throw Error{DSIFT_ESTATE, "scale space: none built"};
        if (octave < 0 || octave >= c->plan.n_oct) invalid("scale space: octave out of range");
        const int nl = kind == 0 ? c->plan.s + 3 : c->plan.s + 2;
        if (level < 0 || level >= nl) invalid("scale space: level out of range");
        set_device(c);
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        const OctaveDesc& od = c->pyr.oct[octave];
        const float* src = (kind == 0 ? od.gauss : od.dog) + (long long)level * od.level_stride;
        cuda_check(cudaMemcpy2D(out, sizeof(float) * od.w, src, sizeof(float) * od.pitch, sizeof(float) * od.w, od.h,
                                cudaMemcpyDeviceToHost), "D2H");
    });
}

static void require_space(dsift_ctx* c) {
    if (c->plan.n_oct == 0) throw Error{DSIFT_ESTATE, "scale space: none built"};
    if (c->batch != 1) throw Error{DSIFT_ESTATE, "stage API needs a single-image scale space"};
}

int dsift_find_extrema(dsift_ctx* c, int32_t* out5, int64_t cap, int64_t* n) {
    return guard([&] {
        if (!c) invalid("null context");
        require_space(c);
        set_device(c);
        long long dcap = 0;
        for (int o = 0; o < c->plan.n_oct; ++o) dcap += (long long)c->plan.ow[o] * c->plan.oh[o] * c->plan.s / 2 + 16;
        reset_counters(c);
        run_detect(c, 1, dcap);
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        Counters h{};
        cuda_check(cudaMemcpy(&h, c->counters.as<void>(), sizeof(h), cudaMemcpyDeviceToHost), "D2H");
        std::vector<DevCandidate> v((size_t)h.n_det);
        if (!v.empty())
            cuda_check(cudaMemcpy(v.data(), c->det_cand.as<void>(), v.size() * sizeof(DevCandidate),
                                  cudaMemcpyDeviceToHost), "D2H");
        std::sort(v.begin(), v.end(), [](const DevCandidate& a, const DevCandidate& b) {
            if (a.octave != b.octave) return a.octave < b.octave;
            if (a.interval != b.interval) return a.interval < b.interval;
            if (a.row != b.row) return a.row < b.row;
            return a.col < b.col;
        });
        *n = (int64_t)v.size();
        for (size_t k = 0; k < v.size() && (int64_t)k < cap; ++k) {
            out5[5 * k + 0] = v[k].octave;
            out5[5 * k + 1] = v[k].interval;
            out5[5 * k + 2] = v[k].row;
            out5[5 * k + 3] = v[k].col;
            out5[5 * k + 4] = v[k].is_max;
        }
    });
}

int dsift_detect(dsift_ctx* c, dsift_keypoint* out, int64_t cap, int64_t* n) {
    return guard([&] {
        if (!c) invalid("null context");
        require_space(c);
        set_device(c);
        long long dcap = 0;
        for (int o = 0; o < c->plan.n_oct; ++o) dcap += (long long)c->plan.ow[o] * c->plan.oh[o] * c->plan.s / 2 + 16;
        reset_counters(c);
        c->keep.ensure(sizeof(int) * (size_t)dcap);
        run_detect(c, 1, dcap);   // the hot path's kernels: extrema, then refine
        run_refine(c, dcap, c->keep.as<int>());
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        Counters h{};
        cuda_check(cudaMemcpy(&h, c->counters.as<void>(), sizeof(h), cudaMemcpyDeviceToHost), "D2H");
        const size_t mc = (size_t)h.n_det, m = (size_t)h.n_kp;
        std::vector<DevKeypoint> kp(m);
        std::vector<DevCandidate> cd(mc);
        std::vector<int> keep(mc);
        if (m) cuda_check(cudaMemcpy(kp.data(), c->det_kps.as<void>(), m * sizeof(DevKeypoint), cudaMemcpyDeviceToHost), "D2H");
        if (mc) {
            cuda_check(cudaMemcpy(cd.data(), c->det_cand.as<void>(), mc * sizeof(DevCandidate), cudaMemcpyDeviceToHost), "D2H");
            cuda_check(cudaMemcpy(keep.data(), c->keep.as<void>(), mc * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
        }
        // survivors are compacted in candidate-array order; pair each with its
        // candidate, then restore the reference's (octave, interval, row, col) order
        std::vector<std::pair<size_t, size_t>> surv;   // (candidate, keypoint)
        for (size_t i = 0, j = 0; i < mc; ++i)
            if (keep[i]) surv.push_back({i, j++});
        std::stable_sort(surv.begin(), surv.end(), [&](const auto& p, const auto& q) {
            const DevCandidate &a = cd[p.first], &b = cd[q.first];
            if (a.octave != b.octave) return a.octave < b.octave;
            if (a.interval != b.interval) return a.interval < b.interval;
            if (a.row != b.row) return a.row < b.row;
            return a.col < b.col;
        });
        std::vector<size_t> order;
        for (const auto& p : surv) order.push_back(p.second);
        *n = (int64_t)order.size();
        for (size_t k = 0; k < order.size() && (int64_t)k < cap; ++k) {
            const DevKeypoint& s = kp[order[k]];
            out[k] = dsift_keypoint{s.x, s.y, s.sigma, s.angle, s.response, s.octave, s.interval};
        }
    });
}

// Stage-level calls: the device error word as the reference's exceptions
// (NaN pixel -> std::out_of_range, detsum.cpp:138-141) or a loud overflow.
static Counters check_stage_errors(dsift_ctx* c) {
    Counters h{};
    cuda_check(cudaMemcpy(&h, c->counters.as<void>(), sizeof(h), cudaMemcpyDeviceToHost), "D2H");
    if (h.err & kErrHistogramRange) throw Error{DSIFT_ERANGE, "histogram: bin index out of range"};
    if (h.err & kErrOrientedCapacity) throw Error{DSIFT_ECAPACITY, "device work list overflow: oriented keypoints"};
    if (h.err & kErrDescriptorLattice) throw Error{DSIFT_ECAPACITY, "descriptor lattice exceeds table capacity"};
    return h;
}

static DevKeypoint* upload_kps(dsift_ctx* c, const dsift_keypoint* kps, int64_t n) {
    std::vector<DevKeypoint> v((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        if (kps[i].octave < 0 || kps[i].octave >= c->plan.n_oct) invalid("keypoint octave out of range");
        v[i] = DevKeypoint{kps[i].x, kps[i].y, kps[i].sigma, kps[i].angle, kps[i].response, kps[i].octave,
                           kps[i].interval, 0};
    }
    c->stage_kps.ensure(sizeof(DevKeypoint) * (size_t)std::max<int64_t>(n, 1));
    if (n) cuda_check(cudaMemcpy(c->stage_kps.as<void>(), v.data(), v.size() * sizeof(DevKeypoint),
                                 cudaMemcpyHostToDevice), "H2D");
    return c->stage_kps.as<DevKeypoint>();
}

static double stage_smax(dsift_ctx* c, const dsift_keypoint* kps, int64_t n) {
    double smax = c->cfg.c.sigma0 * std::pow(2.0, (c->cfg.c.intervals + 0.5) / c->cfg.c.intervals) * 1.001;
    for (int64_t i = 0; i < n; ++i) {
        const double to_input = std::ldexp(1.0, kps[i].octave) * (c->plan.up ? 0.5 : 1.0);
        smax = std::max(smax, kps[i].sigma / to_input * 1.001);
    }
    return smax;
}

int dsift_orientation_histograms(dsift_ctx* c, const dsift_keypoint* kps, int64_t n, float* out) {
    return guard([&] {
        if (!c) invalid("null context");
        require_space(c);
        set_device(c);
        if (n <= 0) return;
        DevKeypoint* dk = upload_kps(c, kps, n);
        std::vector<dsift_keypoint> hk(kps, kps + n);
        const int bins = c->cfg.c.orientation_bins;
        c->stage_out.ensure(sizeof(float) * (size_t)n * bins + sizeof(DevKeypoint) * (size_t)n * bins);
        float* hist = c->stage_out.as<float>();
        DevKeypoint* tmp = reinterpret_cast<DevKeypoint*>(hist + (size_t)n * bins);
        reset_counters(c);
        run_orient(c, dk, n, n, tmp, n * bins, hist, orient_depth(c->cfg.c, &hk, c->plan));
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        check_stage_errors(c);
        cuda_check(cudaMemcpy(out, hist, sizeof(float) * (size_t)n * bins, cudaMemcpyDeviceToHost), "D2H");
    });
}

int dsift_assign_orientations(dsift_ctx* c, const dsift_keypoint* kps, int64_t n, dsift_keypoint* out, int64_t cap,
                              int64_t* n_out) {
    return guard([&] {
        if (!c) invalid("null context");
        require_space(c);
        set_device(c);
        *n_out = 0;
        if (n <= 0) return;
        DevKeypoint* dk = upload_kps(c, kps, n);
        std::vector<dsift_keypoint> hk(kps, kps + n);
        const int bins = c->cfg.c.orientation_bins;
        c->stage_out.ensure(sizeof(DevKeypoint) * (size_t)n * bins);
        DevKeypoint* tmp = c->stage_out.as<DevKeypoint>();
        reset_counters(c);
        run_orient(c, dk, n, n, tmp, n * bins, nullptr, orient_depth(c->cfg.c, &hk, c->plan));
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        const Counters h = check_stage_errors(c);
        std::vector<DevKeypoint> v((size_t)h.n_ori);
        if (!v.empty())
            cuda_check(cudaMemcpy(v.data(), tmp, v.size() * sizeof(DevKeypoint), cudaMemcpyDeviceToHost), "D2H");
        *n_out = (int64_t)v.size();
        for (size_t k = 0; k < v.size() && (int64_t)k < cap; ++k)
            out[k] = dsift_keypoint{v[k].x, v[k].y, v[k].sigma, v[k].angle, v[k].response, v[k].octave, v[k].interval};
    });
}

static void stage_describe(dsift_ctx* c, const dsift_keypoint* kps, int64_t n, float* out, uint8_t* out_u8,
                           int raw_mode, double f) {
    if (!c) invalid("null context");
    require_space(c);
    set_device(c);
    if (raw_mode && !(f > 0.0)) invalid("raw_descriptor: scale_factor must be > 0");
    if (n <= 0) return;
    DevKeypoint* dk = upload_kps(c, kps, n);
    c->stage_out.ensure(sizeof(float) * kDescDim * (size_t)n + (size_t)kDescDim * n);
    float* d = c->stage_out.as<float>();
    unsigned char* d8 = reinterpret_cast<unsigned char*>(d + (size_t)kDescDim * n);
    reset_counters(c);
    run_describe(c, dk, n, d, raw_mode ? nullptr : d8, raw_mode, f, stage_smax(c, kps, n), nullptr);
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    check_stage_errors(c);
    cuda_check(cudaMemcpy(out, d, sizeof(float) * kDescDim * (size_t)n, cudaMemcpyDeviceToHost), "D2H");
    if (out_u8 && !raw_mode)
        cuda_check(cudaMemcpy(out_u8, d8, (size_t)kDescDim * n, cudaMemcpyDeviceToHost), "D2H");
}

int dsift_raw_descriptors(dsift_ctx* c, const dsift_keypoint* kps, int64_t n, double f, float* out) {
    return guard([&] { stage_describe(c, kps, n, out, nullptr, 1, f); });
}

int dsift_dsp_descriptors(dsift_ctx* c, const dsift_keypoint* kps, int64_t n, float* out, uint8_t* out_u8) {
    return guard([&] { stage_describe(c, kps, n, out, out_u8, 0, 0.0); });
}

int dsift_synth_value_noise(dsift_ctx* c, float* dev_out, int n, int w, int h, uint64_t seed0, int octaves,
                            int cells) {
    return guard([&] {
        if (!c || !dev_out) invalid("null argument");
        if (n <= 0 || w <= 0 || h <= 0) invalid("synth: bad size");
        set_device(c);
        const int nparts = 64;
        c->scratch.ensure(sizeof(double) * 2 * (size_t)n * nparts);
        cuda_check(launch_value_noise(dev_out, n, w, h, seed0, octaves, cells, c->scratch.as<double>(), nparts,
                                      c->stream), "synth");
        c->launches += 2;
    });
}

int64_t dsift_kernel_launches(dsift_ctx* c) { return c ? c->launches : 0; }

int dsift_set_option(dsift_ctx* c, int key, int64_t value) {
    return guard([&] {
        if (!c) invalid("null context");
        if (key == DSIFT_OPT_FORCE_EXACT) {
            if (value != 0 && value != 1) invalid("set_option: FORCE_EXACT must be 0 or 1");
            c->force_exact = (int)value;
        } else if (key == DSIFT_OPT_CAPACITY_SCALE) {
            if (value <= 0) invalid("set_option: CAPACITY_SCALE must be > 0 (1/1000 units)");
            c->cap_scale = (double)value / 1000.0;
        } else if (key == DSIFT_OPT_TEXTURE_GATHERS) {
            if (value != 0 && value != 1) invalid("set_option: TEXTURE_GATHERS must be 0 or 1");
            c->tex_gathers = value != 0;
        } else {
            invalid("set_option: unknown key");
        }
    });
}

int64_t dsift_stat(dsift_ctx* c, int key) {
    if (!c) return -1;
    if (key == DSIFT_STAT_EXACT_FALLBACKS) return (int64_t)c->cur->slow;
    if (key == DSIFT_STAT_REPLAYS) return (int64_t)c->cur->retries;
    if (key == DSIFT_STAT_LATTICE_POINTS) return (int64_t)c->cur->lattice;
    if (key == DSIFT_STAT_LATTICE_IN_RANGE) return (int64_t)c->cur->lattice_in;
    return -1;
}

int dsift_set_profiling(dsift_ctx* c, int on) {
    return guard([&] {
        if (!c) invalid("null context");
        set_device(c);
        if (on && !c->stage_ev[0])
            for (auto& e : c->stage_ev) cuda_check(cudaEventCreate(&e), "event");
        c->profiling = on != 0;
    });
}

int dsift_stage_times(dsift_ctx* c, float* ms5) {
    return guard([&] {
        if (!c || !c->profiling) throw Error{DSIFT_ESTATE, "profiling not enabled"};
        set_device(c);
        cuda_check(cudaEventSynchronize(c->stage_ev[5]), "sync");
        for (int i = 0; i < 5; ++i)
            cuda_check(cudaEventElapsedTime(&ms5[i], c->stage_ev[i], c->stage_ev[i + 1]), "elapsed");
    });
}

}  // extern "C"
