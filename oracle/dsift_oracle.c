/* oracle/dsift_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU parity checker.
 *
 * A plain-C restatement of the reference extraction path
 *   detsift::extract  (/root/reference/proj/src/io.cpp:111-142)
 * written stage by stage from the reference's behaviour.  Every floating-point
 * expression keeps the reference's operand order, precision (float vs double)
 * and rounding points, and the file is compiled with -ffp-contract=off so no
 * FMA contraction can occur (the reference is an x86-64 baseline SSE2 build,
 * proj/CMakeLists.txt:2-12).  Transcendentals (exp, atan2f, cos, sin, pow) come
 * from the same host libm the reference links.
 *
 * Parity pinning: tests/test_oracle.py checks every entry point bit-for-bit
 * against the unmodified reference (oracle/_ref/libdetsift_ref.so) and the
 * committed golden vectors under tests/golden/.
 *
 * The product (paper_2605_17869_b200/) never links or calls this file.
 */
#include "dsift_oracle.h"

#include <ctype.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define TWO_PI 6.283185307179586476925286766559 /* orient.cpp:37, describe.cpp:187 */
#define DESC_CELLS 4                            /* describe.hpp:11 */
#define DESC_ORIENTS 8                          /* describe.hpp:12 */
#define DESC_DIM 128                            /* describe.hpp:13 */
#define UNDEFINED_SAMPLE (-1.0f)                /* describe.cpp:188 */

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* dor_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------- */
/* Fixed-tree reduction (detsum.cpp:13-71).                                  */
/* The reference folds leaf pairs (2j, 2j+1) level by level, promoting an odd */
/* tail, in 1024-leaf blocks that compose into the same tree.  That tree is  */
/* exactly the one a streaming binary counter builds: node j holds the sum of */
/* an aligned 2^j-leaf block; the pending nodes are folded smallest-first.   */
/* ------------------------------------------------------------------------- */
typedef struct {
    double node[64];
    uint64_t count;
} tree_acc;

static void tree_init(tree_acc* t) { t->count = 0; }

static void tree_push(tree_acc* t, double leaf) {
    uint64_t c = t->count;
    int level = 0;
    while (c & 1u) {
        leaf = t->node[level] + leaf;
        c >>= 1;
        ++level;
    }
    t->node[level] = leaf;
    t->count++;
}

static double tree_result(const tree_acc* t) {
    if (t->count == 0) return 0.0;
    int level = 0;
    while (!((t->count >> level) & 1u)) ++level;
    double r = t->node[level];
    for (int k = level + 1; k < 64; ++k)
        if ((t->count >> k) & 1u) r = t->node[k] + r;
    return r;
}

double dor_tree_sum_f64(const double* v, int64_t n) {
    tree_acc t;
    tree_init(&t);
    for (int64_t i = 0; i < n; ++i) tree_push(&t, v[i]);
    return tree_result(&t);
}

float dor_tree_sum(const float* v, int64_t n) { /* detsum.cpp:115-117 */
    tree_acc t;
    tree_init(&t);
    for (int64_t i = 0; i < n; ++i) tree_push(&t, (double)v[i]);
    return (float)tree_result(&t);
}

/* tree_accumulate_histogram (detsum.cpp:135-177): per-bin tree over that   */
/* bin's weights in canonical (arrival) order.                              */
typedef struct {
    tree_acc* acc;
    int bins;
} hist_acc;

static int hist_init(hist_acc* h, int bins) {
    h->bins = bins;
    h->acc = (tree_acc*)malloc(sizeof(tree_acc) * (size_t)bins);
    if (!h->acc) return -1;
    for (int b = 0; b < bins; ++b) tree_init(&h->acc[b]);
    return 0;
}
static void hist_add(hist_acc* h, int bin, float w) { tree_push(&h->acc[bin], (double)w); }
static void hist_finish(hist_acc* h, float* out) {
    for (int b = 0; b < h->bins; ++b) out[b] = (float)tree_result(&h->acc[b]);
    free(h->acc);
}

int dor_tree_hist(const int32_t* bins, const float* w, int64_t n, int bin_count, float* out) {
    if (bin_count <= 0) return fail(-1, "histogram: bin_count must be > 0");
    for (int64_t i = 0; i < n; ++i)
        if (bins[i] < 0 || bins[i] >= bin_count)
            return fail(-2, "histogram: bin index out of range");
    hist_acc h;
    if (hist_init(&h, bin_count)) return fail(-2, "out of memory");
    for (int64_t i = 0; i < n; ++i) hist_add(&h, bins[i], w[i]);
    hist_finish(&h, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Config (core.hpp:30-47, core.cpp:17-46)                                   */
/* ------------------------------------------------------------------------- */
void dor_config_default(dor_config* c, double* scales5) {
    c->sigma0 = 1.6f;
    c->intervals = 3;
    c->assumed_blur = 0.5f;
    c->contrast_threshold = 0.04f;
    c->edge_ratio = 10.0f;
    c->max_refine_iters = 5;
    c->upsample_pixel_limit = 4000000;
    scales5[0] = 0.5;
    scales5[1] = 1.0 / 1.4142135623730951;
    scales5[2] = 1.0;
    scales5[3] = 1.4142135623730951;
    scales5[4] = 2.0;
    c->dsp_scales = scales5;
    c->n_dsp_scales = 5;
    c->descriptor_clip = 0.2f;
    c->orientation_bins = 36;
    c->orientation_peak_ratio = 0.8f;
    c->num_octaves = 0;
}

int dor_config_validate(const dor_config* c) {
    if (!(c->sigma0 > 0.0f) || !(c->assumed_blur >= 0.0f) || !(c->sigma0 > c->assumed_blur))
        return fail(-1, "config: require sigma0 > assumed_input_blur >= 0");
    if (c->intervals < 1) return fail(-1, "config: intervals_per_octave must be >= 1");
    if (!(c->contrast_threshold > 0.0f)) return fail(-1, "config: contrast_threshold must be > 0");
    if (!(c->edge_ratio > 1.0f)) return fail(-1, "config: edge_ratio must be > 1");
    if (c->max_refine_iters < 1) return fail(-1, "config: max_refine_iters must be >= 1");
    if (c->upsample_pixel_limit < 0)
        return fail(-1, "config: upsample_pixel_limit must be >= 0");
    if (c->n_dsp_scales <= 0 || !c->dsp_scales)
        return fail(-1, "config: dsp_scales must be nonempty");
    for (int i = 0; i < c->n_dsp_scales; ++i) {
        if (!(c->dsp_scales[i] > 0.0)) return fail(-1, "config: dsp_scales must all be > 0");
        if (i > 0 && !(c->dsp_scales[i] > c->dsp_scales[i - 1]))
            return fail(-1, "config: dsp_scales must be strictly increasing");
    }
    if (!(c->descriptor_clip > 0.0f)) return fail(-1, "config: descriptor_clip must be > 0");
    if (c->orientation_bins < 2) return fail(-1, "config: orientation_bins must be >= 2");
    if (!(c->orientation_peak_ratio > 0.0f) || c->orientation_peak_ratio > 1.0f)
        return fail(-1, "config: orientation_peak_ratio must be in (0,1]");
    if (c->num_octaves < 0) return fail(-1, "config: num_octaves must be >= 0 (0 = auto)");
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Scale space (scalespace.cpp)                                              */
/* ------------------------------------------------------------------------- */
int dor_gaussian_kernel(double sigma, float* out, int cap) { /* scalespace.cpp:23-36 */
    if (!(sigma > 0.0)) return fail(-1, "gaussian_kernel: sigma must be > 0");
    const int radius = (int)ceil(4.0 * sigma);
    const int len = 2 * radius + 1;
    if (len > cap) return len;
    double* raw = (double*)malloc(sizeof(double) * (size_t)len);
    double sum = 0.0;
    for (int k = -radius; k <= radius; ++k) {
        raw[k + radius] = exp(-(double)k * k / (2.0 * sigma * sigma));
        sum += raw[k + radius];
    }
    for (int i = 0; i < len; ++i) out[i] = (float)(raw[i] / sum);
    free(raw);
    return len;
}

static int reflect101(int p, int n) { /* scalespace.cpp:41-48 */
    if (n == 1) return 0;
    for (;;) {
        if (p < 0) p = -p;
        else if (p >= n) p = 2 * n - 2 - p;
        else return p;
    }
}

int dor_convolve(const float* img, int w, int h, const float* k, int len, float* out) {
    /* scalespace.cpp:52-111: H pass into a float temporary, then V pass; each */
    /* output is a left-to-right double accumulation rounded once to float.   */
    if (len == 0 || len % 2 == 0)
        return fail(-1, "convolve_separable: kernel must have odd length");
    if (len > 2 * (w > h ? w : h) + 1)
        return fail(-1, "convolve_separable: kernel longer than image allows");
    const int r = len / 2;
    float* tmp = (float*)malloc(sizeof(float) * (size_t)w * (size_t)h);
    for (int y = 0; y < h; ++y) {
        const float* src = img + (size_t)y * w;
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int t = 0; t < len; ++t) acc += (double)k[t] * src[reflect101(x + t - r, w)];
            tmp[(size_t)y * w + x] = (float)acc;
        }
    }
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            double acc = 0.0;
            for (int t = 0; t < len; ++t)
                acc += (double)k[t] * tmp[(size_t)reflect101(y + t - r, h) * w + x];
            out[(size_t)y * w + x] = (float)acc;
        }
    }
    free(tmp);
    return 0;
}

void dor_upsample2x(const float* img, int w, int h, float* out) { /* scalespace.cpp:113-131 */
    for (int y = 0; y < 2 * h; ++y) {
        const int y0 = y / 2;
        const int y1 = (y & 1) ? (y0 + 1 < h - 1 ? y0 + 1 : h - 1) : y0;
        const float* r0 = img + (size_t)y0 * w;
        const float* r1 = img + (size_t)y1 * w;
        for (int x = 0; x < 2 * w; ++x) {
            const int x0 = x / 2;
            const int x1 = (x & 1) ? (x0 + 1 < w - 1 ? x0 + 1 : w - 1) : x0;
            const double v = 0.25 * ((double)r0[x0] + r0[x1] + r1[x0] + r1[x1]);
            out[(size_t)y * 2 * w + x] = (float)v;
        }
    }
}

void dor_decimate2x(const float* img, int w, int h, float* out) { /* scalespace.cpp:133-142 */
    const int ow = w / 2, oh = h / 2;
    for (int y = 0; y < oh; ++y)
        for (int x = 0; x < ow; ++x) out[(size_t)y * ow + x] = img[(size_t)(2 * y) * w + 2 * x];
}

static double level_sigma(const dor_scale_space* ss, int i) { /* scalespace.cpp:11-13 */
    return ss->sigma0 * pow(2.0, (double)i / ss->s);
}

static double octave_to_input(const dor_scale_space* ss, int o) { /* scalespace.cpp:15-17 */
    return ldexp(1.0, o) * (ss->upsampled ? 0.5 : 1.0);
}

void dor_ss_free(dor_scale_space* ss) {
    if (!ss) return;
    for (int o = 0; o < ss->n_oct; ++o) {
        for (int i = 0; i < ss->s + 3; ++i) free(ss->gauss[o * (ss->s + 3) + i]);
        for (int i = 0; i < ss->s + 2; ++i) free(ss->dog[o * (ss->s + 2) + i]);
    }
    free(ss->w);
    free(ss->h);
    free(ss->gauss);
    free(ss->dog);
    free(ss);
}

static dor_scale_space* ss_alloc(int n_oct, int s) {
    dor_scale_space* ss = (dor_scale_space*)calloc(1, sizeof(dor_scale_space));
    ss->n_oct = n_oct;
    ss->s = s;
    ss->w = (int32_t*)calloc((size_t)n_oct, sizeof(int32_t));
    ss->h = (int32_t*)calloc((size_t)n_oct, sizeof(int32_t));
    ss->gauss = (float**)calloc((size_t)n_oct * (size_t)(s + 3), sizeof(float*));
    ss->dog = (float**)calloc((size_t)n_oct * (size_t)(s + 2), sizeof(float*));
    return ss;
}

int dor_build_scale_space(const float* img, int w, int h, const dor_config* c,
                          dor_scale_space** out) {
    /* scalespace.cpp:144-214 */
    int rc = dor_config_validate(c);
    if (rc) return rc;
    if (w <= 0 || h <= 0) return fail(-1, "build_scale_space: empty image");
    const int up = (int64_t)w * h <= c->upsample_pixel_limit;
    const int bw = up ? 2 * w : w, bh = up ? 2 * h : h;
    const double assumed = up ? 2.0 * c->assumed_blur : c->assumed_blur;
    if (!((double)c->sigma0 > assumed))
        return fail(-1, "build_scale_space: effective input blur exceeds sigma0");
    if ((bw < bh ? bw : bh) < 8)
        return fail(-1, "build_scale_space: image smaller than 8x8 after upsampling policy");

    const int s = c->intervals;
    const int min_dim = bw < bh ? bw : bh;
    int auto_oct = -2;
    for (int d = min_dim; d > 1; d /= 2) ++auto_oct;
    if (auto_oct < 1) auto_oct = 1;

    const double bridge = sqrt((double)c->sigma0 * c->sigma0 - assumed * assumed);
    double* inc = (double*)malloc(sizeof(double) * (size_t)(s + 2));
    for (int i = 1; i < s + 3; ++i)
        inc[i - 1] = c->sigma0 * pow(2.0, (double)(i - 1) / s) * sqrt(pow(2.0, 2.0 / s) - 1.0);
    int max_radius = (int)ceil(4.0 * bridge);
    for (int i = 0; i < s + 2; ++i) {
        const int r = (int)ceil(4.0 * inc[i]);
        if (r > max_radius) max_radius = r;
    }
    if ((bw > bh ? bw : bh) < max_radius) {
        free(inc);
        return fail(-1, "build_scale_space: image too small for the blur ladder");
    }
    int feasible = 1;
    for (int ww = bw / 2, hh = bh / 2;
         (ww < hh ? ww : hh) >= 8 && (ww > hh ? ww : hh) >= max_radius; ww /= 2, hh /= 2)
        ++feasible;
    int n_oct = c->num_octaves > 0 ? (c->num_octaves < auto_oct ? c->num_octaves : auto_oct)
                                   : auto_oct;
    if (feasible < n_oct) n_oct = feasible;

    dor_scale_space* ss = ss_alloc(n_oct, s);
    ss->sigma0 = c->sigma0;
    ss->upsampled = up;

    float* base = (float*)img;
    if (up) {
        base = (float*)malloc(sizeof(float) * (size_t)bw * bh);
        dor_upsample2x(img, w, h, base);
    }
    float kern[512];
    int ow = bw, oh = bh;
    for (int o = 0; o < n_oct; ++o) {
        ss->w[o] = ow;
        ss->h[o] = oh;
        float** g = ss->gauss + o * (s + 3);
        for (int i = 0; i < s + 3; ++i) g[i] = (float*)malloc(sizeof(float) * (size_t)ow * oh);
        if (o == 0) {
            const int len = dor_gaussian_kernel(bridge, kern, 512);
            dor_convolve(base, ow, oh, kern, len, g[0]);
        } else {
            const float* prev = ss->gauss[(o - 1) * (s + 3) + s];
            dor_decimate2x(prev, ss->w[o - 1], ss->h[o - 1], g[0]);
        }
        for (int i = 1; i < s + 3; ++i) {
            const int len = dor_gaussian_kernel(inc[i - 1], kern, 512);
            dor_convolve(g[i - 1], ow, oh, kern, len, g[i]);
        }
        float** d = ss->dog + o * (s + 2);
        for (int i = 0; i < s + 2; ++i) {
            d[i] = (float*)malloc(sizeof(float) * (size_t)ow * oh);
            for (size_t p = 0; p < (size_t)ow * oh; ++p) d[i][p] = g[i + 1][p] - g[i][p];
        }
        ow /= 2;
        oh /= 2;
    }
    if (up) free(base);
    free(inc);
    *out = ss;
    return 0;
}

void dor_ss_info(const dor_scale_space* ss, int32_t* n_oct, int32_t* upsampled, int32_t* dims) {
    *n_oct = ss->n_oct;
    *upsampled = ss->upsampled;
    if (dims)
        for (int o = 0; o < ss->n_oct; ++o) {
            dims[2 * o] = ss->w[o];
            dims[2 * o + 1] = ss->h[o];
        }
}

void dor_ss_level(const dor_scale_space* ss, int o, int kind, int i, float* out) {
    const float* src = kind == 0 ? ss->gauss[o * (ss->s + 3) + i] : ss->dog[o * (ss->s + 2) + i];
    memcpy(out, src, sizeof(float) * (size_t)ss->w[o] * ss->h[o]);
}

dor_scale_space* dor_ss_from_levels(int n_oct, int s, float sigma0, int upsampled,
                                    const int32_t* dims, const float* const* gauss,
                                    const float* const* dog) {
    dor_scale_space* ss = ss_alloc(n_oct, s);
    ss->sigma0 = sigma0;
    ss->upsampled = upsampled;
    for (int o = 0; o < n_oct; ++o) {
        ss->w[o] = dims[2 * o];
        ss->h[o] = dims[2 * o + 1];
        const size_t px = (size_t)ss->w[o] * ss->h[o];
        for (int i = 0; i < s + 3; ++i) {
            ss->gauss[o * (s + 3) + i] = (float*)malloc(sizeof(float) * px);
            memcpy(ss->gauss[o * (s + 3) + i], gauss[o * (s + 3) + i], sizeof(float) * px);
        }
        for (int i = 0; i < s + 2; ++i) {
            ss->dog[o * (s + 2) + i] = (float*)malloc(sizeof(float) * px);
            memcpy(ss->dog[o * (s + 2) + i], dog[o * (s + 2) + i], sizeof(float) * px);
        }
    }
    return ss;
}

/* ------------------------------------------------------------------------- */
/* Detection (detect.cpp)                                                    */
/* ------------------------------------------------------------------------- */
#define AT(img, w, x, y) ((img)[(size_t)(y) * (w) + (x)])

static int strictly_extremal(const float* lo, const float* mid, const float* hi, int w, int x,
                             int y, float v, int is_max) { /* detect.cpp:11-28 */
    for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            const float a = AT(lo, w, x + dx, y + dy), b = AT(hi, w, x + dx, y + dy);
            if (is_max ? (a >= v || b >= v) : (a <= v || b <= v)) return 0;
            if (dx == 0 && dy == 0) continue;
            const float m = AT(mid, w, x + dx, y + dy);
            if (is_max ? m >= v : m <= v) return 0;
        }
    return 1;
}

int64_t dor_find_extrema(const dor_scale_space* ss, const dor_config* c, int32_t* out5,
                         int64_t cap) { /* detect.cpp:32-71, canonical (o, i, row, col) */
    const int s = ss->s;
    const float gate = 0.5f * c->contrast_threshold / s;
    int64_t n = 0;
    for (int o = 0; o < ss->n_oct; ++o) {
        const int w = ss->w[o], h = ss->h[o];
        if (w < 3 || h < 3) continue;
        for (int i = 1; i <= s; ++i) {
            const float* lo = ss->dog[o * (s + 2) + i - 1];
            const float* mid = ss->dog[o * (s + 2) + i];
            const float* hi = ss->dog[o * (s + 2) + i + 1];
            for (int y = 1; y < h - 1; ++y)
                for (int x = 1; x < w - 1; ++x) {
                    const float v = AT(mid, w, x, y);
                    if (!(fabsf(v) > gate)) continue;
                    const int is_max = v > 0.0f;
                    if (!strictly_extremal(lo, mid, hi, w, x, y, v, is_max)) continue;
                    if (n < cap) {
                        int32_t* e = out5 + 5 * n;
                        e[0] = o;
                        e[1] = i;
                        e[2] = y;
                        e[3] = x;
                        e[4] = is_max;
                    }
                    ++n;
                }
        }
    }
    return n;
}

int dor_refine(const dor_scale_space* ss, const int32_t* e5, const dor_config* c,
               dor_keypoint* out) { /* detect.cpp:73-156 */
    const int s = ss->s, oct = e5[0];
    const int w = ss->w[oct], h = ss->h[oct];
    float* const* dog = ss->dog + oct * (s + 2);
    int x = e5[3], y = e5[2], i = e5[1];
    double dx = 0, dy = 0, ds = 0, gx = 0, gy = 0, gs = 0, dxx = 0, dyy = 0, dxy = 0;
    int converged = 0;
    for (int it = 0; it < c->max_refine_iters; ++it) {
        const float* D0 = dog[i - 1];
        const float* D1 = dog[i];
        const float* D2 = dog[i + 1];
        const double v = AT(D1, w, x, y);
        gx = 0.5 * ((double)AT(D1, w, x + 1, y) - AT(D1, w, x - 1, y));
        gy = 0.5 * ((double)AT(D1, w, x, y + 1) - AT(D1, w, x, y - 1));
        gs = 0.5 * ((double)AT(D2, w, x, y) - AT(D0, w, x, y));
        dxx = (double)AT(D1, w, x + 1, y) + AT(D1, w, x - 1, y) - 2.0 * v;
        dyy = (double)AT(D1, w, x, y + 1) + AT(D1, w, x, y - 1) - 2.0 * v;
        const double dss = (double)AT(D2, w, x, y) + AT(D0, w, x, y) - 2.0 * v;
        dxy = 0.25 * ((double)AT(D1, w, x + 1, y + 1) - AT(D1, w, x - 1, y + 1) -
                      AT(D1, w, x + 1, y - 1) + AT(D1, w, x - 1, y - 1));
        const double dxs = 0.25 * ((double)AT(D2, w, x + 1, y) - AT(D2, w, x - 1, y) -
                                   AT(D0, w, x + 1, y) + AT(D0, w, x - 1, y));
        const double dys = 0.25 * ((double)AT(D2, w, x, y + 1) - AT(D2, w, x, y - 1) -
                                   AT(D0, w, x, y + 1) + AT(D0, w, x, y - 1));
        /* Cramer's rule on H * delta = -g (detect.cpp:140-157) */
        const double det = dxx * (dyy * dss - dys * dys) - dxy * (dxy * dss - dys * dxs) +
                           dxs * (dxy * dys - dyy * dxs);
        if (fabs(det) < 1e-12) return 0;
        const double det_x = -gx * (dyy * dss - dys * dys) - dxy * (-gy * dss - dys * -gs) +
                             dxs * (-gy * dys - dyy * -gs);
        const double det_y = dxx * (-gy * dss - dys * -gs) - (-gx) * (dxy * dss - dys * dxs) +
                             dxs * (dxy * -gs - (-gy) * dxs);
        const double det_s = dxx * (dyy * -gs - (-gy) * dys) - dxy * (dxy * -gs - (-gy) * dxs) +
                             (-gx) * (dxy * dys - dyy * dxs);
        dx = det_x / det;
        dy = det_y / det;
        ds = det_s / det;
        if (fabs(dx) <= 0.5 && fabs(dy) <= 0.5 && fabs(ds) <= 0.5) {
            converged = 1;
            break;
        }
        if (dx > 0.5) ++x; else if (dx < -0.5) --x;
        if (dy > 0.5) ++y; else if (dy < -0.5) --y;
        if (ds > 0.5) ++i; else if (ds < -0.5) --i;
        if (x < 1 || x >= w - 1 || y < 1 || y >= h - 1 || i < 1 || i > s) return 0;
    }
    if (!converged) return 0;
    const double value = AT(dog[i], w, x, y) + 0.5 * (gx * dx + gy * dy + gs * ds);
    if (fabs(value) < (double)c->contrast_threshold / s) return 0;
    const double tr = dxx + dyy;
    const double det2 = dxx * dyy - dxy * dxy;
    const double r = c->edge_ratio;
    if (det2 <= 0.0 || tr * tr * r >= det2 * (r + 1.0) * (r + 1.0)) return 0;
    const double to_input = octave_to_input(ss, oct);
    out->x = (float)((x + dx) * to_input);
    out->y = (float)((y + dy) * to_input);
    out->sigma = (float)(ss->sigma0 * pow(2.0, oct + (i + ds) / s) * (ss->upsampled ? 0.5 : 1.0));
    out->angle = 0.0f;
    out->response = (float)fabs(value);
    out->octave = oct;
    out->interval = i;
    return 1;
}

int64_t dor_detect(const dor_scale_space* ss, const dor_config* c, dor_keypoint* out,
                   int64_t cap) { /* detect.cpp:158-172: candidate order kept */
    const int64_t nc = dor_find_extrema(ss, c, NULL, 0);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * 5 * (size_t)(nc > 0 ? nc : 1));
    dor_find_extrema(ss, c, cand, nc);
    int64_t n = 0;
    for (int64_t k = 0; k < nc; ++k) {
        dor_keypoint kp;
        if (dor_refine(ss, cand + 5 * k, c, &kp)) {
            if (n < cap) out[n] = kp;
            ++n;
        }
    }
    free(cand);
    return n;
}

/* ------------------------------------------------------------------------- */
/* Orientation (orient.cpp)                                                  */
/* ------------------------------------------------------------------------- */
int dor_nearest_gauss_level(const dor_scale_space* ss, double sigma_rel) { /* orient.cpp:13-24 */
    int best = 0;
    double best_diff = fabs(level_sigma(ss, 0) - sigma_rel);
    for (int i = 1; i < ss->s + 3; ++i) {
        const double d = fabs(level_sigma(ss, i) - sigma_rel);
        if (d < best_diff) {
            best_diff = d;
            best = i;
        }
    }
    return best;
}

int dor_orientation_histogram(const dor_scale_space* ss, const dor_keypoint* kp,
                              const dor_config* c, float* out) { /* orient.cpp:26-60 */
    const double to_input = octave_to_input(ss, kp->octave);
    const double cx = kp->x / to_input, cy = kp->y / to_input;
    const double sigma_rel = kp->sigma / to_input;
    const int lvl = dor_nearest_gauss_level(ss, sigma_rel);
    const float* img = ss->gauss[kp->octave * (ss->s + 3) + lvl];
    const int w = ss->w[kp->octave], h = ss->h[kp->octave];
    const int radius = (int)lround(3.0 * 1.5 * sigma_rel);
    const double denom = 2.0 * (1.5 * sigma_rel) * (1.5 * sigma_rel);
    const int bins = c->orientation_bins;
    const int x0 = (int)lround(cx), y0 = (int)lround(cy);
    hist_acc hist;
    if (hist_init(&hist, bins)) return fail(-2, "out of memory");
    for (int y = y0 - radius; y <= y0 + radius; ++y) {
        if (y < 1 || y >= h - 1) continue;
        for (int x = x0 - radius; x <= x0 + radius; ++x) {
            if (x < 1 || x >= w - 1) continue;
            const float gx = AT(img, w, x + 1, y) - AT(img, w, x - 1, y);
            const float gy = AT(img, w, x, y + 1) - AT(img, w, x, y - 1);
            const float mag = sqrtf(gx * gx + gy * gy);
            float theta = atan2f(gy, gx);
            if (theta < 0.0f) theta += (float)TWO_PI;
            int bin = (int)(theta * bins / TWO_PI);
            if (bin >= bins) bin -= bins;
            const double ddx = x - cx, ddy = y - cy;
            const float wgt = (float)exp(-(ddx * ddx + ddy * ddy) / denom);
            hist_add(&hist, bin, mag * wgt);
        }
    }
    hist_finish(&hist, out);
    return bins;
}

static void smooth_circular(float* hist, int n, int passes) { /* orient.cpp:62-75 */
    float* next = (float*)malloc(sizeof(float) * (size_t)n);
    for (int p = 0; p < passes; ++p) {
        for (int i = 0; i < n; ++i) {
            const double prev = hist[(i + n - 1) % n], mid = hist[i], succ = hist[(i + 1) % n];
            next[i] = (float)(0.25 * prev + 0.5 * mid + 0.25 * succ);
        }
        memcpy(hist, next, sizeof(float) * (size_t)n);
    }
    free(next);
}

int dor_assign_orientations(const dor_scale_space* ss, const dor_keypoint* kp,
                            const dor_config* c, dor_keypoint* out) { /* orient.cpp:77-113 */
    const int bins = c->orientation_bins;
    float* hist = (float*)malloc(sizeof(float) * (size_t)bins);
    int rc = dor_orientation_histogram(ss, kp, c, hist);
    if (rc < 0) {
        free(hist);
        return rc;
    }
    smooth_circular(hist, bins, 2);
    float max_val = 0.0f;
    for (int b = 0; b < bins; ++b)
        if (max_val < hist[b]) max_val = hist[b];
    int n = 0;
    if (max_val > 0.0f) {
        const float gate = c->orientation_peak_ratio * max_val;
        for (int b = 0; b < bins; ++b) {
            const float h0 = hist[b], hm = hist[(b + bins - 1) % bins], hp = hist[(b + 1) % bins];
            if (!(h0 > hm && h0 > hp && h0 >= gate)) continue;
            const double denom = (double)hm - 2.0 * h0 + hp;
            const double delta = denom != 0.0 ? 0.5 * ((double)hm - hp) / denom : 0.0;
            double angle = (b + delta) * TWO_PI / bins;
            if (angle < 0.0) angle += TWO_PI;
            if (angle >= TWO_PI) angle -= TWO_PI;
            dor_keypoint cp = *kp;
            cp.angle = (float)angle;
            if (cp.angle == 0.0f) cp.angle = 0.0f;
            if (cp.angle >= (float)TWO_PI) cp.angle = 0.0f;
            out[n++] = cp;
        }
    }
    if (n == 0) {
        out[0] = *kp;
        out[0].angle = 0.0f;
        n = 1;
    }
    free(hist);
    return n;
}

/* ------------------------------------------------------------------------- */
/* Descriptor (describe.cpp)                                                 */
/* ------------------------------------------------------------------------- */
static float sample_bilinear(const float* img, int w, int h, double x, double y) {
    /* describe.cpp:17-29 */
    int ix = (int)floor(x), iy = (int)floor(y);
    if (ix > w - 2) ix = w - 2;
    if (iy > h - 2) iy = h - 2;
    const float fx = (float)(x - ix), fy = (float)(y - iy);
    const float v00 = AT(img, w, ix, iy), v10 = AT(img, w, ix + 1, iy);
    const float v01 = AT(img, w, ix, iy + 1), v11 = AT(img, w, ix + 1, iy + 1);
    const float top = v00 + fx * (v10 - v00);
    const float bot = v01 + fx * (v11 - v01);
    return top + fy * (bot - top);
}

int dor_raw_descriptor(const dor_scale_space* ss, const dor_keypoint* kp, double f,
                       const dor_config* c, float* out) { /* describe.cpp:33-127 */
    (void)c;
    if (!(f > 0.0)) return fail(-1, "raw_descriptor: scale_factor must be > 0");
    const double to_input = octave_to_input(ss, kp->octave);
    const double cx = kp->x / to_input, cy = kp->y / to_input;
    const double sigma_rel = kp->sigma / to_input;
    const int lvl = dor_nearest_gauss_level(ss, f * sigma_rel);
    const float* img = ss->gauss[kp->octave * (ss->s + 3) + lvl];
    const int w = ss->w[kp->octave], h = ss->h[kp->octave];
    const int d = DESC_CELLS;
    const double bw = 3.0 * f * sigma_rel;
    const int radius = (int)lround(bw * (d + 1) * 0.5 * sqrt(2.0));
    const double cosa = cos((double)kp->angle), sina = sin((double)kp->angle);
    const int side = 2 * radius + 3;
    float* patch = (float*)malloc(sizeof(float) * (size_t)side * side);
    for (size_t p = 0; p < (size_t)side * side; ++p) patch[p] = UNDEFINED_SAMPLE;
    for (int v = -radius - 1; v <= radius + 1; ++v)
        for (int u = -radius - 1; u <= radius + 1; ++u) {
            const double px = cx + cosa * u - sina * v;
            const double py = cy + sina * u + cosa * v;
            if (px < 0.0 || px > w - 1 || py < 0.0 || py > h - 1) continue;
            patch[(size_t)(v + radius + 1) * side + (u + radius + 1)] =
                sample_bilinear(img, w, h, px, py);
        }
#define PATCH(u, v) patch[(size_t)((v) + radius + 1) * side + ((u) + radius + 1)]
    hist_acc hist;
    hist_init(&hist, DESC_DIM);
    for (int v = -radius; v <= radius; ++v)
        for (int u = -radius; u <= radius; ++u) {
            const float left = PATCH(u - 1, v), right = PATCH(u + 1, v);
            const float up = PATCH(u, v - 1), down = PATCH(u, v + 1);
            if (left == UNDEFINED_SAMPLE || right == UNDEFINED_SAMPLE || up == UNDEFINED_SAMPLE ||
                down == UNDEFINED_SAMPLE)
                continue;
            const double ubin = u / bw + (d / 2 - 0.5);
            const double vbin = v / bw + (d / 2 - 0.5);
            if (ubin <= -1.0 || ubin >= d || vbin <= -1.0 || vbin >= d) continue;
            const float du = 0.5f * (right - left);
            const float dv = 0.5f * (down - up);
            const float mag = sqrtf(du * du + dv * dv);
            float theta = atan2f(dv, du);
            if (theta < 0.0f) theta += (float)TWO_PI;
            double obin = theta * DESC_ORIENTS / TWO_PI;
            if (obin >= DESC_ORIENTS) obin -= DESC_ORIENTS;
            const double uu = u / bw, vv = v / bw;
            const float wgt = (float)exp(-(uu * uu + vv * vv) / (2.0 * (0.5 * d) * (0.5 * d)));
            const float value = mag * wgt;
            const int r0 = (int)floor(vbin), c0 = (int)floor(ubin), o0 = (int)floor(obin);
            const float fr = (float)(vbin - r0), fc = (float)(ubin - c0), fo = (float)(obin - o0);
            for (int ri = 0; ri < 2; ++ri) {
                const int row = r0 + ri;
                if (row < 0 || row >= d) continue;
                const float wr = ri ? fr : 1.0f - fr;
                for (int ci = 0; ci < 2; ++ci) {
                    const int col = c0 + ci;
                    if (col < 0 || col >= d) continue;
                    const float wc = ci ? fc : 1.0f - fc;
                    for (int oi = 0; oi < 2; ++oi) {
                        const int ob = (o0 + oi) % DESC_ORIENTS;
                        const float wo = oi ? fo : 1.0f - fo;
                        hist_add(&hist, (row * d + col) * DESC_ORIENTS + ob, value * wr * wc * wo);
                    }
                }
            }
        }
#undef PATCH
    hist_finish(&hist, out);
    free(patch);
    return 0;
}

int dor_root_sift(float* v, int n) { /* describe.cpp:129-136 */
    for (int i = 0; i < n; ++i)
        if (v[i] < 0.0f) return fail(-1, "root_sift: negative component");
    const float l1 = dor_tree_sum(v, n);
    if (l1 == 0.0f) return 0;
    for (int i = 0; i < n; ++i) v[i] = sqrtf(v[i] / l1);
    return 0;
}

static float l2_norm(const float* v, int n) { /* describe.cpp:140-144 */
    float sq[DESC_DIM];
    for (int i = 0; i < n; ++i) sq[i] = v[i] * v[i];
    return sqrtf(dor_tree_sum(sq, n));
}

int dor_dsp_descriptor(const dor_scale_space* ss, const dor_keypoint* kp, const dor_config* c,
                       float* out) { /* describe.cpp:148-173 */
    const int ns = c->n_dsp_scales;
    float* raws = (float*)malloc(sizeof(float) * DESC_DIM * (size_t)ns);
    for (int k = 0; k < ns; ++k) {
        int rc = dor_raw_descriptor(ss, kp, c->dsp_scales[k], c, raws + k * DESC_DIM);
        if (rc) {
            free(raws);
            return rc;
        }
    }
    float stack[64];
    for (int b = 0; b < DESC_DIM; ++b) {
        for (int k = 0; k < ns; ++k) stack[k] = raws[k * DESC_DIM + b];
        out[b] = dor_tree_sum(stack, ns) / (float)ns;
    }
    free(raws);
    float norm = l2_norm(out, DESC_DIM);
    if (norm == 0.0f) return 0;
    for (int b = 0; b < DESC_DIM; ++b) out[b] /= norm;
    for (int b = 0; b < DESC_DIM; ++b)
        if (c->descriptor_clip < out[b]) out[b] = c->descriptor_clip;
    norm = l2_norm(out, DESC_DIM);
    if (norm > 0.0f)
        for (int b = 0; b < DESC_DIM; ++b) out[b] /= norm;
    return dor_root_sift(out, DESC_DIM);
}

/* ------------------------------------------------------------------------- */
/* Canonical order + DSF1 + SHA-256 (core.cpp:116-196, sha256.cpp)           */
/* ------------------------------------------------------------------------- */
static const dor_keypoint* g_sort_kps;
static const float* g_sort_desc;

static int kp_cmp(const void* pa, const void* pb) { /* core.cpp:116-128 total order */
    const int64_t i = *(const int64_t*)pa, j = *(const int64_t*)pb;
    const dor_keypoint *a = &g_sort_kps[i], *b = &g_sort_kps[j];
#define KEY(f) if (a->f != b->f) return a->f < b->f ? -1 : 1
    KEY(octave);
    KEY(interval);
    KEY(y);
    KEY(x);
    KEY(angle);
    KEY(sigma);
    KEY(response);
#undef KEY
    const float *ra = g_sort_desc + i * DESC_DIM, *rb = g_sort_desc + j * DESC_DIM;
    for (int k = 0; k < DESC_DIM; ++k)
        if (ra[k] != rb[k]) return ra[k] < rb[k] ? -1 : 1;
    return 0;
}

void dor_canonical_sort(dor_keypoint* kps, float* desc, int64_t n) {
    if (n <= 1) return;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_sort_kps = kps;
    g_sort_desc = desc;
    qsort(order, (size_t)n, sizeof(int64_t), kp_cmp);
    dor_keypoint* k2 = (dor_keypoint*)malloc(sizeof(dor_keypoint) * (size_t)n);
    float* d2 = (float*)malloc(sizeof(float) * DESC_DIM * (size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        k2[i] = kps[order[i]];
        memcpy(d2 + i * DESC_DIM, desc + order[i] * DESC_DIM, sizeof(float) * DESC_DIM);
    }
    memcpy(kps, k2, sizeof(dor_keypoint) * (size_t)n);
    memcpy(desc, d2, sizeof(float) * DESC_DIM * (size_t)n);
    free(k2);
    free(d2);
    free(order);
}

int64_t dor_serialize(const dor_keypoint* kps, const float* desc, int64_t n, uint8_t* out,
                      int64_t cap) {
    /* DSF1: "DSF1", u32 version 1, u32 count, u32 dim, 28 B/keypoint, N x dim f32. */
    /* Input must already be in canonical order (dor_extract guarantees it).       */
    const int64_t size = 16 + n * (28 + DESC_DIM * 4);
    if (!out || cap < size) return size;
    const uint32_t hdr[3] = {1u, (uint32_t)n, (uint32_t)DESC_DIM};
    memcpy(out, "DSF1", 4);
    memcpy(out + 4, hdr, 12);
    memcpy(out + 16, kps, (size_t)n * 28);
    memcpy(out + 16 + n * 28, desc, (size_t)n * DESC_DIM * 4);
    return size;
}

/* SHA-256 (FIPS 180-4) */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

#define ROR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void sha_block(uint32_t st[8], const uint8_t* p) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
        w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 |
               (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
        const uint32_t s0 = ROR(w[i - 15], 7) ^ ROR(w[i - 15], 18) ^ (w[i - 15] >> 3);
        const uint32_t s1 = ROR(w[i - 2], 17) ^ ROR(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6],
             h = st[7];
    for (int i = 0; i < 64; ++i) {
        const uint32_t t1 = h + (ROR(e, 6) ^ ROR(e, 11) ^ ROR(e, 25)) + ((e & f) ^ (~e & g)) +
                            K256[i] + w[i];
        const uint32_t t2 = (ROR(a, 2) ^ ROR(a, 13) ^ ROR(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g;
        g = f;
        f = e;
        e = d + t1;
        d = c;
        c = b;
        b = a;
        a = t1 + t2;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d;
    st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

void dor_sha256(const uint8_t* p, int64_t n, char* hex65) {
    uint32_t st[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                      0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    int64_t i = 0;
    for (; i + 64 <= n; i += 64) sha_block(st, p + i);
    uint8_t tail[128];
    memset(tail, 0, sizeof tail);
    const int rem = (int)(n - i);
    memcpy(tail, p + i, (size_t)rem);
    tail[rem] = 0x80;
    const int tl = rem + 9 <= 64 ? 64 : 128;
    const uint64_t bits = (uint64_t)n * 8u;
    for (int k = 0; k < 8; ++k) tail[tl - 1 - k] = (uint8_t)(bits >> (8 * k));
    sha_block(st, tail);
    if (tl == 128) sha_block(st, tail + 64);
    for (int k = 0; k < 8; ++k) sprintf(hex65 + 8 * k, "%08x", st[k]);
    hex65[64] = 0;
}

void dor_hash_features(const dor_keypoint* kps, const float* desc, int64_t n, char* hex65) {
    const int64_t size = dor_serialize(kps, desc, n, NULL, 0);
    uint8_t* buf = (uint8_t*)malloc((size_t)size);
    dor_serialize(kps, desc, n, buf, size);
    dor_sha256(buf, size, hex65);
    free(buf);
}

/* ------------------------------------------------------------------------- */
/* Full pipeline (io.cpp:111-142)                                            */
/* ------------------------------------------------------------------------- */
void dor_free(void* p) { free(p); }

int dor_extract(const float* img, int w, int h, const dor_config* c, dor_keypoint** kps_out,
                float** desc_out, int64_t* n_out) {
    dor_scale_space* ss = NULL;
    int rc = dor_build_scale_space(img, w, h, c, &ss);
    if (rc) return rc;
    const int64_t nk = dor_detect(ss, c, NULL, 0);
    dor_keypoint* det = (dor_keypoint*)malloc(sizeof(dor_keypoint) * (size_t)(nk ? nk : 1));
    dor_detect(ss, c, det, nk);
    /* orientation fan-out, flattened in detection order */
    int64_t cap = nk * 4 + 16, n = 0;
    dor_keypoint* kps = (dor_keypoint*)malloc(sizeof(dor_keypoint) * (size_t)cap);
    dor_keypoint* tmp =
        (dor_keypoint*)malloc(sizeof(dor_keypoint) * (size_t)(c->orientation_bins + 1));
    for (int64_t k = 0; k < nk; ++k) {
        const int m = dor_assign_orientations(ss, &det[k], c, tmp);
        if (n + m > cap) {
            cap = 2 * (n + m);
            kps = (dor_keypoint*)realloc(kps, sizeof(dor_keypoint) * (size_t)cap);
        }
        memcpy(kps + n, tmp, sizeof(dor_keypoint) * (size_t)m);
        n += m;
    }
    free(tmp);
    free(det);
    float* desc = (float*)malloc(sizeof(float) * DESC_DIM * (size_t)(n ? n : 1));
    for (int64_t k = 0; k < n; ++k) dor_dsp_descriptor(ss, &kps[k], c, desc + k * DESC_DIM);
    dor_canonical_sort(kps, desc, n);
    dor_ss_free(ss);
    *kps_out = kps;
    *desc_out = desc;
    *n_out = n;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Synthetic input (tests/support/synth.cpp:14-66)                           */
/* ------------------------------------------------------------------------- */
static uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

static double lattice(uint64_t seed, int64_t gx, int64_t gy) {
    const uint64_t hsh =
        mix64(seed ^ mix64((uint64_t)gx * 0x9e3779b97f4a7c15ull ^ (uint64_t)gy * 0xbf58476d1ce4e5b9ull));
    return (double)(hsh >> 11) * (1.0 / 9007199254740992.0);
}

static double smooth_noise(uint64_t seed, double x, double y) {
    const int64_t gx = (int64_t)floor(x), gy = (int64_t)floor(y);
    const double fx = x - gx, fy = y - gy;
    const double sx = fx * fx * (3.0 - 2.0 * fx), sy = fy * fy * (3.0 - 2.0 * fy);
    const double v00 = lattice(seed, gx, gy), v10 = lattice(seed, gx + 1, gy);
    const double v01 = lattice(seed, gx, gy + 1), v11 = lattice(seed, gx + 1, gy + 1);
    const double top = v00 + sx * (v10 - v00), bot = v01 + sx * (v11 - v01);
    return top + sy * (bot - top);
}

void dor_value_noise(int w, int h, uint64_t seed, int octaves, int cells, float* out) {
    double lo = 1e9, hi = -1e9;
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x) {
            double v = 0.0, amp = 1.0, cl = cells;
            for (int o = 0; o < octaves; ++o) {
                v += amp * smooth_noise(seed + (uint64_t)o, x * cl / w, y * cl / h);
                amp *= 0.55;
                cl *= 2.0;
            }
            out[(size_t)y * w + x] = (float)v;
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
    const double span = hi > lo ? hi - lo : 1.0;
    for (size_t p = 0; p < (size_t)w * h; ++p) out[p] = (float)((out[p] - lo) / span);
}

/* ------------------------------------------------------------------------- */
/* load_image (io.cpp:17-81): binary P5/P6, maxval 255.  Returns 0, or -2 with
 * the reference's std::runtime_error message.  With out == NULL only *w, *h
 * are set; out receives w*h floats. */
static int pnm_token(FILE* f, char* tok, int cap) { /* io.cpp:17-35 */
    int n = 0, ch;
    while ((ch = fgetc(f)) != EOF) {
        if (ch == '#') {
            while ((ch = fgetc(f)) != EOF && ch != '\n') {
            }
            continue;
        }
        if (isspace(ch)) {
            if (n) break;
            continue;
        }
        if (n < cap - 1) tok[n++] = (char)ch;
    }
    tok[n] = 0;
    return n;
}

static int pnm_dim(const char* tok, int* v) { /* io.cpp:37-45: std::stoi, > 0 */
    const char* p = tok;
    long long x = 0;
    int sign = 1, digits = 0;
    if (*p == '+' || *p == '-') sign = (*p++ == '-') ? -1 : 1;
    while (*p >= '0' && *p <= '9') {
        x = x * 10 + (*p++ - '0');
        ++digits;
        if (x > 2147483647LL) return 0;
    }
    x *= sign;
    if (!digits || x <= 0) return 0;
    *v = (int)x;
    return 1;
}

int dor_load_image(const char* path, int* w, int* h, float* out) {
    char tok[64], msg[200];
    int width, height, maxval;
    FILE* f = fopen(path, "rb");
    if (!f) {
        snprintf(msg, sizeof msg, "cannot open: %.150s", path);
        return fail(-2, msg);
    }
    pnm_token(f, tok, sizeof tok);
    const int color = strcmp(tok, "P6") == 0;
    if (!color && strcmp(tok, "P5") != 0) {
        snprintf(msg, sizeof msg, "image: unsupported format '%s' (want P5/P6)", tok);
        fclose(f);
        return fail(-2, msg);
    }
    pnm_token(f, tok, sizeof tok);
    if (!pnm_dim(tok, &width)) { fclose(f); return fail(-2, "image: bad width"); }
    pnm_token(f, tok, sizeof tok);
    if (!pnm_dim(tok, &height)) { fclose(f); return fail(-2, "image: bad height"); }
    pnm_token(f, tok, sizeof tok);
    if (!pnm_dim(tok, &maxval)) { fclose(f); return fail(-2, "image: bad maxval"); }
    if (maxval != 255) { fclose(f); return fail(-2, "image: maxval must be 255"); }
    *w = width;
    *h = height;
    if (!out) { fclose(f); return 0; }
    const size_t pixels = (size_t)width * height, payload = pixels * (color ? 3 : 1);
    unsigned char* bytes = (unsigned char*)malloc(payload ? payload : 1);
    const size_t got = fread(bytes, 1, payload, f);
    fclose(f);
    if (got != payload) { free(bytes); return fail(-2, "image: truncated payload"); }
    for (size_t i = 0; i < pixels; ++i) {
        if (color) { /* io.cpp:71-75 */
            const double r = bytes[3 * i], g = bytes[3 * i + 1], b = bytes[3 * i + 2];
            out[i] = (float)((0.299 * r + 0.587 * g + 0.114 * b) * (1.0 / 255.0));
        } else { /* io.cpp:77-78 */
            out[i] = (float)(bytes[i] * (1.0 / 255.0));
        }
    }
    free(bytes);
    return 0;
}
