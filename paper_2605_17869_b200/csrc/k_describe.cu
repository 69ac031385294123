// k_describe.cu — K5+K6: DSP-SIFT descriptors with the reference's exact
// arithmetic (describe.cpp:17-173, detsum.cpp:13-127).
//
// One CTA (128 threads) per keypoint, persistent over the keypoint list.  Per
// support scale f the CTA:
//   1. builds the per-axis lattice tables: u/bin_width, bin = u/bw + 1.5, its
//      floor and float fraction, (u/bw)^2, and the rotated-frame coordinate
//      partials cx + cos*u, cy + sin*u, sin*v, cos*v (describe.cpp:48-52,
//      72-73, 89-99) — so every per-point double op is the reference's own;
//   2. walks the in-range lattice rows in chunks: samples the Gaussian level
//      bilinearly (float lerp, describe.cpp:17-29) on the chunk rows + guard
//      ring, then computes per point the float gradient, sqrtf, glibc-exact
//      atan2f, orientation bin and float(exp()) weight (describe.cpp:76-100);
//      lattice points outside the (-1, 4) bin range are never sampled — they
//      contribute nothing in the reference either;
//   3. accumulates: thread b owns histogram bin b = (row, col, ori) and scans
//      the points of its 2x2-cell rectangle in the reference's scan order,
//      forming value*wr*wc*wo in float and pushing it into a register binary
//      counter — the exact per-bin tree of tree_accumulate_histogram.
// The epilogue forms the DSP mean (fixed tree over scales), L2 -> clip 0.2 ->
// L2 -> RootSIFT with 128-leaf trees done as warp xor-shuffles (the complete
// dyadic tree), and writes float32 plus the uint8 export q(v).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_math.cuh"
#include "dsift_tree.cuh"


namespace dsift {

DSIFT_BOUNDS_UNIT(describe)
#ifdef DSIFT_BOUNDS_CHECK
// the counters' own check: one deliberately failing condition (site 999)
__global__ void bounds_selftest_kernel() { DSIFT_BOUND(threadIdx.x > 0, 999); }
extern "C" int dsift_test_bounds_selftest(void) {
    bounds_selftest_kernel<<<1, 1>>>();
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : -1;
}
#endif

constexpr int kDescThreads = 128;
// per-bin tree depth: DescArgs::tree_depth (13 for the defaults, at most 24: leaves < 2^24)
constexpr int kRing = 32;
constexpr float kUndef = -1.0f;  // describe.cpp:188

struct DescSmem {
    // per-axis tables indexed by k - kbase, k in [-r-1, r+1]
    double* q2;
    double* bin;
    double* ax;     // cx + cos*u
    double* cy_su;  // cy + sin*u
    double* sv;     // sin*v
    double* cv;     // cos*v
    float* frac;
    int* c0;
    float* samp;    // [(chunk+2)][max_axis]
    float* pval;    // [chunk][pw]
    float* pfo;     // [chunk][pw]
    unsigned* omask;  // [chunk][8][nw]: bit cc set iff point o0 == o
    float* raw;     // [n_dsp][128]
    float* ring;    // [kRing][128]: per-bin leaves not yet folded (slot-major)
    double* node;   // [tree_depth-3][128]: per-bin pending 8-leaf-aligned tree nodes
};

__device__ __forceinline__ int nearest_level_d(const PyramidDesc& p, double sigma_rel) {
    int best = 0;
    double best_diff = fabs(p.level_sigma[0] - sigma_rel);
    for (int i = 1; i < p.s + 3; ++i) {
        const double d = fabs(p.level_sigma[i] - sigma_rel);
        if (d < best_diff) {
            best_diff = d;
            best = i;
        }
    }
    return best;
}

// sample_bilinear (describe.cpp:17-29)
__device__ __forceinline__ float sample_bilinear(const float* __restrict__ img, int w, int h, int pitch,
                                                 double x, double y) {
    int ix = (int)floor(x), iy = (int)floor(y);
    ix = min(ix, w - 2);
    iy = min(iy, h - 2);
    const float fx = (float)D_SUB(x, (double)ix), fy = (float)D_SUB(y, (double)iy);
    const float* r0 = img + (long long)iy * pitch + ix;
    const float v00 = __ldg(r0), v10 = __ldg(r0 + 1);
    const float v01 = __ldg(r0 + pitch), v11 = __ldg(r0 + pitch + 1);
    const float top = F_ADD(v00, F_MUL(fx, F_SUB(v10, v00)));
    const float bot = F_ADD(v01, F_MUL(fx, F_SUB(v11, v01)));
    return F_ADD(top, F_MUL(fy, F_SUB(bot, top)));
}

// 128-leaf fixed tree over one value per thread (complete dyadic tree).
__device__ __forceinline__ double tree128(double v, double* red) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) v = v + __shfl_xor_sync(0xffffffffu, v, d);
    const int warp = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[warp] = v;
    __syncthreads();
    return (red[0] + red[1]) + (red[2] + red[3]);
}

__device__ __forceinline__ void raw_descriptor_cta(const DescArgs& a, const DescSmem& S, const DevKeypoint& kp,
                                                   double f, double cosa, double sina, float* raw_out) {
    const PyramidDesc& p = a.pyr;
    const OctaveDesc& od = p.oct[kp.octave];
    const double to_input = ldexp(1.0, kp.octave) * (p.upsampled ? 0.5 : 1.0);
    const double cx = kp.x / to_input, cy = kp.y / to_input;
    const double sigma_rel = kp.sigma / to_input;
    const int lvl = nearest_level_d(p, f * sigma_rel);
    const float* __restrict__ img =
        od.gauss + (long long)kp.image * p.gauss_img_stride(kp.octave) + (long long)lvl * od.level_stride;
    const int w = od.w, h = od.h, pitch = od.pitch;
    const double bw = 3.0 * f * sigma_rel;
    const int radius = (int)llround(bw * (kDescCells + 1) * 0.5 * 1.4142135623730951);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (2 * radius + 3 > a.max_axis) {   // host sized the tables for r_max; never silently clip
        if (tid == 0) atomicOr(a.err, kErrDescriptorLattice);
        raw_out[tid] = 0.0f;
        __syncthreads();
        return;
    }
    const int kbase = -radius - 1;
    const int naxis = 2 * radius + 3;

    // 1. per-axis tables (describe.cpp:48-52, 72-73, 89-99 per-axis factors)
    for (int i = tid; i < naxis; i += kDescThreads) {
        const int k = kbase + i;
        const double q = D_DIV((double)k, bw);
        const double bn = D_ADD(q, (double)(kDescCells / 2 - 0.5));
        const int c = (int)floor(bn);
        S.q2[i] = D_MUL(q, q);
        S.bin[i] = bn;
        S.c0[i] = c;
        S.frac[i] = (float)D_SUB(bn, (double)c);
        S.ax[i] = D_ADD(cx, D_MUL(cosa, (double)k));
        S.cy_su[i] = D_ADD(cy, D_MUL(sina, (double)k));
        S.sv[i] = D_MUL(sina, (double)k);
        S.cv[i] = D_MUL(cosa, (double)k);
    }
    __syncthreads();
    // in-range lattice span [kmin, kmax] (bin in (-1, 4), contiguous since k/bw is monotone)
    int kmin = 1 << 30, kmax = -(1 << 30);
    for (int i = 1; i < naxis - 1; ++i) {   // k in [-r, r]
        const double bn = S.bin[i];
        if (bn > -1.0 && bn < (double)kDescCells) {
            kmin = min(kmin, kbase + i);
            kmax = max(kmax, kbase + i);
        }
    }
    const int width = kmax - kmin + 1;       // points per lattice row
    const int swidth = width + 2;            // samples per row (guard ring)
    const int nw = (width + 31) >> 5;        // 32-point mask words per row
    const int pw = nw << 5;
    // bin owned by this thread: (row, col, ori) = describe.cpp:116 bin layout
    const int brow = tid >> 5, bcol = (tid >> 3) & 3, bori = tid & 7;
    int ua = 1 << 30, ub = -(1 << 30), va = 1 << 30, vb = -(1 << 30);
    for (int k = kmin; k <= kmax; ++k) {
        const int c = S.c0[k - kbase];
        if (c == bcol - 1 || c == bcol) { ua = min(ua, k); ub = max(ub, k); }
        if (c == brow - 1 || c == brow) { va = min(va, k); vb = max(vb, k); }
    }
    const int ca = ua - kmin, cb = ub - kmin;   // this bin's column span in the point rows
    // Per-bin fixed tree (detsum.cpp:13-71) as a binary counter whose three
    // lowest levels are folded 8 leaves at a time: leaves land in a shared
    // ring; every complete aligned 8-leaf block is reduced with the reference's
    // pairing ((l0+l1)+(l2+l3))+((l4+l5)+(l6+l7)) and pushed as one node into
    // a shared-memory counter over 8-blocks.  Same tree, no per-leaf branching.
    float* ring = S.ring + tid;
    double* node = S.node + tid;
    unsigned cnt = 0, flushed = 0;
    auto flush = [&]() {
        while (cnt - flushed >= 8u) {
            double l[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) l[i] = (double)ring[((flushed + i) & (kRing - 1)) * kDescThreads];
            double t = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
            unsigned m = flushed >> 3;
            int j = 0;
            while (m & 1u) {
                t = node[j * kDescThreads] + t;
                m >>= 1;
                ++j;
            }
            node[j * kDescThreads] = t;
            flushed += 8;
        }
    };

    const int ch = a.chunk_rows;
    for (int v0 = kmin; v0 <= kmax; v0 += ch) {
        const int v1 = min(v0 + ch - 1, kmax);
        const int nrows = v1 - v0 + 1;
        // 2a. samples on rows [v0-1, v1+1] x cols [kmin-1, kmax+1]
        for (int idx = tid; idx < (nrows + 2) * swidth; idx += kDescThreads) {
            const int rr = idx / swidth, cc = idx - rr * swidth;
            const int v = v0 - 1 + rr, u = kmin - 1 + cc;
            const double px = D_SUB(S.ax[u - kbase], S.sv[v - kbase]);
            const double py = D_ADD(S.cy_su[u - kbase], S.cv[v - kbase]);
            float sv = kUndef;
            if (!(px < 0.0 || px > (double)(w - 1) || py < 0.0 || py > (double)(h - 1)))
                sv = sample_bilinear(img, w, h, pitch, px, py);
            S.samp[idx] = sv;
        }
        __syncthreads();
        // 2b. per-point gradient, orientation, weight; a warp owns 32 aligned points
        //     of one row and publishes 8 orientation-membership masks by ballot
        for (int task = warp; task < nrows * nw; task += kDescThreads / 32) {
            const int rr = task / nw, wd = task - rr * nw;
            const int cc = (wd << 5) + lane;
            const int v = v0 + rr, u = kmin + cc;
            int o0 = 8;
            float value = 0.0f, fo = 0.0f;
            if (cc < width) {
                const float* sr = S.samp + (rr + 1) * swidth + (cc + 1);
                const float left = sr[-1], right = sr[1], up = sr[-swidth], down = sr[swidth];
                if (!(left == kUndef || right == kUndef || up == kUndef || down == kUndef)) {
                    const float du = F_MUL(0.5f, F_SUB(right, left));
                    const float dv = F_MUL(0.5f, F_SUB(down, up));
                    const float mag = F_SQRT(F_ADD(F_MUL(du, du), F_MUL(dv, dv)));
                    float theta = dsift_atan2f(dv, du);
                    if (theta < 0.0f) theta = F_ADD(theta, (float)kTwoPi);
                    if (isnan(theta)) {   // reference: negative bin -> std::out_of_range
                        atomicOr(a.err, kErrHistogramRange);
                        theta = 0.0f;
                    }
                    double obin = ds_div_2pi((double)F_MUL(theta, (float)kDescOrients));
                    if (obin >= (double)kDescOrients) obin = D_SUB(obin, (double)kDescOrients);
                    // -(uu^2 + vv^2) / 8: division by 8 is an exact scaling, == * 0.125
                    const double arg = D_MUL(-D_ADD(S.q2[u - kbase], S.q2[v - kbase]), 0.125);
                    const float wgt = (float)dsift_exp(arg);
                    value = F_MUL(mag, wgt);
                    o0 = (int)floor(obin);
                    fo = (float)D_SUB(obin, (double)o0);
                }
            }
            S.pval[rr * pw + cc] = value;
            S.pfo[rr * pw + cc] = fo;
#pragma unroll
            for (int o = 0; o < kDescOrients; ++o) {
                const unsigned m = __ballot_sync(0xffffffffu, o0 == o);
                if (lane == o) S.omask[(rr * kDescOrients + o) * nw + wd] = m;
            }
        }
        __syncthreads();
        // 3. bin-owner accumulation in scan order (describe.cpp:102-126): only the
        //    points whose o0 or o0+1 is this bin's orientation are visited.
        const int ra = max(va, v0), rb = min(vb, v1);
        const int om1 = (bori + kDescOrients - 1) & (kDescOrients - 1);
        for (int v = ra; v <= rb; ++v) {
            const int rr = v - v0;
            const int r0 = S.c0[v - kbase];
            const float fr = S.frac[v - kbase];
            const float wr = (brow - r0) ? fr : F_SUB(1.0f, fr);
            const unsigned* mo = S.omask + (rr * kDescOrients + bori) * nw;
            const unsigned* mp = S.omask + (rr * kDescOrients + om1) * nw;
            for (int hw = (ca >> 4); hw <= (cb >> 4); ++hw) {   // 16-point half words
                const int wd = hw >> 1;
                const int lo = max(ca - (wd << 5), 0), hi = min(cb - (wd << 5), 31);
                const unsigned range = (hi >= 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u) &
                                       ((hw & 1) ? 0xffff0000u : 0x0000ffffu);
                const unsigned a0 = mo[wd];
                unsigned bits = (a0 | mp[wd]) & range;
                while (bits) {
                    const int bpos = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int cc = (wd << 5) + bpos;
                    const int u = kmin + cc;
                    const int c0 = S.c0[u - kbase];
                    const float fc = S.frac[u - kbase];
                    const float wc = (bcol - c0) ? fc : F_SUB(1.0f, fc);
                    const float fo = S.pfo[rr * pw + cc];
                    const float wo = ((a0 >> bpos) & 1u) ? F_SUB(1.0f, fo) : fo;
                    const float val = F_MUL(F_MUL(F_MUL(S.pval[rr * pw + cc], wr), wc), wo);
                    ring[(cnt & (kRing - 1)) * kDescThreads] = val;
                    ++cnt;
                }
                flush();
            }
        }
        __syncthreads();
    }
    // fold the pending nodes smallest-first: the < 8 tail leaves (as their
    // 4/2/1 aligned blocks), then the 8-block counter levels
    {
        const unsigned m = cnt - flushed;
        double r = 0.0;
        bool have = false;
        unsigned p = flushed + (m & 4u) + (m & 2u);
        if (m & 1u) {
            r = (double)ring[(p & (kRing - 1)) * kDescThreads];
            have = true;
        }
        if (m & 2u) {
            p = flushed + (m & 4u);
            const double v2 = (double)ring[(p & (kRing - 1)) * kDescThreads] +
                              (double)ring[((p + 1) & (kRing - 1)) * kDescThreads];
            r = have ? v2 + r : v2;
            have = true;
        }
        if (m & 4u) {
            double l[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) l[i] = (double)ring[((flushed + i) & (kRing - 1)) * kDescThreads];
            const double v4 = (l[0] + l[1]) + (l[2] + l[3]);
            r = have ? v4 + r : v4;
            have = true;
        }
        unsigned hb = flushed >> 3;
        for (int j = 0; hb; ++j, hb >>= 1)
            if (hb & 1u) {
                r = have ? node[j * kDescThreads] + r : node[j * kDescThreads];
                have = true;
            }
        raw_out[tid] = (float)r;
    }
    __syncthreads();
}

// DSP mean over scales, L2 -> clip -> L2 -> RootSIFT, float + uint8 outputs
// (describe.cpp:138-173); one value per thread (bin = threadIdx.x).
__device__ __forceinline__ void dsp_epilogue(const DescArgs& a, const float* raw, long long k, double* red) {
    const int tid = threadIdx.x;
    TreeCounter<5> tc;   // n_dsp <= kMaxDsp = 16 leaves
    tc.reset();
    for (int fi = 0; fi < a.n_dsp; ++fi) tc.push((double)raw[fi * kDescDim + tid]);
    float d = F_DIV((float)tc.result(), (float)a.n_dsp);
    float norm = F_SQRT((float)tree128((double)F_MUL(d, d), red));
    if (norm != 0.0f) {
        d = F_DIV(d, norm);
        d = (a.clip < d) ? a.clip : d;
        norm = F_SQRT((float)tree128((double)F_MUL(d, d), red));
        if (norm > 0.0f) d = F_DIV(d, norm);
        const float l1 = (float)tree128((double)d, red);
        if (l1 != 0.0f) d = F_SQRT(F_DIV(d, l1));
    }
    a.desc[k * kDescDim + tid] = d;
    if (a.desc_u8) {
        long long q = llround((double)d * 255.0);
        a.desc_u8[k * kDescDim + tid] = (unsigned char)(q > 255 ? 255 : (q < 0 ? 0 : q));
    }
}

// Shared-memory carve of the exact path: raw[nraw][128] first, then the
// per-scale working set (whose size exact_work_bytes reports).
__device__ __forceinline__ DescSmem carve_exact_smem(unsigned char* pbuf, const DescArgs& a, int nraw) {
    const int A = a.max_axis;
    const int PW = ((A + 31) >> 5) << 5;
    DescSmem S;
    S.raw = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * kDescDim * nraw;
    S.q2 = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.bin = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.ax = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.cy_su = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.sv = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.cv = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.frac = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * A;
    S.c0 = reinterpret_cast<int*>(pbuf); pbuf += sizeof(int) * A;
    S.samp = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * (a.chunk_rows + 2) * A;
    S.pval = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * a.chunk_rows * PW;
    S.pfo = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * a.chunk_rows * PW;
    S.omask = reinterpret_cast<unsigned*>(pbuf); pbuf += sizeof(unsigned) * a.chunk_rows * kDescOrients * (PW >> 5);
    pbuf += (16u - ((unsigned)__cvta_generic_to_shared(pbuf) & 15u)) & 15u;   // 16-byte align, stays a shared pointer
    S.node = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * (a.tree_depth - 3) * kDescThreads;
    S.ring = reinterpret_cast<float*>(pbuf);
    return S;
}

// Exact path: per-bin scan-order trees (bit-identical by construction).  Runs
// over all keypoints in stage mode, and over the keypoints the fast path
// could not certify in the hot path.
__global__ void __launch_bounds__(kDescThreads, 4)
describe_exact_kernel(const __grid_constant__ DescArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[4];
    DescSmem S = carve_exact_smem(sm, a, a.raw_mode ? 1 : a.n_dsp);

    const long long n = a.slow_list ? (long long)*a.n_slow : (a.n_host >= 0 ? a.n_host : (long long)*a.n_dev);
    const int tid = threadIdx.x;
    for (long long i = blockIdx.x; i < n; i += gridDim.x) {
        const long long k = a.slow_list ? (long long)a.slow_list[i] : i;
        const DevKeypoint kp = a.kps[k];
        const double2 cs = a.trig[k];   // (cos, sin) of the keypoint angle (trig_kernel)
        const double cosa = cs.x, sina = cs.y;
        if (a.raw_mode) {
            raw_descriptor_cta(a, S, kp, a.raw_scale, cosa, sina, S.raw);
            a.desc[k * kDescDim + tid] = S.raw[tid];
            __syncthreads();
            continue;
        }
        for (int fi = 0; fi < a.n_dsp; ++fi)
            raw_descriptor_cta(a, S, kp, a.dsp[fi], cosa, sina, S.raw + fi * kDescDim);
        dsp_epilogue(a, S.raw, k, red);
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------
// Certified order-free accumulation.
//
// Every histogram bin of describe.cpp:126 is the reference's pairwise tree
// over float leaves (detsum.cpp:19-31).  For nonnegative leaves that tree is
// within D*u*S of the exact sum S (D = depth <= 13, u = 2^-53), and any FP64
// summation whose terms nest at most K deep is within K*u*S of S.  The stream
// kernel below sums each bin's leaves in a point-parallel order; if the
// interval [S(1-e), S(1+e)] with e = (K+D+slack)*u rounds to a single float,
// that float IS the reference's bit pattern (rounding is monotone).  Bins that
// fail the test are recomputed with the exact kernel above, so the output is
// bit-identical either way.
// ------------------------------------------------------------------------------

// ------------------------------------------------------------------------------
// Stream path (the production certified kernel): band-streamed, cell-lane.
//
// Per (keypoint, DSP scale) the in-range lattice (bins in (-1, 4) on both
// axes, describe.cpp:84-87) splits into 5 x 5 cells (R, C) = (floor(vbin),
// floor(ubin)).  Every point of cell (R, C) feeds exactly the bins
// (R+ri, C+ci, o0+oi), ri, ci, oi in {0, 1} (describe.cpp:102-124).  The
// lattice is processed in passes of whole cell-rows (<= 30 lattice rows):
//   P1  bilinear samples of the pass rows + guard rows into a 32-row ring
//       (rows shared with the previous pass are kept);
//   P2  lane (cell, part) walks its share of the cell's points: gradient,
//       sqrtf, glibc-exact atan2f, orientation bin, float(exp()) weight, the
//       8 exact float leaves value*wr*wc*wo, each added in FP64 to the lane's
//       private slot [ri][ci][o] in shared memory (no divergence, no atomics);
//   P3  bin-owner threads fold the lane slots of the pass into their FP64 bin
//       sum (fixed lane order), overlapped with the next pass's P1.
// Each bin is then certified as described above (exact-span or
// rounding-interval test against the reference's pairwise tree); keypoints
// with an uncertified bin go to the exact kernel.
// ------------------------------------------------------------------------------
#ifndef DSIFT_P1_TH
#define DSIFT_P1_TH 4
#endif
#ifndef DSIFT_P1_ILP
#define DSIFT_P1_ILP 3
#endif
constexpr int kP1Ilp = DSIFT_P1_ILP;   // interior samples in flight per thread
constexpr int kSRing = 32;                 // sample rows resident (power of two)
constexpr int kSMaxPassRows = kSRing - 2;  // lattice rows per pass (+2 guard rows)
// accumulation lanes: 125 = 5 cells x 25 parts ... 25 cells x 5 parts (tid < 125)
// Lane slots: double slot[lane >> 4][32 entries (ri, ci, o)][lane & 15].  A
// lane's 32 entries all sit in bank pair (lane & 15), so the random-entry
// read-modify-writes of a half-warp never conflict.
// pair (o, ri) of a lane = {ci = 0, ci = 1}, 16 bytes; lanes contiguous per pair
// slot e of lane l at e * 128 + l: a lane's 32 entries share one bank pair
// (l mod 16), so the random-entry read-modify-writes of a half-warp never
// conflict, and consecutive lanes of one entry are consecutive (P3's fold
// walks them with one add per read)
__device__ __forceinline__ int slot_index(int lane, int e) {
    return (((e & 7) * 2 + (e >> 4)) * kDescThreads + lane) * 2 + ((e >> 3) & 1);
}
// Ring row pitch: >= the widest ring row 2*ceil(2.5 bw) + 1 (host: max_span = that
// + 7), and = 16 (mod 32) so two adjacent rows fall in opposite bank halves.
__host__ __device__ __forceinline__ int ring_pitch_for(int max_span) {
    const int need = max_span - 7;
    return need + ((16 - need % 32) + 32) % 32;
}

// floor of 0 <= x < 2^31 on the FP64 pipe: x + 2^52 rounded down is 2^52 +
// floor(x) exactly (unit ulp), its low word is floor(x) and subtracting 2^52
// back gives (double)floor(x) exactly; replaces an F2I + I2F pair on the
// conversion pipe
__device__ __forceinline__ int floor_nonneg(double x, double& fl) {
    const double t = __dadd_rd(x, 0x1p52);
    fl = D_SUB(t, 0x1p52);
    return __double2loint(t);
}

// per-axis weights of lattice index k, one 16-byte load
struct __align__(16) AxisW {
    double e8;      // exp(-(k/bw)^2 / 8): per-axis factor of the window weight
    float g, fr;    // (1 - frac, frac): weight of histogram index floor(bin) + {0, 1}
};

// one 16-byte shared load of an AxisW
__device__ __forceinline__ AxisW ld_axisw(const AxisW* p) {
    const double2 d = *reinterpret_cast<const double2*>(p);
    AxisW w;
    w.e8 = d.x;
    const unsigned long long b = (unsigned long long)__double_as_longlong(d.y);
    w.g = __uint_as_float((unsigned)b);
    w.fr = __uint_as_float((unsigned)(b >> 32));
    return w;
}

// The 2x2 footprint (ix, iy) .. (ix + 1, iy + 1) of one bilinear sample
// (describe.cpp:17-29), 0 <= ix <= w - 2, 0 <= iy <= h - 2, as the stored
// floats bit for bit.  With a texture: one tld4 at unnormalised
// (ix + 1, row0 + iy + 1), whose footprint is texels floor(c - 0.5) and + 1 on
// each axis (c - 0.5 is exact), coordinates formed exactly on the FMA pipe
// (integers < 2^23).  Without: four loads.
__device__ __forceinline__ void gather2x2_tex(cudaTextureObject_t tex, int row0, int ix, int iy, float& v00,
                                              float& v10, float& v01, float& v11) {
    const float xf = F_SUB(__int_as_float(0x4B000000 + ix + 1), 8388608.0f);
    const float yf = F_SUB(__int_as_float(0x4B000000 + row0 + iy + 1), 8388608.0f);
    const float4 g = tex2Dgather<float4>(tex, xf, yf, 0);
    v01 = g.x;   // (ix, iy + 1)
    v11 = g.y;   // (ix + 1, iy + 1)
    v10 = g.z;   // (ix + 1, iy)
    v00 = g.w;   // (ix, iy)
}
__device__ __forceinline__ void gather2x2_ldg(const float* __restrict__ img, int pitch, int ix, int iy, float& v00,
                                              float& v10, float& v01, float& v11) {
    const float* r0 = img + iy * pitch + ix;
    v00 = __ldg(r0);
    v10 = __ldg(r0 + 1);
    v01 = __ldg(r0 + pitch);
    v11 = __ldg(r0 + pitch + 1);
}

struct StreamSmem {
    double2* axy;   // (cx + cos*k, cy + sin*k)   [span] indexed k - kA: one 16-byte load per column
    double2* svc;   // (sin*k, cos*k)                                     and per row
    AxisW* aw;      // [span]
    double* slot;   // [32 entries (ri, ci, o)][128 lanes]
    float* ring;    // [kSRing][ring_pitch] bilinear samples, -1 = undefined
    float* raw;     // [n_dsp][128]
    int* cellmin;   // [2][32]: per pass (double-buffered), per cell: lower bound on the lowest-bit
                    // exponent of the cell's leaves (biased: lowest bit >= 2^(e - 127 - 23))
    const uint32_t* atan_tab;   // atanf's 5-row reduction table (40 words)
    int* misc;      // [2][16]: kmin, kmax, start of cell c = -1..3 (misc[2 + c + 1]);
                    // double-buffered per scale
};

// Biased exponent of x > 0 (floor(log2 x) + 127); denormals map to -22
// (= -149 + 127, their smallest possible value).  For a chain of float
// products leaf = fl(fl(fl(a*b)*c)*d) of positive factors, leaf >= 2^(sum of
// floor(log2)) (rounding is monotone and 2^k is representable), so the leaf's
// lowest bit is >= 2^(sum E - 23).
__device__ __forceinline__ int efield1(float x) {
    const int e = (int)((__float_as_uint(x) >> 23) & 0xffu);
    return e ? e : -22;
}

__device__ __forceinline__ void stream_misc_init(int* misc) {
    const int t = threadIdx.x;
    if (t < 32) misc[t] = ((t & 15) == 1) ? -(1 << 30) : (1 << 30);
}
// Re-arm one misc buffer after its last read.  The buffer is next written two
// scale calls later, with at least one CTA barrier in between.
__device__ __forceinline__ void stream_misc_rearm(int* misc) {
    const int t = threadIdx.x;
    if (t < 16) misc[t] = (t == 1) ? -(1 << 30) : (1 << 30);
}

// Per-(keypoint, DSP scale) scalars (describe.cpp:37-47), formed once per
// keypoint by one thread per scale instead of redundantly by every thread.
struct ScaleSetup {
    double cx, cy, bw;
    int lvl, radius, kA, kB;
};
__device__ __forceinline__ ScaleSetup make_scale_setup(const PyramidDesc& p, const DevKeypoint& kp, double f) {
    ScaleSetup r;
    const double to_input = ldexp(1.0, kp.octave) * (p.upsampled ? 0.5 : 1.0);
    r.cx = kp.x / to_input;
    r.cy = kp.y / to_input;
    const double sigma_rel = kp.sigma / to_input;
    r.lvl = nearest_level_d(p, f * sigma_rel);
    r.bw = 3.0 * f * sigma_rel;
    r.radius = (int)llround(r.bw * (kDescCells + 1) * 0.5 * 1.4142135623730951);
    // table span [kA, kB] contains the in-range span and its guard entries
    const double hb = 2.5 * r.bw;
    r.kA = max(-r.radius - 1, (int)floor(-hb) - 3);
    r.kB = min(r.radius + 1, (int)ceil(hb) + 3);
    return r;
}

__device__ __forceinline__ bool raw_descriptor_stream(const DescArgs& a, const StreamSmem& S, const DevKeypoint& kp,
                                                      const ScaleSetup& ss, double cosa, double sina,
                                                      float* raw_out, int ring_pitch, int* misc) {
    const PyramidDesc& p = a.pyr;
    const OctaveDesc& od = p.oct[kp.octave];
    const double cx = ss.cx, cy = ss.cy, bw = ss.bw;
    const int lvl = ss.lvl, radius = ss.radius, kA = ss.kA, kB = ss.kB;
    const float* __restrict__ img =
        od.gauss + (long long)kp.image * p.gauss_img_stride(kp.octave) + (long long)lvl * od.level_stride;
    const int w = od.w, h = od.h, pitch = od.pitch;
    // this image's level stack as one texture (level lvl from row tex_row0), if the host made one
    const cudaTextureObject_t tex = a.gauss_tex ? a.gauss_tex[kp.image * kMaxOctaves + kp.octave] : 0;
    const int tex_row0 = lvl * (int)(od.level_stride / pitch);   // level_stride = pitch * (rows per level)
    const int tid = threadIdx.x;
    const int span = kB - kA + 1;
    if (span > a.max_span) {   // host sized the tables from the largest sigma; never clip silently
        if (tid == 0) atomicOr(a.err, kErrDescriptorLattice);
        raw_out[tid] = 0.0f;
        __syncthreads();
        return true;
    }
    // ---- per-axis tables (describe.cpp:48-52, 72-73, 84-99 per-axis factors)
    for (int i = tid; i < span; i += kDescThreads) {
        const int k = kA + i;
        DSIFT_BOUND(i < a.max_span, 508);
        const double q = D_DIV((double)k, bw);
        const double bn = D_ADD(q, (double)(kDescCells / 2 - 0.5));
        const int c = (int)floor(bn);
        const float fr = (float)D_SUB(bn, (double)c);
        const float gr = F_SUB(1.0f, fr);
        AxisW w;
        w.e8 = dsift_exp_mid(D_MUL(-D_MUL(q, q), 0.125));
        w.g = gr;
        w.fr = fr;
        S.aw[i] = w;
        S.axy[i] = make_double2(D_ADD(cx, D_MUL(cosa, (double)k)), D_ADD(cy, D_MUL(sina, (double)k)));
        S.svc[i] = make_double2(D_MUL(sina, (double)k), D_MUL(cosa, (double)k));
        if (k >= -radius && k <= radius && bn > -1.0 && bn < (double)kDescCells) {
            atomicMin(&misc[0], k);
            atomicMax(&misc[1], k);
            atomicMin(&misc[2 + (c + 1)], k);
        }
    }
#ifdef DSIFT_NONDET_TEST_HOOK
    if (a.nondet) raw_out[tid] = 0.0f;
#endif
    __syncthreads();
    const int kmin = misc[0], kmax = misc[1];
    if (tid == 0 && a.lattice) atomicAdd(a.lattice, (unsigned long long)(2 * radius + 1) * (2 * radius + 1));
    if (kmin > kmax) {   // no in-range lattice point: an all-zero histogram
        raw_out[tid] = 0.0f;
        __syncthreads();
        stream_misc_rearm(misc);
        return true;
    }
    if (tid == 0 && a.lattice_in) atomicAdd(a.lattice_in, (unsigned long long)(kmax - kmin + 1) * (kmax - kmin + 1));
    int st[6];   // first lattice index of cell c = -1..3 at st[c + 1]; st[5] = kmax + 1
    st[5] = kmax + 1;
#pragma unroll
    for (int c = 4; c >= 0; --c) st[c] = min(misc[2 + c], st[c + 1]);
    int maxnc = 0;
#pragma unroll
    for (int c = 0; c < 5; ++c) maxnc = max(maxnc, st[c + 1] - st[c]);
    // run-time indexed copy in shared memory (misc[8..13] of this scale's
    // buffer): one LDS replaces a 5-deep select chain per lookup
    int* sts = misc + 8;
    if (tid < 6) sts[tid] = st[0] * (tid == 0) + st[1] * (tid == 1) + st[2] * (tid == 2) + st[3] * (tid == 3) +
                            st[4] * (tid == 4) + st[5] * (tid == 5);
    __syncthreads();
    const int ub = kmin - 1;        // lattice index of ring column 0
    const int sw = kmax - kmin + 3; // ring columns in use
    const double wm1 = (double)(w - 1), hm1 = (double)(h - 1);
    const int brow = tid >> 5, bcol = (tid >> 3) & 3, bori = tid & 7;
    // the sample coordinates are monotone in u and in v (each rounding step is),
    // so the lattice's 4 corners bound every sample: if they all lie in
    // [0, w-2] x [0, h-2] no sample is undefined or needs the border clamp
    bool interior = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int u = (q & 1) ? kmax + 1 : kmin - 1, v = (q & 2) ? kmax + 1 : kmin - 1;
        const double2 cu_ = S.axy[u - kA], rv_ = S.svc[v - kA];
        const double px = D_SUB(cu_.x, rv_.x);
        const double py = D_ADD(cu_.y, rv_.y);
        interior = interior && px >= 0.0 && px <= (double)(w - 2) && py >= 0.0 && py <= (double)(h - 2);
    }

    double binacc = 0.0;
    int binlsb = 1 << 20;   // biased exponent of the bin's smallest leaf (lowest bit >= 2^(binlsb - 150))
    int kchain = 0;         // longest in-lane addition chain of any pass
    int npass = 0;
    int pRa = 0, pRb = -1, pP = 1;
    bool pending = false;
    int R = -1, sub = 0, have_hi = kmin - 3;
    while (true) {
        const bool have = R <= 3;
        int Ra = 0, Rb = -1, va = 0, vb = -1, P = 1;
        if (have) {
            const int rows = sts[(R + 2)] - sts[(R + 1)];
            if (sub > 0 || rows > kSMaxPassRows) {   // a cell-row taller than a pass: equal row splits
                const int nsplit = (rows + kSMaxPassRows - 1) / kSMaxPassRows;
                const int chunk = (rows + nsplit - 1) / nsplit;
                va = sts[(R + 1)] + sub * chunk;
                vb = min(va + chunk, sts[(R + 2)]) - 1;
                Ra = Rb = R;
                if (++sub == nsplit) {
                    sub = 0;
                    ++R;
                }
            } else {                                 // whole cell-rows while they fit
                Ra = R;
                int tot = rows;
                ++R;
                while (R <= 3) {
                    const int rr = sts[(R + 2)] - sts[(R + 1)];
                    if (rr > kSMaxPassRows || tot + rr > kSMaxPassRows) break;
                    tot += rr;
                    ++R;
                }
                Rb = R - 1;
                va = sts[(Ra + 1)];
                vb = sts[(Rb + 2)] - 1;
            }
            P = (Rb - Ra + 1) == 1 ? 25 : (Rb - Ra + 1) == 2 ? 12 : (Rb - Ra + 1) == 3 ? 8 : (Rb - Ra + 1) == 4 ? 6 : 5;   // 125 / (5 * cell rows)
            // P1: samples of rows [va-1, vb+1] not yet in the ring (describe.cpp:56-65)
            const int s0 = max(va - 1, have_hi + 1), s1 = vb + 1;
            if (s1 >= s0) {
                // two samples per thread per iteration, branch-free (the loads of
                // both are in flight together); out-of-image samples read a
                // clamped pixel and are replaced by kUndef
                const float inv_sw = 1.0f / (float)sw;   // exact row split for idx < 2^16
                const int ns = (s1 - s0 + 1) * sw;
                if (interior) {   // every lattice sample in [0, w-2] x [0, h-2]: no tests, no clamps
#if DSIFT_P1_TH > 1
                    // warp = TH x TW block of samples: its bilinear footprints
                    // share fewer cache lines than a 32-sample row segment
                    constexpr int TH = DSIFT_P1_TH, TW = 32 / DSIFT_P1_TH;
                    const int tpr = (sw + TW - 1) / TW, nr = s1 - s0 + 1;
                    const float inv_tpr = 1.0f / (float)tpr;
                    const int nsb = ((nr + TH - 1) / TH) * tpr * 32;
#else
                    const int nsb = ns;
#endif
                    for (int idx = tid; idx < nsb; idx += kP1Ilp * kDescThreads) {
                        int ixs[kP1Ilp], iys[kP1Ilp], slot[kP1Ilp];
                        float fx[kP1Ilp], fy[kP1Ilp];
                        bool ok[kP1Ilp];
#pragma unroll
                        for (int j = 0; j < kP1Ilp; ++j) {
#if DSIFT_P1_TH > 1
                            const int id = idx + j * kDescThreads;
                            const int t = id >> 5, l = id & 31;
                            const int tr = (int)(((float)t + 0.5f) * inv_tpr), tc = t - tr * tpr;
                            int rr = tr * TH + l / TW, cc = tc * TW + (l & (TW - 1));
                            ok[j] = id < nsb && rr < nr && cc < sw;
                            rr = min(rr, nr - 1);
                            cc = min(cc, sw - 1);
#else
                            const int id = min(idx + j * kDescThreads, ns - 1);
                            ok[j] = idx + j * kDescThreads < ns;
                            const int rr = (int)(((float)id + 0.5f) * inv_sw), cc = id - rr * sw;
#endif
                            const int vv = s0 + rr, u = ub + cc;
                            const double2 cu_ = S.axy[u - kA], rv_ = S.svc[vv - kA];
                            const double px = D_SUB(cu_.x, rv_.x);
                            const double py = D_ADD(cu_.y, rv_.y);
                            double flx, fly;
                            const int ix = floor_nonneg(px, flx), iy = floor_nonneg(py, fly);
                            fx[j] = (float)D_SUB(px, flx);
                            fy[j] = (float)D_SUB(py, fly);
                            ixs[j] = ix;
                            iys[j] = iy;
                            slot[j] = (vv & (kSRing - 1)) * ring_pitch + cc;
                        }
                        float v00[kP1Ilp], v10[kP1Ilp], v01[kP1Ilp], v11[kP1Ilp];
#ifdef DSIFT_BOUNDS_CHECK
#pragma unroll
                        for (int j = 0; j < kP1Ilp; ++j) {   // no clamp on this path: the corner bound must hold
                            DSIFT_BOUND(ixs[j] >= 0 && ixs[j] <= w - 2 && iys[j] >= 0 && iys[j] <= h - 2, 501);
                            DSIFT_BOUND(!ok[j] || (slot[j] >= 0 && slot[j] < kSRing * ring_pitch), 502);
                        }
#endif
                        if (tex) {   // uniform: the loads of all kP1Ilp samples issue back to back
#pragma unroll
                            for (int j = 0; j < kP1Ilp; ++j)
                                gather2x2_tex(tex, tex_row0, ixs[j], iys[j], v00[j], v10[j], v01[j], v11[j]);
                        } else {
#pragma unroll
                            for (int j = 0; j < kP1Ilp; ++j)
                                gather2x2_ldg(img, pitch, ixs[j], iys[j], v00[j], v10[j], v01[j], v11[j]);
                        }
#pragma unroll
                        for (int j = 0; j < kP1Ilp; ++j) {
                            const float top = F_ADD(v00[j], F_MUL(fx[j], F_SUB(v10[j], v00[j])));
                            const float bot = F_ADD(v01[j], F_MUL(fx[j], F_SUB(v11[j], v01[j])));
                            if (ok[j]) S.ring[slot[j]] = F_ADD(top, F_MUL(fy[j], F_SUB(bot, top)));
                        }
                    }
                } else
                for (int idx = tid; idx < ns; idx += 2 * kDescThreads) {
                    int ixs[2], iys[2], slot[2];
                    float fx[2], fy[2];
                    bool inb[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const int id = min(idx + j * kDescThreads, ns - 1);
                        const int rr = (int)(((float)id + 0.5f) * inv_sw), cc = id - rr * sw;
                        const int vv = s0 + rr, u = ub + cc;
                        const double2 cu_ = S.axy[u - kA], rv_ = S.svc[vv - kA];
                        const double px = D_SUB(cu_.x, rv_.x);
                        const double py = D_ADD(cu_.y, rv_.y);
                        inb[j] = !(px < 0.0 || px > wm1 || py < 0.0 || py > hm1);
                        // sample_bilinear (describe.cpp:17-29); the clamp at 0 only
                        // affects samples that are discarded
                        const int ix = min(max((int)floor(px), 0), w - 2);
                        const int iy = min(max((int)floor(py), 0), h - 2);
                        fx[j] = (float)D_SUB(px, (double)ix);
                        fy[j] = (float)D_SUB(py, (double)iy);
                        ixs[j] = ix;
                        iys[j] = iy;
                        slot[j] = (vv & (kSRing - 1)) * ring_pitch + cc;
                    }
                    float v00[2], v10[2], v01[2], v11[2];
                    if (tex) {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            gather2x2_tex(tex, tex_row0, ixs[j], iys[j], v00[j], v10[j], v01[j], v11[j]);
                    } else
                    {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            gather2x2_ldg(img, pitch, ixs[j], iys[j], v00[j], v10[j], v01[j], v11[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const float top = F_ADD(v00[j], F_MUL(fx[j], F_SUB(v10[j], v00[j])));
                        const float bot = F_ADD(v01[j], F_MUL(fx[j], F_SUB(v11[j], v01[j])));
                        const float sv = F_ADD(top, F_MUL(fy[j], F_SUB(bot, top)));
                        DSIFT_BOUND(idx + j * kDescThreads >= ns || (slot[j] >= 0 && slot[j] < kSRing * ring_pitch), 503);
                        if (idx + j * kDescThreads < ns) S.ring[slot[j]] = inb[j] ? sv : kUndef;
                    }
                }
                have_hi = s1;
            }
        }
        if (pending) {   // P3 of the previous pass: fold the lane slots into this thread's bin
            double se = 0.0, so = 0.0;
            int lm = 1 << 20;
#pragma unroll
            for (int dr = 0; dr < 2; ++dr) {
                const int Rc = brow - 1 + dr;          // ri = 1 - dr
                if (Rc < pRa || Rc > pRb) continue;
#pragma unroll
                for (int dc = 0; dc < 2; ++dc) {
                    const int Cc = bcol - 1 + dc;      // ci = 1 - dc
                    const int cell = (Rc - pRa) * 5 + (Cc + 1);
                    const int e = ((1 - dr) * 2 + (1 - dc)) * 8 + bori;
                    const int l0 = cell * pP;
                    DSIFT_BOUND(cell >= 0 && cell < 25 && l0 + pP <= kDescThreads, 507);
                    // lanes in a rotated (per-orientation) fixed order: the 8
                    // orientations of one cell hit 8 different bank pairs
                    int qq = bori < pP ? bori : bori - pP;   // bori % pP (bori < 8 <= 2 * pP)
                    int q = 0;
                    for (; q + 1 < pP; q += 2) {
                        const int qa = qq, qb = (qq + 1 == pP) ? 0 : qq + 1;
                        qq = (qb + 1 == pP) ? 0 : qb + 1;
                        se = se + S.slot[slot_index(l0 + qa, e)];
                        so = so + S.slot[slot_index(l0 + qb, e)];
                    }
                    if (q < pP) se = se + S.slot[slot_index(l0 + qq, e)];
                    lm = min(lm, S.cellmin[((npass - 1) & 1) * 32 + cell]);
                }
            }
            binacc = binacc + (se + so);
            binlsb = min(binlsb, lm);
        }
        __syncthreads();
        if (!have) break;
        // P2: lane (cell, part) over its share of the cell's points
        {
            const int ncells = (Rb - Ra + 1) * 5;
            const int cell = (int)(((float)tid + 0.5f) * (1.0f / (float)P)), part = tid - cell * P;   // tid / P (exact)
            int npts = 0, nc = 1, rv0 = 0, cu0 = 0;
            if (cell < ncells) {
                const int Rl = Ra + cell / 5, Cl = cell % 5 - 1;
                const int r0 = max(va, sts[(Rl + 1)]), r1 = min(vb, sts[(Rl + 2)] - 1);
                cu0 = sts[(Cl + 1)];
                nc = sts[(Cl + 2)] - cu0;
                rv0 = r0;
                if (r1 >= r0 && nc > 0) npts = (r1 - r0 + 1) * nc;
            }
            if (tid < 32) S.cellmin[((npass + 1) & 1) * 32 + tid] = 1 << 20;   // next pass's buffer (read two passes ago)
            double2* myv = reinterpret_cast<double2*>(S.slot) + tid;
#pragma unroll
            for (int e = 0; e < 16; ++e) myv[e * kDescThreads] = make_double2(0.0, 0.0);
            int lmin = 1 << 20;
            bool nan_seen = false;
            // point pi = part + j*P of the cell in row-major order: (rr, cc),
            // advanced incrementally (dq rows + dr columns per step)
            const int ncs = max(nc, 1);
            const float inv_ncs = 1.0f / (float)ncs;   // exact quotients for operands < 2^10
            int rr = (int)(((float)part + 0.5f) * inv_ncs), cc = part - rr * ncs;
            const int dq = (int)(((float)P + 0.5f) * inv_ncs), dr = P - dq * ncs;
            for (int pi = part; pi < npts; pi += P) {
                const int v = rv0 + rr, u = cu0 + cc;
                cc += dr;
                rr += dq;
                const int wrapc = cc >= ncs;   // branch-free carry
                cc -= wrapc * ncs;
                rr += wrapc;
                const int col = u - ub;
                DSIFT_BOUND(col >= 1 && col + 1 < ring_pitch && col + 1 < sw, 504);
                DSIFT_BOUND(u - kA >= 0 && u - kA < span && v - kA >= 0 && v - kA < span, 505);
                DSIFT_BOUND(v - 1 >= have_hi - (kSRing - 1) && v + 1 <= have_hi, 506);   // rows resident in the ring
                const float* mid = S.ring + (v & (kSRing - 1)) * ring_pitch + col;
                const float left = mid[-1], right = mid[1];
                const float up = S.ring[((v - 1) & (kSRing - 1)) * ring_pitch + col];
                const float down = S.ring[((v + 1) & (kSRing - 1)) * ring_pitch + col];
                if (!interior && (left == kUndef || right == kUndef || up == kUndef || down == kUndef)) continue;
                // the lanes at this point of the iteration: both votes below are
                // reached by exactly these (nothing between them diverges)
                const unsigned am = __activemask();
                // describe.cpp:89-100
                const float du = F_MUL(0.5f, F_SUB(right, left));
                const float dv = F_MUL(0.5f, F_SUB(down, up));
                const float mag = F_SQRT(F_ADD(F_MUL(du, du), F_MUL(dv, dv)));
                float theta = dsift_atan2f_mask(dv, du, am, S.atan_tab);
                theta = (theta < 0.0f) ? F_ADD(theta, (float)kTwoPi) : theta;
                nan_seen |= isnan(theta);   // reference: negative bin -> std::out_of_range (reported after the loop)
                theta = isnan(theta) ? 0.0f : theta;
                double obin = ds_div_2pi((double)F_MUL(theta, (float)kDescOrients));
                const double obw = D_SUB(obin, (double)kDescOrients);
                obin = (obin >= (double)kDescOrients) ? obw : obin;
                const AxisW wu = ld_axisw(S.aw + (u - kA)), wv = ld_axisw(S.aw + (v - kA));
                // window weight float(exp(-(uu^2 + vv^2) / 8)) (describe.cpp:96-98) as the
                // product of the two per-axis factors, proven to round to the same
                // float; otherwise (~1e-8 of points) evaluated as the reference does
                float wgt;
                const bool wok = ds_separable_weight<47>(D_MUL(wu.e8, wv.e8), wgt);
                // warp-uniform fallback (~1e-8 of points): the reference's own
                // evaluation equals the certified product wherever that is proven,
                // so a warp with any unproven lane takes it for all of its lanes
                if (__any_sync(am, !wok)) {
                    const double qu = D_DIV((double)u, bw), qv = D_DIV((double)v, bw);
                    wgt = (float)dsift_exp_mid(D_MUL(-D_ADD(D_MUL(qu, qu), D_MUL(qv, qv)), 0.125));
                }
                const float val = F_MUL(mag, wgt);
                double flo;
                const int o0 = floor_nonneg(obin, flo);
                const float fo = (float)D_SUB(obin, flo);
                const float go = F_SUB(1.0f, fo);
                // leaves value*wr*wc*wo (describe.cpp:102-124), FP64 slot accumulation
                const float a0 = F_MUL(val, wv.g), a1 = F_MUL(val, wv.fr);
                const float t00 = F_MUL(a0, wu.g), t01 = F_MUL(a0, wu.fr);
                const float t10 = F_MUL(a1, wu.g), t11 = F_MUL(a1, wu.fr);
                // 8 leaves = 4 pairs {ci = 0, 1}: (o0, ri 0), (o0, ri 1), (o0+1, ri 0), (o0+1, ri 1)
                double2* pa = myv + ((o0 & 7) * 2) * kDescThreads;
                double2* pb = myv + (((o0 + 1) & 7) * 2) * kDescThreads;
                double2 x0 = pa[0], x1 = pa[kDescThreads], x2 = pb[0], x3 = pb[kDescThreads];
                x0.x = x0.x + (double)F_MUL(t00, go);
                x0.y = x0.y + (double)F_MUL(t01, go);
                x1.x = x1.x + (double)F_MUL(t10, go);
                x1.y = x1.y + (double)F_MUL(t11, go);
                x2.x = x2.x + (double)F_MUL(t00, fo);
                x2.y = x2.y + (double)F_MUL(t01, fo);
                x3.x = x3.x + (double)F_MUL(t10, fo);
                x3.y = x3.y + (double)F_MUL(t11, fo);
                pa[0] = x0;
                pa[kDescThreads] = x1;
                pb[0] = x2;
                pb[kDescThreads] = x3;
                {
                    // the lane's smallest leaf: leaves are RN(t * wo), monotone in t and
                    // wo, so it is RN(min t * min nonzero wo); its exponent bounds every
                    // leaf's lowest bit (a zero t, from an exactly-integral spatial bin,
                    // only makes the bound pessimistic); points with value 0 add nothing
                    const float tmin = fminf(fminf(t00, t01), fminf(t10, t11));
                    const float mo = fo > 0.0f ? fminf(fo, go) : go;
                    const int ef = efield1(F_MUL(tmin, mo));
                    lmin = (val > 0.0f) ? min(lmin, ef) : lmin;
                }
            }
            if (nan_seen) atomicOr(a.err, kErrHistogramRange);
            if (cell < ncells && lmin < (1 << 20)) atomicMin(&S.cellmin[(npass & 1) * 32 + cell], lmin);
#ifdef DSIFT_NONDET_TEST_HOOK
            if (a.nondet && cell < ncells) {   // order-fragile: float atomics in scheduling order
                const int Rl = Ra + cell / 5, Cl = cell % 5 - 1;
                for (int e = 0; e < 32; ++e) {
                    const int row = Rl + (e >> 4), col = Cl + ((e >> 3) & 1);
                    const double sv = S.slot[slot_index(tid, e)];
                    if (row >= 0 && row < kDescCells && col >= 0 && col < kDescCells && sv != 0.0)
                        atomicAdd(&raw_out[(row * kDescCells + col) * kDescOrients + (e & 7)], (float)sv);
                }
            }
#endif
        }
        kchain = max(kchain, (int)((float)((vb - va + 1) * maxnc) * (1.0f / (float)P)) + 1);   // >= ceil(./P): a bound
        ++npass;
        __syncthreads();
        pending = true;
        pRa = Ra;
        pRb = Rb;
        pP = P;
    }
    stream_misc_rearm(misc);   // every thread read misc before the pass barriers
    if (tid < 32) S.cellmin[((npass - 1) & 1) * 32 + tid] = 1 << 20;   // folded before the last barrier
    // certificate (see above): chain <= kchain in a lane slot, <= 51 in
    // the fold, <= npass across passes; the reference tree is <= tree_depth deep
    bool ok;
    float res;
    const int top = (int)((__double_as_longlong(binacc) >> 52) & 0x7ff) - 1023;
    if (binacc == 0.0 || top - (binlsb - 127 - 23) <= 52) {
        ok = true;
        res = __double2float_rn(binacc);
    } else {
        const double e = (double)(kchain + npass + 51 + a.tree_depth + 64) * 0x1p-53;
        const double lo = binacc * (1.0 - e), hi = binacc * (1.0 + e);
        const float flo = __double2float_rn(lo), fhi = __double2float_rn(hi);
        ok = (flo == fhi);
        res = flo;
    }
#ifdef DSIFT_NONDET_TEST_HOOK
    if (a.nondet) {
        __syncthreads();
        return true;   // raw_out holds the atomically accumulated histogram
    }
#endif
    raw_out[tid] = res;
    return ok && !a.force_slow;
}

__global__ void __launch_bounds__(kDescThreads, 4)
describe_stream_kernel(const __grid_constant__ DescArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[4];
    __shared__ int misc[32];
    __shared__ int cellmin[64];
    __shared__ ScaleSetup sscale[kMaxDsp];
    __shared__ __align__(16) uint32_t atan_tab[40];
    if (threadIdx.x < 40) atan_tab[threadIdx.x] = DS_ATAN_ROW_D[threadIdx.x];
    const int SP = a.max_span;
    const int RP = ring_pitch_for(SP);
    StreamSmem S;
    unsigned char* pbuf = sm;
    S.raw = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * kDescDim * a.n_dsp;
    S.axy = reinterpret_cast<double2*>(pbuf); pbuf += sizeof(double2) * SP;
    S.svc = reinterpret_cast<double2*>(pbuf); pbuf += sizeof(double2) * SP;
    S.aw = reinterpret_cast<AxisW*>(pbuf); pbuf += sizeof(AxisW) * SP;
    S.slot = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * 32 * kDescThreads;
    S.ring = reinterpret_cast<float*>(pbuf);
    S.cellmin = cellmin;
    S.misc = misc;
    S.atan_tab = atan_tab;
    stream_misc_init(misc);
    if (threadIdx.x < 64) cellmin[threadIdx.x] = 1 << 20;
    __syncthreads();

    const long long n = a.n_host >= 0 ? a.n_host : (long long)*a.n_dev;
    const int tid = threadIdx.x;
    int call = 0;
    // keypoints are claimed one at a time from a global ticket: a keypoint
    // costs up to ~16x another (its DSP lattices scale with sigma^2), so a
    // static stride would leave the slowest CTA ~10% behind the mean
    __shared__ unsigned s_k;
    for (;;) {
        __syncthreads();                   // everyone is done with the previous s_k
        if (tid == 0) s_k = atomicAdd(a.ticket, 1u);
        __syncthreads();
        if ((long long)s_k >= n) break;
        // claimed in reverse canonical order: octaves and intervals descending,
        // so the last claims are the cheapest keypoints (small sigma) and the
        // CTAs finish together (longest-first, approximately)
        const long long k = n - 1 - (long long)s_k;
        const DevKeypoint kp = a.kps[k];
        const double2 cs = a.trig[k];
        if (tid < a.n_dsp) sscale[tid] = make_scale_setup(a.pyr, kp, a.dsp[tid]);
        __syncthreads();
        bool all_ok = true;
        for (int fi = 0; fi < a.n_dsp; ++fi, ++call) {
            const bool ok = raw_descriptor_stream(a, S, kp, sscale[fi], cs.x, cs.y, S.raw + fi * kDescDim, RP,
                                                  misc + 16 * (call & 1));
            const bool sok = __syncthreads_and(ok);
            if (!sok && !a.force_slow) {
                // a bin the certificate could not prove: recompute this scale with
                // the exact scan-order trees, in place (the stream working set is
                // dead; the exact working set aliases it, raw[] is kept)
                const DescSmem E = carve_exact_smem(sm, a, a.n_dsp);
                raw_descriptor_cta(a, E, kp, a.dsp[fi], cs.x, cs.y, S.raw + fi * kDescDim);
                if (tid == 0 && a.fix_count) atomicAdd(a.fix_count, 1u);
            } else {
                all_ok &= sok;
            }
        }
        if (!all_ok) {
            if (tid == 0) {
                const unsigned slot = atomicAdd(a.slow_count, 1u);
                if ((long long)slot < a.slow_cap) a.slow_out[slot] = (int)k;
                else atomicOr(a.err, kErrDescriptorLattice);
            }
            continue;   // the exact kernel writes this keypoint's descriptor
        }
        dsp_epilogue(a, S.raw, k, red);
        __syncthreads();
    }
}

size_t describe_stream_exact_smem_bytes(int max_axis, int chunk_rows, int n_dsp, int tree_depth) {
    // carve_exact_smem: raw + working set (+16 alignment slack)
    const size_t A = (size_t)max_axis;
    const size_t PW = ((A + 31) / 32) * 32, NW = PW / 32;
    return sizeof(float) * kDescDim * n_dsp + sizeof(double) * 6 * A + sizeof(float) * A + sizeof(int) * A +
           sizeof(float) * (chunk_rows + 2) * A + sizeof(float) * 2 * chunk_rows * PW +
           sizeof(unsigned) * chunk_rows * kDescOrients * NW + 16 + sizeof(double) * (tree_depth - 3) * kDescThreads +
           sizeof(float) * kRing * kDescThreads;
}

size_t describe_stream_smem_bytes(int max_span, int n_dsp) {
    const size_t SP = (size_t)max_span, RP = (size_t)ring_pitch_for(max_span);
    return sizeof(float) * kDescDim * n_dsp + sizeof(double) * 4 * SP + sizeof(AxisW) * SP +
           sizeof(double) * 32 * kDescThreads + sizeof(float) * kSRing * RP;
}

int describe_stream_blocks_per_sm(size_t smem) {
    cudaFuncSetAttribute(describe_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, describe_stream_kernel, kDescThreads, smem) != cudaSuccess)
        n = 1;
    return n;
}

cudaError_t launch_describe_stream(const DescArgs& a, int grid, cudaStream_t st) {
    const size_t smem = describe_stream_smem_bytes(a.max_span, a.n_dsp);
    cudaError_t e = cudaFuncSetAttribute(describe_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    describe_stream_kernel<<<grid, kDescThreads, smem, st>>>(a);
    return cudaGetLastError();
}

size_t describe_smem_bytes(int max_axis, int chunk_rows, int n_dsp, int tree_depth) {
    const size_t A = (size_t)max_axis;
    const size_t PW = ((A + 31) / 32) * 32, NW = PW / 32;
    return sizeof(double) * 6 * A + sizeof(float) * A + sizeof(int) * A + sizeof(float) * kDescDim * n_dsp +
           sizeof(float) * (chunk_rows + 2) * A + sizeof(float) * 2 * chunk_rows * PW +
           sizeof(unsigned) * chunk_rows * kDescOrients * NW + 16 + sizeof(double) * (tree_depth - 3) * kDescThreads +
           sizeof(float) * kRing * kDescThreads;
}

// cos/sin of every keypoint angle (describe.cpp:51-52), once per keypoint.
__global__ void trig_kernel(const DevKeypoint* __restrict__ kps, const unsigned long long* n_dev, long long n_host,
                            double2* __restrict__ trig) {
    const long long n = n_host >= 0 ? n_host : (long long)*n_dev;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        double sn, cs;
        dsift_sincos((double)kps[k].angle, &sn, &cs);
        trig[k] = make_double2(cs, sn);
    }
}

cudaError_t launch_trig(const DevKeypoint* kps, const unsigned long long* n_dev, long long n_host, double2* trig,
                        long long cap, cudaStream_t st) {
    const long long n = n_host >= 0 ? n_host : cap;
    const int grid = (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
    trig_kernel<<<grid, 256, 0, st>>>(kps, n_dev, n_host, trig);
    return cudaGetLastError();
}

cudaError_t launch_describe(const DescArgs& a, int grid, cudaStream_t st) {
    const size_t smem = describe_smem_bytes(a.max_axis, a.chunk_rows, a.raw_mode ? 1 : a.n_dsp, a.tree_depth);
    cudaError_t e = cudaFuncSetAttribute(describe_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    describe_exact_kernel<<<grid, kDescThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace dsift
