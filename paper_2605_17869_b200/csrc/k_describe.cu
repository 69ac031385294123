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

constexpr int kDescThreads = 128;
constexpr int kTreeDepth = 16;   // per-bin leaves < 65536 (checked on the host)
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
    float* samp;    // [(chunk+2)][width+2]
    float* pval;    // [chunk][width]
    float* pfo;
    unsigned char* po0;
    float* raw;     // [n_dsp][128]
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

__device__ void raw_descriptor_cta(const DescArgs& a, const DescSmem& S, const DevKeypoint& kp,
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
    const int tid = threadIdx.x;
    if (2 * radius + 3 > a.max_axis) {   // host sized the tables for r_max; never silently clip
        if (tid == 0) atomicOr(a.err, kErrDescriptorLattice);
        raw_out[tid] = 0.0f;
        __syncthreads();
        return;
    }
    const int kbase = -radius - 1;
    const int naxis = 2 * radius + 3;

    // 1. per-axis tables
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
    // bin owned by this thread: (row, col, ori)
    const int brow = tid >> 5, bcol = (tid >> 3) & 3, bori = tid & 7;
    // u / v ranges of this bin's 2x2-cell rectangle: c0 in {b-1, b}
    int ua = 1 << 30, ub = -(1 << 30), va = 1 << 30, vb = -(1 << 30);
    for (int k = kmin; k <= kmax; ++k) {
        const int c = S.c0[k - kbase];
        if (c == bcol - 1 || c == bcol) { ua = min(ua, k); ub = max(ub, k); }
        if (c == brow - 1 || c == brow) { va = min(va, k); vb = max(vb, k); }
    }
    TreeCounter<kTreeDepth> tc;
    tc.reset();

    const int ch = a.chunk_rows;
    for (int v0 = kmin; v0 <= kmax; v0 += ch) {
        const int v1 = min(v0 + ch - 1, kmax);
        const int nrows = v1 - v0 + 1;
        // 2a. samples on rows [v0-1, v1+1] x cols [kmin-1, kmax+1]
        for (int idx = tid; idx < (nrows + 2) * swidth; idx += kDescThreads) {
            const int rr = idx / swidth, cc = idx % swidth;
            const int v = v0 - 1 + rr, u = kmin - 1 + cc;
            const double px = D_SUB(S.ax[u - kbase], S.sv[v - kbase]);
            const double py = D_ADD(S.cy_su[u - kbase], S.cv[v - kbase]);
            float sv = kUndef;
            if (!(px < 0.0 || px > (double)(w - 1) || py < 0.0 || py > (double)(h - 1)))
                sv = sample_bilinear(img, w, h, pitch, px, py);
            S.samp[idx] = sv;
        }
        __syncthreads();
        // 2b. per-point gradient, orientation, weight
        for (int idx = tid; idx < nrows * width; idx += kDescThreads) {
            const int rr = idx / width, cc = idx % width;
            const int v = v0 + rr, u = kmin + cc;
            const float* sr = S.samp + (rr + 1) * swidth + (cc + 1);
            const float left = sr[-1], right = sr[1], up = sr[-swidth], down = sr[swidth];
            unsigned char o0 = 0xff;
            float value = 0.0f, fo = 0.0f;
            if (!(left == kUndef || right == kUndef || up == kUndef || down == kUndef)) {
                const float du = F_MUL(0.5f, F_SUB(right, left));
                const float dv = F_MUL(0.5f, F_SUB(down, up));
                const float mag = F_SQRT(F_ADD(F_MUL(du, du), F_MUL(dv, dv)));
                float theta = dsift_atan2f(dv, du);
                if (theta < 0.0f) theta = F_ADD(theta, (float)kTwoPi);
                double obin = D_DIV((double)F_MUL(theta, (float)kDescOrients), kTwoPi);
                if (obin >= (double)kDescOrients) obin = D_SUB(obin, (double)kDescOrients);
                const double arg = D_DIV(-D_ADD(S.q2[u - kbase], S.q2[v - kbase]), 8.0);
                const float wgt = (float)dsift_exp(arg);
                value = F_MUL(mag, wgt);
                const int o = (int)floor(obin);
                fo = (float)D_SUB(obin, (double)o);
                o0 = (unsigned char)o;
            }
            S.pval[idx] = value;
            S.pfo[idx] = fo;
            S.po0[idx] = o0;
        }
        __syncthreads();
        // 3. bin-owner accumulation in scan order (describe.cpp:102-126)
        const int ra = max(va, v0), rb = min(vb, v1);
        for (int v = ra; v <= rb; ++v) {
            const int r0 = S.c0[v - kbase];
            const float fr = S.frac[v - kbase];
            const float wr = (brow - r0) ? fr : F_SUB(1.0f, fr);
            const int rowoff = (v - v0) * width - kmin;
            for (int u = ua; u <= ub; ++u) {
                const int o0 = S.po0[rowoff + u];
                if (o0 == 0xff) continue;
                const int oi = (bori - o0) & (kDescOrients - 1);
                if (oi > 1) continue;
                const int c0 = S.c0[u - kbase];
                const float fc = S.frac[u - kbase];
                const float wc = (bcol - c0) ? fc : F_SUB(1.0f, fc);
                const float fo = S.pfo[rowoff + u];
                const float wo = oi ? fo : F_SUB(1.0f, fo);
                const float val = F_MUL(F_MUL(F_MUL(S.pval[rowoff + u], wr), wc), wo);
                tc.push((double)val);
            }
        }
        __syncthreads();
    }
    raw_out[tid] = (float)tc.result();
    __syncthreads();
}

__global__ void __launch_bounds__(kDescThreads)
describe_kernel(const __grid_constant__ DescArgs a) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double red[4];
    __shared__ double trig[2];
    const int A = a.max_axis;
    DescSmem S;
    unsigned char* pbuf = sm;
    S.q2 = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.bin = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.ax = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.cy_su = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.sv = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.cv = reinterpret_cast<double*>(pbuf); pbuf += sizeof(double) * A;
    S.frac = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * A;
    S.c0 = reinterpret_cast<int*>(pbuf); pbuf += sizeof(int) * A;
    S.raw = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * kDescDim * (a.raw_mode ? 1 : a.n_dsp);
    S.samp = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * (a.chunk_rows + 2) * A;
    S.pval = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * a.chunk_rows * A;
    S.pfo = reinterpret_cast<float*>(pbuf); pbuf += sizeof(float) * a.chunk_rows * A;
    S.po0 = pbuf;

    const long long n = a.n_host >= 0 ? a.n_host : (long long)*a.n_dev;
    const int tid = threadIdx.x;
    for (long long k = blockIdx.x; k < n; k += gridDim.x) {
        const DevKeypoint kp = a.kps[k];
        if (tid == 0) {
            double sn, cs;
            dsift_sincos((double)kp.angle, &sn, &cs);
            trig[0] = cs;
            trig[1] = sn;
        }
        __syncthreads();
        const double cosa = trig[0], sina = trig[1];
        if (a.raw_mode) {
            raw_descriptor_cta(a, S, kp, a.raw_scale, cosa, sina, S.raw);
            a.desc[k * kDescDim + tid] = S.raw[tid];
            __syncthreads();
            continue;
        }
        for (int fi = 0; fi < a.n_dsp; ++fi)
            raw_descriptor_cta(a, S, kp, a.dsp[fi], cosa, sina, S.raw + fi * kDescDim);
        // DSP mean: tree over scales / (float)n (describe.cpp:153-162)
        TreeCounter<kTreeDepth> tc;
        tc.reset();
        for (int fi = 0; fi < a.n_dsp; ++fi) tc.push((double)S.raw[fi * kDescDim + tid]);
        float d = F_DIV((float)tc.result(), (float)a.n_dsp);
        // L2 -> clip -> L2 -> RootSIFT (describe.cpp:138-173)
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
        __syncthreads();
    }
}

size_t describe_smem_bytes(int max_axis, int chunk_rows, int n_dsp) {
    const size_t A = (size_t)max_axis;
    return sizeof(double) * 6 * A + sizeof(float) * A + sizeof(int) * A + sizeof(float) * kDescDim * n_dsp +
           sizeof(float) * (chunk_rows + 2) * A + sizeof(float) * 2 * chunk_rows * A + chunk_rows * A + 16;
}

int describe_blocks_per_sm(size_t smem) {
    cudaFuncSetAttribute(describe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, describe_kernel, kDescThreads, smem) != cudaSuccess) n = 1;
    return n;
}

cudaError_t launch_describe(const DescArgs& a, int grid, cudaStream_t st) {
    const size_t smem = describe_smem_bytes(a.max_axis, a.chunk_rows, a.raw_mode ? 1 : a.n_dsp);
    cudaError_t e = cudaFuncSetAttribute(describe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    describe_kernel<<<grid, kDescThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace dsift
