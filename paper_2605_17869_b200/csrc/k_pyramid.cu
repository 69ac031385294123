// k_pyramid.cu — K1: Gaussian scale space + DoG (reference:
// scalespace.cpp:52-111 convolve_separable, :113-131 upsample2x,
// :133-142 decimate2x, :144-214 build_scale_space).
//
// One launch produces one Gaussian level for every image of the batch
// (grid.z = image) and, in the same pass, the DoG level below it
// (DoG[i-1] = G[i] - G[i-1], scalespace.cpp:204-211): the previous level is
// already staged in shared memory as the blur input, so each level is read
// once and G/DoG are each written once.
//
// Tile: 64 x 64 outputs, 256 threads.  The (64+2R)^2 input tile is staged in
// shared memory with reflect-101 indexing (multi-bounce, scalespace.cpp:41-48),
// the horizontal pass writes a float-rounded (64+2R) x 64 temporary to shared
// memory, the vertical pass produces the outputs.  Every output is
// Sum_t k[t] * x[t] accumulated left-to-right in FP64 and rounded to float
// once, exactly as the reference; the products of two binary32 values are
// exact in binary64, so each step is one DFMA (bit-identical to mul+add).
// Each thread computes 4 adjacent outputs from a sliding register window so a
// staged value is converted to double once and feeds 4 DFMAs.
//
// Modes (where the loader gets level-0 input from):
//   LEVEL     G[i-1] of the same octave                       (incremental blur)
//   RAW       the input image, no upsampling                  (bridge blur)
//   UPSAMPLE  2x bilinear upsample of the input on the fly    (bridge blur)
//   DECIMATE  even samples of G[s] of the previous octave; the kernel also
//             writes those samples as this octave's G[0]      (seed + first blur)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"

namespace dsift {

constexpr int kTileW = 64;
constexpr int kTileH = 64;
constexpr int kBlurThreads = 256;

__device__ __forceinline__ int reflect101(int p, int n) {
    if (n == 1) return 0;
    while (p < 0 || p >= n) {
        if (p < 0) p = -p;
        if (p >= n) p = 2 * n - 2 - p;
    }
    return p;
}

template <int MODE>
__device__ __forceinline__ float fetch_input(const BlurArgs& a, const float* __restrict__ src,
                                             int gx, int gy) {
    if (MODE == kModeUpsample) {
        // upsample2x (scalespace.cpp:113-131): 0.25 * (((a + b) + c) + d) in double
        const int y0 = gy >> 1, x0 = gx >> 1;
        const int y1 = (gy & 1) ? min(y0 + 1, a.src_h - 1) : y0;
        const int x1 = (gx & 1) ? min(x0 + 1, a.src_w - 1) : x0;
        const float* r0 = src + (long long)y0 * a.src_pitch;
        const float* r1 = src + (long long)y1 * a.src_pitch;
        const double s = (((double)__ldg(r0 + x0) + (double)__ldg(r0 + x1)) + (double)__ldg(r1 + x0)) +
                         (double)__ldg(r1 + x1);
        return (float)(0.25 * s);
    } else if (MODE == kModeDecimate) {
        return __ldg(src + (long long)(2 * gy) * a.src_pitch + 2 * gx);
    } else {
        return __ldg(src + (long long)gy * a.src_pitch + gx);
    }
}

// Generic-radius path (16 < R <= kMaxRadius, configs with a large sigma0);
// same arithmetic as the tiled kernel below, runtime taps.
template <int MODE>
__global__ void __launch_bounds__(kBlurThreads)
blur_level_kernel_any(const __grid_constant__ BlurArgs a, int R) {
    const int kLen = 2 * R + 1, kInH = kTileH + 2 * R, kInW = kTileW + 2 * R;
    const int kInPitch = (kInW + 3) & ~3;
    extern __shared__ __align__(16) float smem[];
    float* in_s = smem;
    float* tmp_s = smem + kInH * kInPitch;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kTileW, y0 = blockIdx.y * kTileH;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float* __restrict__ src = a.src + b * a.src_img_stride;
    for (int r = warp; r < kInH; r += kBlurThreads / 32) {
        const int gy = reflect101(y0 - R + r, a.h);
        for (int c = lane; c < kInW; c += 32)
            in_s[r * kInPitch + c] = fetch_input<MODE>(a, src, reflect101(x0 - R + c, a.w), gy);
    }
    __syncthreads();
    for (int item = tid; item < kInH * kTileW; item += kBlurThreads) {
        const int r = item / kTileW, c = item % kTileW;
        double acc = 0.0;
        for (int t = 0; t < kLen; ++t) acc = __fma_rn(a.taps[t], (double)in_s[r * kInPitch + c + t], acc);
        tmp_s[r * kTileW + c] = (float)acc;
    }
    __syncthreads();
    float* __restrict__ dst = a.dst + b * a.dst_img_stride;
    float* __restrict__ dog = a.dog ? a.dog + b * a.dog_img_stride : nullptr;
    float* __restrict__ seed = (MODE == kModeDecimate) ? a.seed + b * a.seed_img_stride : nullptr;
    for (int item = tid; item < kTileW * kTileH; item += kBlurThreads) {
        const int c = item % kTileW, r = item / kTileW;
        const int x = x0 + c, y = y0 + r;
        double acc = 0.0;
        for (int t = 0; t < kLen; ++t) acc = __fma_rn(a.taps[t], (double)tmp_s[(r + t) * kTileW + c], acc);
        if (x < a.w && y < a.h) {
            const float g = (float)acc;
            const long long o = (long long)y * a.pitch + x;
            dst[o] = g;
            if (MODE == kModeLevel || MODE == kModeDecimate) {
                const float prev = in_s[(r + R) * kInPitch + c + R];
                if (MODE == kModeDecimate) seed[o] = prev;
                if (dog) dog[o] = g - prev;
            }
        }
    }
}

static size_t blur_smem_bytes(int R) {
    const int in_h = kTileH + 2 * R, in_w = kTileW + 2 * R;
    const int in_pitch = (in_w + 3) & ~3;
    return sizeof(float) * (size_t)(in_h * in_pitch + in_h * kTileW);
}

template <int MODE>
static cudaError_t launch_any(const BlurArgs& a, int R, int batch, cudaStream_t st) {
    const dim3 grid((a.w + kTileW - 1) / kTileW, (a.h + kTileH - 1) / kTileH, batch);
    const size_t smem = blur_smem_bytes(R);
    cudaError_t e = cudaFuncSetAttribute(blur_level_kernel_any<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    blur_level_kernel_any<MODE><<<grid, kBlurThreads, smem, st>>>(a, R);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// LEVEL-mode blur, v2 (the 5 incremental levels of every octave).
//
// The FP64 tap sums and the f32->f64 conversions (XU pipe, 1/4 of the FP64
// rate) bound this stage, not HBM.  v2 therefore
//   * stages the (64+2R)^2 input tile with 16-byte coalesced loads (interior
//     tiles; border tiles use reflect-101 per element), 16-byte aligned so the
//     H pass can read its window with LDS.128;
//   * computes 8 outputs per thread in both passes: each staged value is
//     converted to FP64 once per 8-output window (v1: per 4) and feeds 8
//     independent DFMA chains.
// Each output is still Sum_t k[t] * x[t] accumulated left to right in FP64
// and rounded to float once per pass (scalespace.cpp:63-109).
// ---------------------------------------------------------------------------
constexpr int kB2W = 64, kB2H = 64, kB2Seg = 8, kB2Threads = 256;

template <int R>
struct B2Geom {
    static constexpr int kLen = 2 * R + 1;
    static constexpr int kWin = kB2Seg + 2 * R;                 // inputs per 8 outputs
    static constexpr int kHR = kB2H + 2 * R;                    // input / tmp rows
    static constexpr int kM = (4 - (R & 3)) & 3;                // (x - R) mod 4 for x = 0 mod 8
    static constexpr int kNV = (kWin + kM + 3) / 4;             // float4 per window
    static constexpr int kInW = ((kB2W + 2 * R + kM + 3) / 4) * 4;
    static constexpr int kInPitch = kInW + 4;                   // floats; +4 spreads LDS.128 rows over banks
    static constexpr int kTmpPitch = kB2W + 1;
    static constexpr int kItems = (kHR * (kB2W / kB2Seg) + kB2Threads - 1) / kB2Threads;   // H items per thread
    // the float tmp overwrites the staged input once the H pass has read it
    static constexpr size_t kSmem = sizeof(float) * (size_t)kHR * (kInPitch > kTmpPitch ? kInPitch : kTmpPitch);
};

// float -> double for a positive normal float, on the integer pipe: the
// exponent is rebiased (+896) and the mantissa shifted into place.  Exact for
// exactly those inputs; the XU conversion (a quarter of the FP64 rate) is the
// stage's co-bottleneck otherwise.
__device__ __forceinline__ double widen_pos_normal(float x) {
    const unsigned b = __float_as_uint(x);
    return __hiloint2double((int)((b >> 3) + 0x38000000u), (int)(b << 29));
}

template <int R, bool kAlu>
__device__ __forceinline__ double b2_widen(float x) {
    if (kAlu) return widen_pos_normal(x);
    return (double)x;
}

// H pass of one tile: results stay in registers until every thread has read
// the staged input, then overwrite it as the float tmp.
template <int R, bool kAlu>
__device__ __forceinline__ void b2_hpass(const BlurArgs& a, float* sm) {
    using G = B2Geom<R>;
    float hres[G::kItems][kB2Seg];
#pragma unroll
    for (int it = 0; it < G::kItems; ++it) {
        const int item = threadIdx.x + it * kB2Threads;
        if (item < G::kHR * (kB2W / kB2Seg)) {
            const int r = item >> 3, sg = item & 7;
            const float4* v4 = reinterpret_cast<const float4*>(sm + r * G::kInPitch + sg * kB2Seg);
            float win[4 * G::kNV];
#pragma unroll
            for (int q = 0; q < G::kNV; ++q) {
                const float4 t = v4[q];
                win[4 * q] = t.x; win[4 * q + 1] = t.y; win[4 * q + 2] = t.z; win[4 * q + 3] = t.w;
            }
            double acc[kB2Seg];
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) acc[j] = 0.0;
#pragma unroll
            for (int e = 0; e < G::kWin; ++e) {
                const double x = b2_widen<R, kAlu>(win[G::kM + e]);
#pragma unroll
                for (int j = 0; j < kB2Seg; ++j) {
                    const int t = e - j;
                    if (t >= 0 && t < G::kLen) acc[j] = __fma_rn(a.taps[t], x, acc[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) hres[it][j] = (float)acc[j];   // float tmp (scalespace.cpp:86)
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < G::kItems; ++it) {
        const int item = threadIdx.x + it * kB2Threads;
        if (item < G::kHR * (kB2W / kB2Seg)) {
            float* o = sm + (item >> 3) * G::kTmpPitch + (item & 7) * kB2Seg;
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) o[j] = hres[it][j];
        }
    }
    __syncthreads();
}

// V pass: item = (column c, 8-row group), lanes along x; writes G and, for
// LEVEL / DECIMATE, DoG (and the DECIMATE seed = this octave's G[0]).
template <int R, int MODE, bool kAlu>
__device__ __forceinline__ void b2_vpass(const BlurArgs& a, const float* sm, int b, int x0, int y0) {
    using G = B2Geom<R>;
    const int w = a.w, h = a.h, pitch = a.pitch;
    const float* __restrict__ src = a.src + b * a.src_img_stride;
    float* __restrict__ dst = a.dst + b * a.dst_img_stride;
    float* __restrict__ dog = a.dog ? a.dog + b * a.dog_img_stride : nullptr;
    float* __restrict__ seed = (MODE == kModeDecimate) ? a.seed + b * a.seed_img_stride : nullptr;
    for (int item = threadIdx.x; item < kB2W * (kB2H / kB2Seg); item += kB2Threads) {
        const int c = item & (kB2W - 1), rg = item >> 6;
        const int x = x0 + c;
        double acc[kB2Seg];
#pragma unroll
        for (int j = 0; j < kB2Seg; ++j) acc[j] = 0.0;
        const float* col = sm + (rg * kB2Seg) * G::kTmpPitch + c;
#pragma unroll
        for (int e = 0; e < G::kWin; ++e) {
            const double v = b2_widen<R, kAlu>(col[e * G::kTmpPitch]);
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) {
                const int t = e - j;
                if (t >= 0 && t < G::kLen) acc[j] = __fma_rn(a.taps[t], v, acc[j]);
            }
        }
        if (x < w) {
            const int yb = y0 + rg * kB2Seg;
            const long long ob = (long long)yb * pitch + x;
            float* dp = dst + ob;                            // row bases of this item, once
            const float* sp = src + ob;
            float* gp = dog ? dog + ob : dst;
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) {
                const int y = yb + j;
                if (y < h) {
                    const float g = (float)acc[j];
                    const long long off = ob + j * pitch;
                    dp[j * pitch] = g;
                    // DoG[i-1] = G[i] - G[i-1] (scalespace.cpp:209); G[i-1] was just read (L2)
                    if (MODE == kModeLevel) {
                        if (dog) gp[j * pitch] = g - __ldg(sp + j * pitch);
                    } else if (MODE == kModeDecimate) {
                        // G[0] of this octave = even samples of G[s] of the previous one (scalespace.cpp:133-142)
                        const float prev = __ldg(src + (long long)(2 * y) * a.src_pitch + 2 * x);
                        seed[off] = prev;
                        if (dog) gp[j * pitch] = g - prev;
                    }
                }
            }
        }
    }
}

template <int R, int MODE>
__global__ void __launch_bounds__(kB2Threads)
blur_level2_kernel(const __grid_constant__ BlurArgs a) {
    using G = B2Geom<R>;
    extern __shared__ __align__(16) float sm2[];       // staged input [kHR][kInPitch], then tmp [kHR][kTmpPitch]
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kB2W, y0 = blockIdx.y * kB2H;
    const int w = a.w, h = a.h, pitch = a.pitch;
    const float* __restrict__ src = a.src + b * a.src_img_stride;
    const int cx0 = x0 - R - G::kM;                    // 16-byte aligned column of staged column 0

    // ---- stage the input tile; note whether every value is a positive normal
    //      float >= 2^-100 (then the tmp values are positive normals too: the
    //      smallest tap is > 2^-20) so both passes may widen on the ALU pipe
    bool alu_ok = true;
    const bool interior = MODE == kModeLevel && cx0 >= 0 && cx0 + G::kInW <= pitch && x0 + kB2W + R <= w &&
                          y0 - R >= 0 && y0 + kB2H + R <= h;
    if (interior) {
        // asynchronous 16-byte copies: the whole tile is in flight at once
        // (chunk i = r * kV + q of thread t: t, t + 256, ...; the row / column
        // and both addresses advance incrementally)
        constexpr int kV = G::kInW / 4;
        constexpr int kDr = kB2Threads / kV, kDq = kB2Threads % kV;
        const int r0 = threadIdx.x / kV, q0 = threadIdx.x - r0 * kV;
        {
            int r = r0, q = q0;
            const float* gp = src + (long long)(y0 - R + r) * pitch + cx0 + 4 * q;
            unsigned sa = (unsigned)__cvta_generic_to_shared(sm2 + r * G::kInPitch + 4 * q);
            while (r < G::kHR) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gp));
                r += kDr;
                q += kDq;
                gp += kDr * pitch + 4 * kDq;
                sa += 4 * (kDr * G::kInPitch + 4 * kDq);
                if (q >= kV) {
                    q -= kV;
                    ++r;
                    gp += pitch - 4 * kV;
                    sa += 4 * (G::kInPitch - 4 * kV);
                }
            }
        }
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
        {
            int r = r0, q = q0, m = 0x7fffffff, M = 0;
            const float* sp = sm2 + r * G::kInPitch + 4 * q;
            while (r < G::kHR) {
                const int4 v = *reinterpret_cast<const int4*>(sp);
                m = min(m, min(min(v.x, v.y), min(v.z, v.w)));
                M = max(M, max(max(v.x, v.y), max(v.z, v.w)));
                r += kDr;
                q += kDq;
                sp += kDr * G::kInPitch + 4 * kDq;
                if (q >= kV) {
                    q -= kV;
                    ++r;
                    sp += G::kInPitch - 4 * kV;
                }
            }
            alu_ok = (m >= 0x0d800000) & (M < 0x7f800000);
        }
    } else if (MODE == kModeUpsample && cx0 >= 0 && cx0 + G::kInW <= w - 1 && y0 - R >= 0 &&
               y0 + kB2H + R <= h - 1) {
        // interior bridge tile: stage the half-resolution patch once, then form
        // each 2x sample from shared memory (upsample2x, scalespace.cpp:113-131;
        // no reflection and no edge clamp can occur inside this tile)
        constexpr int kPW = G::kInW / 2 + 2, kPH = G::kHR / 2 + 2;
        float* patch = sm2 + G::kHR * G::kInPitch;          // [kPH][kPW]
        const int lx0 = cx0 >> 1, ly0 = (y0 - R) >> 1;
        for (int i = threadIdx.x; i < kPH * kPW; i += kB2Threads) {
            const int r = i / kPW, c = i - r * kPW;
            const float v = __ldg(src + (long long)min(ly0 + r, a.src_h - 1) * a.src_pitch + min(lx0 + c, a.src_w - 1));
            patch[i] = v;
            alu_ok &= (__float_as_int(v) >= 0x0d800000) & (__float_as_int(v) < 0x7f800000);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < G::kHR * G::kInW; i += kB2Threads) {
            const int r = i / G::kInW, c = i - r * G::kInW;
            const int gx = cx0 + c, gy = y0 - R + r;
            const float* p0 = patch + ((gy >> 1) - ly0) * kPW + ((gx >> 1) - lx0);
            const float* p1 = p0 + ((gy & 1) ? kPW : 0);
            const int dx = gx & 1;
            const double s4 = (((double)p0[0] + (double)p0[dx]) + (double)p1[0]) + (double)p1[dx];
            sm2[r * G::kInPitch + c] = (float)(0.25 * s4);
        }
    } else if (MODE == kModeDecimate && cx0 >= 0 && cx0 + G::kInW <= w && y0 - R >= 0 && y0 + kB2H + R <= h) {
        // interior seed tile: even samples of the previous octave's G[s]
        // (decimate2x, scalespace.cpp:133-142), no reflection needed
        const float* gsrc = src + (long long)(2 * (y0 - R)) * a.src_pitch + 2 * cx0;
#pragma unroll 4
        for (int i = threadIdx.x; i < G::kHR * (G::kInW / 2); i += kB2Threads) {
            const int r = i / (G::kInW / 2), c2 = i - r * (G::kInW / 2);
            const float4 v = __ldg(reinterpret_cast<const float4*>(gsrc + (long long)(2 * r) * a.src_pitch) + c2);
            *reinterpret_cast<float2*>(sm2 + r * G::kInPitch + 2 * c2) = make_float2(v.x, v.z);
            alu_ok &= (__float_as_int(v.x) >= 0x0d800000) & (__float_as_int(v.x) < 0x7f800000) &
                      (__float_as_int(v.z) >= 0x0d800000) & (__float_as_int(v.z) < 0x7f800000);
        }
    } else {   // gather with reflect-101 (scalespace.cpp:41-48) through the mode's input
               // mapping: level / raw pixel, 2x upsample (:113-131), decimation (:133-142)
#pragma unroll 4
        for (int i = threadIdx.x; i < G::kHR * G::kInW; i += kB2Threads) {
            const int r = i / G::kInW, c = i - r * G::kInW;
            const float v = fetch_input<MODE>(a, src, reflect101(cx0 + c, w), reflect101(y0 - R + r, h));
            sm2[r * G::kInPitch + c] = v;
            alu_ok &= (__float_as_int(v) >= 0x0d800000) & (__float_as_int(v) < 0x7f800000);
        }
    }
    if (__syncthreads_and(alu_ok)) {
        b2_hpass<R, true>(a, sm2);
        b2_vpass<R, MODE, true>(a, sm2, b, x0, y0);
    } else {
        b2_hpass<R, false>(a, sm2);
        b2_vpass<R, MODE, false>(a, sm2, b, x0, y0);
    }
}

template <int MODE>
static cudaError_t launch_v2(const BlurArgs& a, int R, int batch, cudaStream_t st) {
    const dim3 grid((a.w + kB2W - 1) / kB2W, (a.h + kB2H - 1) / kB2H, batch);
    size_t smem = 0;
    void (*fn)(BlurArgs) = nullptr;
    switch (R) {
#define DSIFT_R2(r) case r: fn = blur_level2_kernel<r, MODE>; smem = B2Geom<r>::kSmem + (MODE == kModeUpsample ? \
        sizeof(float) * (size_t)(B2Geom<r>::kHR / 2 + 2) * (B2Geom<r>::kInW / 2 + 2) : 0); break;
        DSIFT_R2(1) DSIFT_R2(2) DSIFT_R2(3) DSIFT_R2(4) DSIFT_R2(5) DSIFT_R2(6) DSIFT_R2(7) DSIFT_R2(8)
        DSIFT_R2(9) DSIFT_R2(10) DSIFT_R2(11) DSIFT_R2(12) DSIFT_R2(13) DSIFT_R2(14) DSIFT_R2(15)
        DSIFT_R2(16)
#undef DSIFT_R2
        default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kB2Threads, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_blur(const BlurArgs& a, int mode, int R, int batch, cudaStream_t st) {
    const bool tiled = R >= 1 && R <= 16;
    switch (mode) {
        case kModeLevel: return tiled ? launch_v2<kModeLevel>(a, R, batch, st) : launch_any<kModeLevel>(a, R, batch, st);
        case kModeRaw: return tiled ? launch_v2<kModeRaw>(a, R, batch, st) : launch_any<kModeRaw>(a, R, batch, st);
        case kModeUpsample:
            return tiled ? launch_v2<kModeUpsample>(a, R, batch, st) : launch_any<kModeUpsample>(a, R, batch, st);
        default: return tiled ? launch_v2<kModeDecimate>(a, R, batch, st) : launch_any<kModeDecimate>(a, R, batch, st);
    }
}

}  // namespace dsift
