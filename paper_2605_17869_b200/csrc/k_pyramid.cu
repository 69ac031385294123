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
#include "dsift_tma.cuh"

namespace dsift {

DSIFT_BOUNDS_UNIT(pyramid)

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
// Tiled bridge blur of upsampled configs (UPSAMPLE mode; every other level
// runs in the strip kernel below).
//
//   * the (64+2R)^2 input tile of the 2x upsampled base is formed from a
//     staged half-resolution patch (interior tiles) or gathered with
//     reflect-101 (border tiles), 16-byte aligned so the H pass reads its
//     window with LDS.128;
//   * 8 outputs per thread in both passes: each staged value is converted to
//     FP64 once per 8-output window and feeds 8 independent DFMA chains.
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

// V pass: item = (column c, 8-row group), lanes along x; writes the bridge
// level G[0] (the octave's first level has no DoG below it).
template <int R, bool kAlu>
__device__ __forceinline__ bool b2_vpass(const BlurArgs& a, const float* sm, int b, int x0, int y0) {
    bool ok = true;   // every output a positive normal >= 2^-100 (the consumer's ALU widen)
    using G = B2Geom<R>;
    const int w = a.w, h = a.h, pitch = a.pitch;
    float* __restrict__ dst = a.dst + b * a.dst_img_stride;
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
        const int yb = y0 + rg * kB2Seg;
        float* dp = dst + (long long)yb * pitch + x;
        if (x < w && yb + kB2Seg <= h) {
            // every row exists; positive-normal test as one unsigned max
            unsigned m = 0u;
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) {
                const float g = (float)acc[j];
                m = max(m, __float_as_uint(g) - 0x0d800000u);
                dp[j * pitch] = g;
            }
            ok &= m < (0x7f800000u - 0x0d800000u);
        } else if (x < w) {
#pragma unroll
            for (int j = 0; j < kB2Seg; ++j) {
                if (yb + j < h) {
                    const float g = (float)acc[j];
                    ok &= (unsigned)(__float_as_uint(g) - 0x0d800000u) < (0x7f800000u - 0x0d800000u);
                    dp[j * pitch] = g;
                }
            }
        }
    }
    return ok;
}

template <int R, int MODE>
__global__ void __launch_bounds__(kB2Threads, 5)   // swept 3-6 CTAs/SM: 5 best
blur_level2_kernel(const __grid_constant__ BlurArgs a) {
    static_assert(MODE == kModeUpsample, "the tiled kernel is the upsampled bridge; levels use the strip kernel");
    using G = B2Geom<R>;
    extern __shared__ __align__(16) float sm2[];       // staged input [kHR][kInPitch], then tmp [kHR][kTmpPitch]
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kB2W, y0 = blockIdx.y * kB2H;
    const int w = a.w, h = a.h;
    const float* __restrict__ src = a.src + b * a.src_img_stride;
    const int cx0 = x0 - R - G::kM;                    // 16-byte aligned column of staged column 0

    // ---- stage the input tile; note whether every value is a positive normal
    //      float >= 2^-100 (then the tmp values are positive normals too: the
    //      smallest tap is > 2^-20) so both passes may widen on the ALU pipe
    bool alu_ok = true;
    if (MODE == kModeUpsample && cx0 >= 0 && cx0 + G::kInW <= w - 1 && y0 - R >= 0 &&
               y0 + kB2H + R <= h - 1) {
        // interior bridge tile: stage the half-resolution patch once, then form
        // each 2x sample from shared memory (upsample2x, scalespace.cpp:113-131;
        // no reflection and no edge clamp can occur inside this tile)
        // (the patch is widened to FP64 once; each of the ~4 upsampled samples
        // per patch value then needs no conversion of its own)
        constexpr int kPW = G::kInW / 2 + 2, kPH = G::kHR / 2 + 2;
        double* patch = reinterpret_cast<double*>(sm2 + G::kHR * G::kInPitch);   // [kPH][kPW]
        const int lx0 = cx0 >> 1, ly0 = (y0 - R) >> 1;
        for (int i = threadIdx.x; i < kPH * kPW; i += kB2Threads) {
            const int r = i / kPW, c = i - r * kPW;
            const float v = __ldg(src + (long long)min(ly0 + r, a.src_h - 1) * a.src_pitch + min(lx0 + c, a.src_w - 1));
            patch[i] = (double)v;
            alu_ok &= (__float_as_int(v) >= 0x0d800000) & (__float_as_int(v) < 0x7f800000);
        }
        __syncthreads();
        // one thread per patch cell (a, b / c, d): the 2x2 block of samples
        // gx = 2X + {0, 1}, gy = 2Y + {0, 1} it defines, each
        // ((p0[0] + p0[dx]) + p1[0]) + p1[dx] with the reference's operands
        // (a + b is shared by the two odd-x samples).  cx0 is even, so block
        // column X covers staged columns 2X, 2X + 1; block row Y covers
        // staged rows r0 + 2Y, + 1 with r0 = 0 or -1 (y0 - R odd).
        static_assert((G::kInW & 1) == 0 && (G::kInPitch & 1) == 0, "float2 block rows");
        constexpr int kBX = G::kInW / 2;
        const int r0 = 2 * ly0 - (y0 - R);
        const int nby = (G::kHR - r0 + 1) >> 1;
        for (int i = threadIdx.x; i < nby * kBX; i += kB2Threads) {
            const int by = i / kBX, bx = i - by * kBX;
            const double* p = patch + by * kPW + bx;
            const double pa = p[0], pb = p[1], pc = p[kPW], pd = p[kPW + 1];
            const double a2 = pa + pa, ab = pa + pb;
            const int r = r0 + 2 * by;
            float2* o = reinterpret_cast<float2*>(sm2 + r * G::kInPitch + 2 * bx);
            if (r >= 0) o[0] = make_float2((float)(0.25 * ((a2 + pa) + pa)), (float)(0.25 * ((ab + pa) + pb)));
            if (r + 1 < G::kHR)
                o[G::kInPitch / 2] = make_float2((float)(0.25 * ((a2 + pc) + pc)), (float)(0.25 * ((ab + pc) + pd)));
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
    bool out_ok;
    if (__syncthreads_and(alu_ok)) {
        b2_hpass<R, true>(a, sm2);
        out_ok = b2_vpass<R, true>(a, sm2, b, x0, y0);
    } else {
        b2_hpass<R, false>(a, sm2);
        out_ok = b2_vpass<R, false>(a, sm2, b, x0, y0);
    }
    if (!__syncthreads_and(out_ok) && a.dst_flag && threadIdx.x == 0) atomicOr(a.dst_flag, 1);
}

// ---------------------------------------------------------------------------
// Strip kernel (LEVEL, RAW and DECIMATE modes).
//
// A CTA owns a 32-column strip of one image over a segment of rows and slides
// down it 32 rows per step, so every horizontal-pass row is computed once per
// segment (64x64 tiles recompute 2R halo rows per tile: +15% DFMA):
//   1. the step's 32 new input rows (32 + 2R columns) arrive by TMA in a
//      double-buffered float stage, issued one step ahead (decimation is a
//      TMA element stride of 2); border strips and border rows are gathered
//      with reflect-101 instead (scalespace.cpp:41-48);
//   2. H pass: thread (row, 8-column segment) forms 8 outputs, each the
//      left-to-right FP64 tap sum rounded to float (scalespace.cpp:63-86),
//      stored as FP64 in a ring of >= 32 + 2R rows;
//   3. V pass: thread (column pair, 4-row group) forms 8 outputs from the
//      ring (scalespace.cpp:88-109) and writes G, DoG and the DECIMATE seed
//      with 8-byte stores.
// Inputs are widened to FP64 on the integer pipe when the producer of the
// level flagged every value a positive normal >= 2^-100 (then every tmp
// value is one too); otherwise by the conversion unit.
// ---------------------------------------------------------------------------
constexpr int kSW = 32, kSR = 32, kS3Threads = 128;

template <int R>
struct S3 {
    static constexpr int kLen = 2 * R + 1;
    static constexpr int kWinN = 8 + 2 * R;                       // inputs of 8 outputs
    static constexpr int kM = (4 - (R & 3)) & 3;                  // x0 - R - kM = 0 (mod 4)
    static constexpr int kInW0 = ((kSW + 2 * R + kM + 3) / 4) * 4;
    // staged columns (TMA box width): an odd number of 16-byte chunks per row,
    // so the 8 rows of a quarter-warp's LDS.128 fall in 8 different bank groups
    static constexpr int kInW = ((kInW0 / 4) & 1) ? kInW0 : kInW0 + 4;
    static constexpr int kNV = (kM + kWinN + 3) / 4;              // float4 reads per H window
    static constexpr int kRS = (kSR + 2 * R + 3) / 4 * 4;         // ring rows (a multiple of 4)
    static constexpr int kTP = kSW + 2;                           // ring pitch (doubles), = 2 (mod 16)
    static constexpr size_t kStageBytes = sizeof(float) * (size_t)kSR * kInW;   // one TMA box
    static constexpr size_t kSmem = 2 * kStageBytes + sizeof(double) * (size_t)kRS * kTP + 128;
};

__device__ __forceinline__ int reflect_fast(int p, int n) {
    return ((unsigned)p < (unsigned)n) ? p : reflect101(p, n);
}

// a positive normal float >= 2^-100, finite
__device__ __forceinline__ bool alu_widenable(float v) {
    return (unsigned)(__float_as_uint(v) - 0x0d800000u) < (0x7f800000u - 0x0d800000u);
}

template <bool kAlu>
__device__ __forceinline__ double s3_widen(float x) {
    if (kAlu) return widen_pos_normal(x);
    return (double)x;
}

// Gather virtual rows [t0, t0 + n) of the level's input (columns [xs, xs + kInW))
// into a float stage: reflect-101 at the image border (scalespace.cpp:41-48),
// even samples (DECIMATE).
// Returns whether every staged value this thread wrote is ALU-widenable.
template <int R, int MODE>
__device__ __forceinline__ bool s3_gather(const BlurArgs& a, const float* __restrict__ src, float* stg, int t0, int n,
                                          int xs) {
    using G = S3<R>;
    bool ok = true;
    const bool inner = xs >= 0 && xs + G::kInW <= a.w && t0 >= 0 && t0 + n <= a.h;
    if (MODE == kModeDecimate && inner && ((a.src_pitch | (int)(a.src_img_stride & 3)) & 3) == 0) {
        // interior rows of the previous octave's level: even samples of
        // 16-byte loads (decimate2x, scalespace.cpp:133-142), two per staged float4
        constexpr int kV = G::kInW / 4;
        constexpr int kIt = (kSR * kV + kS3Threads - 1) / kS3Threads;
        float4 u0[kIt], u1[kIt];
#pragma unroll
        for (int k = 0; k < kIt; ++k) {   // every load of the step in flight at once
            const int q = threadIdx.x + k * kS3Threads;
            if (q < n * kV) {
                const int r = q / kV, c4 = q - r * kV;
                const float4* p =
                    reinterpret_cast<const float4*>(src + (long long)(2 * (t0 + r)) * a.src_pitch + 2 * xs) + 2 * c4;
                u0[k] = __ldg(p);
                u1[k] = __ldg(p + 1);
            }
        }
#pragma unroll
        for (int k = 0; k < kIt; ++k) {
            const int q = threadIdx.x + k * kS3Threads;
            if (q < n * kV) {
                const float4 v = make_float4(u0[k].x, u0[k].z, u1[k].x, u1[k].z);
                ok &= alu_widenable(v.x) & alu_widenable(v.y) & alu_widenable(v.z) & alu_widenable(v.w);
                reinterpret_cast<float4*>(stg)[q] = v;
            }
        }
        return ok;
    }
    for (int q = threadIdx.x; q < n * G::kInW; q += kS3Threads) {
        const int r = q / G::kInW, c = q - r * G::kInW;
        const float v = fetch_input<MODE>(a, src, reflect_fast(xs + c, a.w), reflect_fast(t0 + r, a.h));
        ok &= alu_widenable(v);
        stg[q] = v;
    }
    return ok;
}

// H pass over n staged rows; their ring slot is (k0 + row) mod RS.
template <int R, bool kAlu>
__device__ __forceinline__ void s3_hpass(const BlurArgs& a, const float* stg, double* ring, int n, int k0) {
    using G = S3<R>;
    const int seg = threadIdx.x >> 5, r = threadIdx.x & 31;   // a warp = 32 rows of one segment
    if (r >= n) return;
    const float4* wp = reinterpret_cast<const float4*>(stg + r * G::kInW + 8 * seg);
    float win[4 * G::kNV];
#pragma unroll
    for (int q = 0; q < G::kNV; ++q) {
        const float4 t = wp[q];
        win[4 * q] = t.x;
        win[4 * q + 1] = t.y;
        win[4 * q + 2] = t.z;
        win[4 * q + 3] = t.w;
    }
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
    for (int e = 0; e < G::kWinN; ++e) {
        const double x = s3_widen<kAlu>(win[G::kM + e]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int t = e - j;
            if (t >= 0 && t < G::kLen) acc[j] = __fma_rn(a.taps[t], x, acc[j]);
        }
    }
    int k = k0 + r;
    if (k >= G::kRS) k -= G::kRS;
    DSIFT_BOUND(k >= 0 && k < G::kRS && 8 * seg + 8 <= G::kTP && r * G::kInW + 8 * seg + 4 * G::kNV <= kSR * G::kInW, 101);
    double2* o0 = reinterpret_cast<double2*>(ring + k * G::kTP + 8 * seg);
#pragma unroll
    for (int j = 0; j < 8; j += 2)   // the float tmp of scalespace.cpp:86, kept as FP64
        o0[j / 2] = make_double2(s3_widen<kAlu>((float)acc[j]), s3_widen<kAlu>((float)acc[j + 1]));
}

template <int R, int MODE>
__device__ __forceinline__ void blur_strip_body(const BlurArgs& a, int seg_h, float* stage0, double* ring,
                                                uint64_t* bar, bool alu_level) {
    using G = S3<R>;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kSW;
    const int y_begin = blockIdx.y * seg_h;
    const int w = a.w, h = a.h, pitch = a.pitch, sp = a.src_pitch;
    const int y_end = min(h, y_begin + seg_h);
    const float* __restrict__ src = a.src + b * a.src_img_stride;
    const int xs = x0 - R - G::kM;
    const bool strip_in = a.use_tma && xs >= 0 && xs + G::kInW <= w;
    constexpr int kStageF = (int)(G::kStageBytes / sizeof(float));
    // rows [t0, t0 + n) come by TMA iff they are inside the image (no
    // reflection); gathered rows report whether they are ALU-widenable
    auto issue = [&](int t0, int n, int buf, bool& gok) -> bool {
        float* st = stage0 + buf * kStageF;
        if (strip_in && t0 >= 0 && t0 + n <= h) {
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&bar[buf], (unsigned)G::kStageBytes);
                tma_load_3d(st, &a.src_map, xs, t0, b, &bar[buf]);
            }
            return true;
        }
        gok = s3_gather<R, MODE>(a, src, st, t0, n, xs);
        return false;
    };
    float* __restrict__ dst = a.dst + b * a.dst_img_stride;
    float* __restrict__ dog = a.dog ? a.dog + b * a.dog_img_stride : nullptr;
    float* __restrict__ seed = (MODE == kModeDecimate) ? a.seed + b * a.seed_img_stride : nullptr;
    // V-pass thread: column pair cp (x = x0 + 2cp, +1), 4-row group g
    const int cp = threadIdx.x & 15, g = threadIdx.x >> 4;
    const int xv = x0 + 2 * cp;
    bool out_ok = true;   // every output a positive normal >= 2^-100 (the consumer's ALU widen)

    // prologue: virtual rows [y_begin - R, y_begin + R) through stage 1
    unsigned ph0 = 0u, ph1 = 0u;
    bool tma0, tma1, gok0 = true, gok1 = true;
    tma1 = issue(y_begin - R, 2 * R, 1, gok1);
    const bool alu_pro = tma1 ? alu_level : (bool)__syncthreads_and(gok1);
    tma0 = issue(y_begin + R, min(kSR, y_end - y_begin), 0, gok0);   // step 0's rows
    __syncthreads();
    if (tma1) {
        mbar_wait(&bar[1], ph1);
        ph1 ^= 1u;
    }
    if (alu_pro) s3_hpass<R, true>(a, stage0 + kStageF, ring, 2 * R, 0);
    else s3_hpass<R, false>(a, stage0 + kStageF, ring, 2 * R, 0);
    int kn = 2 * R;   // ring slot of the next new row
    int kv = 4 * g;   // ring slot of this thread's first V-window row
    int cur = 0;
    for (int ys = y_begin; ys < y_end; ys += kSR) {
        const int nnew = min(kSR, y_end - ys);
        __syncthreads();   // the previous H pass has read the other stage buffer
        if (ys + kSR < y_end) {
            if (cur) tma0 = issue(ys + kSR + R, min(kSR, y_end - ys - kSR), 0, gok0);
            else tma1 = issue(ys + kSR + R, min(kSR, y_end - ys - kSR), 1, gok1);
        }
        // the previous level's values at this thread's outputs (DoG / seed),
        // loaded now so their latency hides behind the passes
        const int yb = ys + 4 * g;
        const bool full = x0 + kSW <= w && ys + kSR <= y_end;   // CTA-uniform: no edge checks
        float2 prev[4];
        if ((MODE == kModeLevel || MODE == kModeDecimate) && full) {
            // interior step: rows yb .. yb + 3 all exist; one base pointer
            const float* p0 = src + (long long)(MODE == kModeLevel ? yb : 2 * yb) * sp +
                              (MODE == kModeLevel ? xv : 2 * xv);
            const int rstep = MODE == kModeLevel ? sp : 2 * sp;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (MODE == kModeLevel) {
                    prev[j] = __ldg(reinterpret_cast<const float2*>(p0 + j * rstep));
                } else {
                    const float4 q = __ldg(reinterpret_cast<const float4*>(p0 + j * rstep));
                    prev[j] = make_float2(q.x, q.z);
                }
            }
        } else if (MODE == kModeLevel || MODE == kModeDecimate) {
            const int xa = min(xv, w - 1), xb = min(xv + 1, w - 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int y = min(yb + j, y_end - 1);
                if (MODE == kModeLevel) {
                    const float* p = src + (long long)y * sp;
                    prev[j] = full ? __ldg(reinterpret_cast<const float2*>(p + xv)) : make_float2(__ldg(p + xa), __ldg(p + xb));
                } else {
                    const float* p = src + (long long)(2 * y) * sp;
                    if (full) {
                        const float4 q = __ldg(reinterpret_cast<const float4*>(p + 2 * xv));
                        prev[j] = make_float2(q.x, q.z);
                    } else {
                        prev[j] = make_float2(__ldg(p + 2 * xa), __ldg(p + 2 * xb));
                    }
                }
            }
        }
        const bool tcur = cur ? tma1 : tma0;
        bool alu_step = alu_level;
        if (!tcur) {
            alu_step = __syncthreads_and(cur ? gok1 : gok0);   // gathered rows: visible to all threads
        } else if (cur) {
            mbar_wait(&bar[1], ph1);
            ph1 ^= 1u;
        } else {
            mbar_wait(&bar[0], ph0);
            ph0 ^= 1u;
        }
        if (alu_step) s3_hpass<R, true>(a, stage0 + cur * kStageF, ring, nnew, kn);
        else s3_hpass<R, false>(a, stage0 + cur * kStageF, ring, nnew, kn);
        kn += nnew;
        if (kn >= G::kRS) kn -= G::kRS;
        cur ^= 1;
        __syncthreads();
        // V pass: columns xv, xv + 1, rows yb .. yb + 3; the window's ring rows
        // kv .. kv + 4 + 2R - 1 (mod RS): kv and RS are multiples of 4, so each
        // aligned block of 4 rows wraps as a whole
        if (4 * g < nnew) {
            const double* colp = ring + kv * G::kTP + 2 * cp;
            double acc[8];   // [row j][column k] = acc[2j + k]
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] = 0.0;
            constexpr int kWinV = 4 + 2 * R;
#pragma unroll
            for (int e0 = 0; e0 < kWinV; e0 += 4) {
                const double* cb = (kv + e0 < G::kRS) ? colp + e0 * G::kTP : colp + (e0 - G::kRS) * G::kTP;
                DSIFT_BOUND(((kv + e0 < G::kRS) ? kv + e0 : kv + e0 - G::kRS) + 3 < G::kRS && 2 * cp + 2 <= G::kTP, 102);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int e = e0 + i;
                    if (e < kWinV) {
                        const double2 v = *reinterpret_cast<const double2*>(cb + i * G::kTP);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int t = e - j;
                            if (t >= 0 && t < G::kLen) {
                                acc[2 * j] = __fma_rn(a.taps[t], v.x, acc[2 * j]);
                                acc[2 * j + 1] = __fma_rn(a.taps[t], v.y, acc[2 * j + 1]);
                            }
                        }
                    }
                }
            }
            float* dp = dst + (long long)yb * pitch + xv;
            float* gp = dog ? dog + (long long)yb * pitch + xv : nullptr;
            float* sd = (MODE == kModeDecimate) ? seed + (long long)yb * pitch + xv : nullptr;
            DSIFT_BOUND(!full || (yb + 3 < y_end && xv + 1 < w), 103);
            if (full) {
                unsigned um = 0u;   // positive-normal test of the 8 outputs as one unsigned max
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 gv = make_float2((float)acc[2 * j], (float)acc[2 * j + 1]);
                    um = max(um, max(__float_as_uint(gv.x) - 0x0d800000u, __float_as_uint(gv.y) - 0x0d800000u));
                    *reinterpret_cast<float2*>(dp + j * pitch) = gv;
                    if (MODE == kModeLevel || MODE == kModeDecimate) {
                        // DoG[i-1] = G[i] - G[i-1] (scalespace.cpp:209); DECIMATE also
                        // writes this octave's G[0] (scalespace.cpp:133-142)
                        if (MODE == kModeDecimate) *reinterpret_cast<float2*>(sd + j * pitch) = prev[j];
                        if (gp) *reinterpret_cast<float2*>(gp + j * pitch) = make_float2(gv.x - prev[j].x, gv.y - prev[j].y);
                    }
                }
                out_ok &= um < (0x7f800000u - 0x0d800000u);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (yb + j < y_end) {
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            if (xv + k < w) {
                                const float gv = (float)acc[2 * j + k];
                                const float pv = k ? prev[j].y : prev[j].x;
                                out_ok &= alu_widenable(gv);
                                dp[j * pitch + k] = gv;
                                if (MODE == kModeDecimate) sd[j * pitch + k] = pv;
                                if ((MODE == kModeLevel || MODE == kModeDecimate) && gp) gp[j * pitch + k] = gv - pv;
                            }
                        }
                    }
                }
            }
        }
        kv += kSR;
        if (kv >= G::kRS) kv -= G::kRS;
    }
    if (!__syncthreads_and(out_ok) && a.dst_flag && threadIdx.x == 0) atomicOr(a.dst_flag, 1);
}

template <int R, int MODE>
__global__ void __launch_bounds__(kS3Threads, 6)   // 5 / 7 / 8 measured slower
blur_strip_kernel(const __grid_constant__ BlurArgs a, int seg_h) {
    using G = S3<R>;
    extern __shared__ __align__(128) unsigned char sm3_raw[];
    // 128-byte aligned TMA destination; offset from the array itself so the
    // compiler keeps every access in the shared window (LDS, not generic LD)
    unsigned char* base = sm3_raw + ((128u - (smem_u32(sm3_raw) & 127u)) & 127u);
    float* stage0 = reinterpret_cast<float*>(base);                          // [2][kSR][kInW] (TMA boxes)
    double* ring = reinterpret_cast<double*>(base + 2 * G::kStageBytes);    // [kRS][kTP]
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
    }
    __syncthreads();
    // ALU widening needs every source value to be a positive normal >= 2^-100
    // (flag written by the level's producer; the input image has none)
    const bool alu = a.src_flag != nullptr && *a.src_flag == 0;
    blur_strip_body<R, MODE>(a, seg_h, stage0, ring, bar, alu);
}

// rows per CTA segment: long segments amortise the 2R-row prologue, short ones
// give small octaves enough CTAs (>= ~2 waves of 6 per SM)
static int s3_seg_h(int w, int h, int batch) {
    const long long strips = (long long)((w + kSW - 1) / kSW) * batch;
    // ~256-row segments: swept 128..1024 on C3 (8.39 / 8.38 / 8.38 / 8.43 / 8.84 / 9.64
    // ms per 32 images at 128 / 192 / 256 / 320 / 512 / 1024) — the 2R-row prologue
    // per segment costs less than the tail of fewer, longer CTAs
    int nseg = std::max(1, (h + 128) / 256);
    // small octaves: split into >= 64-row segments until there are ~2 CTAs per
    // resident slot.  More (8 / 16 waves, 32-row minimums) shortens the device-
    // resident pyramid (8.37 -> 8.17 ms) but floods the block scheduler while the
    // other context's descriptor kernel waits for SMs: the two-context end-to-end
    // number falls from 256 to 241 images/s (measured; from 4 waves on)
    const long long want = 148LL * 6 * 2;
    while ((long long)nseg * strips < want && (h + nseg) / (nseg + 1) >= 64) ++nseg;
    const int per = (h + nseg - 1) / nseg;
    return ((per + kSR - 1) / kSR) * kSR;
}

int blur_strip_box_w(int R) {
    switch (R) {
#define DSIFT_BW(r) case r: return S3<r>::kInW;
        DSIFT_BW(1) DSIFT_BW(2) DSIFT_BW(3) DSIFT_BW(4) DSIFT_BW(5) DSIFT_BW(6) DSIFT_BW(7) DSIFT_BW(8)
        DSIFT_BW(9) DSIFT_BW(10) DSIFT_BW(11) DSIFT_BW(12) DSIFT_BW(13) DSIFT_BW(14) DSIFT_BW(15) DSIFT_BW(16)
#undef DSIFT_BW
        default: return 0;
    }
}

template <int MODE>
static cudaError_t launch_strip(const BlurArgs& a, int R, int batch, cudaStream_t st) {
    const int seg_h = s3_seg_h(a.w, a.h, batch);
    const dim3 grid((a.w + kSW - 1) / kSW, (a.h + seg_h - 1) / seg_h, batch);
    size_t smem = 0;
    void (*fn)(BlurArgs, int) = nullptr;
    switch (R) {
#define DSIFT_R3(r) case r: fn = blur_strip_kernel<r, MODE>; smem = S3<r>::kSmem; break;
        DSIFT_R3(1) DSIFT_R3(2) DSIFT_R3(3) DSIFT_R3(4) DSIFT_R3(5) DSIFT_R3(6) DSIFT_R3(7) DSIFT_R3(8)
        DSIFT_R3(9) DSIFT_R3(10) DSIFT_R3(11) DSIFT_R3(12) DSIFT_R3(13) DSIFT_R3(14) DSIFT_R3(15)
        DSIFT_R3(16)
#undef DSIFT_R3
        default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, kS3Threads, smem, st>>>(a, seg_h);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_v2(const BlurArgs& a, int R, int batch, cudaStream_t st) {
    const dim3 grid((a.w + kB2W - 1) / kB2W, (a.h + kB2H - 1) / kB2H, batch);
    size_t smem = 0;
    void (*fn)(BlurArgs) = nullptr;
    switch (R) {
#define DSIFT_R2(r) case r: fn = blur_level2_kernel<r, MODE>; smem = B2Geom<r>::kSmem + (MODE == kModeUpsample ? \
        sizeof(double) * (size_t)(B2Geom<r>::kHR / 2 + 2) * (B2Geom<r>::kInW / 2 + 2) : 0); break;
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
        case kModeLevel: return tiled ? launch_strip<kModeLevel>(a, R, batch, st) : launch_any<kModeLevel>(a, R, batch, st);
        case kModeRaw: return tiled ? launch_strip<kModeRaw>(a, R, batch, st) : launch_any<kModeRaw>(a, R, batch, st);
        case kModeUpsample:   // the tiled kernel stages the half-resolution patch once per tile (faster here
                              // than forming the 2x rows per strip step: 1.22 vs 1.33 ms per 32 C3 images)
            return tiled ? launch_v2<kModeUpsample>(a, R, batch, st) : launch_any<kModeUpsample>(a, R, batch, st);
        default: return tiled ? launch_strip<kModeDecimate>(a, R, batch, st) : launch_any<kModeDecimate>(a, R, batch, st);
    }
}

}  // namespace dsift

namespace dsift {

// ---------------------------------------------------------------------------
// Small octaves, fused: one CTA per image runs every level of the octaves
// o_first..n_oct-1 (each small enough for two whole levels in shared memory)
// in one launch, instead of 5 launches per octave whose CTAs are mostly
// latency.  Per level: H pass G -> tmp (float-rounded FP64 tap sums,
// scalespace.cpp:63-86), V pass tmp -> G' (:88-109) writing G' and the DoG
// G' - G (:209) to HBM and G' over G in shared memory (each element is read
// and replaced by the same thread).  The next octave's G[0] is the even
// samples of G[s] (decimate2x, :133-142), kept in a third buffer.  Same
// arithmetic as the strip kernel; reflect-101 per element (:41-48).
// ---------------------------------------------------------------------------
constexpr int kSmallThreads = 1024;

__global__ void __launch_bounds__(kSmallThreads, 1)
blur_small_octaves_kernel(const __grid_constant__ SmallOctArgs a) {
    extern __shared__ __align__(16) float smo[];
    const PyramidDesc& p = a.pyr;
    const int b = blockIdx.x, s = p.s;
    const int o0 = a.o_first;
    const int cap = a.cap_px;              // floats per full buffer
    float* G = smo;                        // [h][w] current level
    float* T = smo + cap;                  // [h][w] H-pass tmp
    float* D = smo + 2 * cap;              // [h/2][w/2] next octave's G[0]
    for (int o = o0; o < p.n_oct; ++o) {
        const OctaveDesc& od = p.oct[o];
        const int w = od.w, h = od.h, pitch = od.pitch, n = w * h;
        float* gimg = od.gauss + (long long)b * p.gauss_img_stride(o);
        float* dimg = od.dog + (long long)b * p.dog_img_stride(o);
        // G[0]: even samples of the previous octave's G[s]
        if (o == o0) {
            const OctaveDesc& pd = p.oct[o - 1];
            const float* src = pd.gauss + (long long)b * p.gauss_img_stride(o - 1) + (long long)s * pd.level_stride;
            for (int i = threadIdx.x; i < n; i += kSmallThreads) {
                const int y = i / w, x = i - y * w;
                const float v = __ldg(src + (long long)(2 * y) * pd.pitch + 2 * x);
                G[i] = v;
                gimg[(long long)y * pitch + x] = v;
            }
        } else {
            for (int i = threadIdx.x; i < n; i += kSmallThreads) {
                const int y = i / w, x = i - y * w;
                G[i] = D[i];
                gimg[(long long)y * pitch + x] = D[i];
            }
        }
        __syncthreads();
        for (int lv = 1; lv < s + 3; ++lv) {
            const int R = a.radius[lv - 1];
            const double* taps = a.taps[lv - 1];
            // H pass (scalespace.cpp:63-86)
            for (int i = threadIdx.x; i < n; i += kSmallThreads) {
                const int y = i / w, x = i - y * w;
                const float* row = G + y * w;
                double acc = 0.0;
                for (int t = -R; t <= R; ++t) acc = __fma_rn(taps[t + R], (double)row[reflect101(x + t, w)], acc);
                T[i] = (float)acc;
            }
            __syncthreads();
            // V pass (scalespace.cpp:88-109) + DoG (scalespace.cpp:209)
            float* gl = gimg + (long long)lv * od.level_stride;
            float* dl = dimg + (long long)(lv - 1) * od.level_stride;
            for (int i = threadIdx.x; i < n; i += kSmallThreads) {
                const int y = i / w, x = i - y * w;
                double acc = 0.0;
                for (int t = -R; t <= R; ++t) acc = __fma_rn(taps[t + R], (double)T[reflect101(y + t, h) * w + x], acc);
                const float g = (float)acc;
                const long long off = (long long)y * pitch + x;
                gl[off] = g;
                dl[off] = g - G[i];
                G[i] = g;
            }
            __syncthreads();
            if (lv == s && o + 1 < p.n_oct) {   // decimate2x of G[s] (scalespace.cpp:133-142)
                const int w2 = p.oct[o + 1].w, h2 = p.oct[o + 1].h;
                for (int i = threadIdx.x; i < w2 * h2; i += kSmallThreads) {
                    const int y = i / w2, x = i - y * w2;
                    D[i] = G[(2 * y) * w + 2 * x];
                }
                // D is read only after the next octave's first barrier
            }
        }
    }
}

size_t small_octaves_smem(int cap_px) { return sizeof(float) * (size_t)(2 * cap_px + (cap_px + 3) / 4 + 4); }

cudaError_t launch_small_octaves(const SmallOctArgs& a, cudaStream_t st) {
    const size_t smem = small_octaves_smem(a.cap_px);
    cudaError_t e = cudaFuncSetAttribute(blur_small_octaves_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    blur_small_octaves_kernel<<<a.pyr.batch, kSmallThreads, smem, st>>>(a);
    return cudaGetLastError();
}

}  // namespace dsift
