// k_orient.cu — K4: dominant orientations + fan-out (reference:
// orient.cpp:13-113, io.cpp:117-125).
//
// A warp owns one keypoint at a time; a CTA (4 warps) owns a ticket-ordered
// tile of 16 keypoints.  The warp walks the window in the reference's scan
// order (row-major, 32 pixels per step), computes float central differences,
// sqrtf, the glibc-exact atan2f and float(exp()) weight per pixel, and feeds
// each bin's contributions, in scan order, into that bin's binary-counter
// tree (dsift_tree.cuh) — __match_any_sync groups the lanes that hit the same
// bin, the bin's owner lane pushes them in lane order.  No float atomics; the
// per-bin sums are bit-identical to tree_accumulate_histogram.  Smoothing,
// peak picking and parabolic refinement follow orient.cpp:62-113 in the
// reference's precision; peaks are ranked by warp ballot, and the tile's copy
// count goes through the decoupled look-back so oriented keypoints land in
// keypoint order (the reference's flattened per-candidate slots).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_math.cuh"
#include "dsift_scan.cuh"
#include "dsift_tree.cuh"

namespace dsift {

DSIFT_BOUNDS_UNIT(orient)

constexpr int kOriWarps = 4;
constexpr int kOriPerWarp = 4;
constexpr int kOriTile = kOriWarps * kOriPerWarp;
constexpr int kOriAxis = 64;   // per-axis weight factors held (window side 2R+1 <= 64 uses them)

__device__ __forceinline__ int nearest_level(const PyramidDesc& p, double sigma_rel) {
    // nearest_gauss_level (orient.cpp:13-24): strict < keeps the lower index on ties
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

__global__ void __launch_bounds__(kOriWarps * 32)
orient_kernel(const __grid_constant__ OrientArgs a) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    // atanf's 5-row reduction table in shared memory: the per-pixel row lookup
    // sits on the atan2f dependency chain (an LDS instead of a read-only-cache load)
    __shared__ __align__(16) uint32_t atan_tab[40];
    if (threadIdx.x < 40) atan_tab[threadIdx.x] = DS_ATAN_ROW_D[threadIdx.x];
    __syncthreads();
    const int bins = a.bins;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per-warp: union{ acc[bins][32] doubles (certified pass) | node[bins][depth]
    // doubles, count[bins], mask[bins], vals[32] (exact pass) } | hist[2][bins]
    const size_t exact_bytes = sizeof(double) * bins * a.depth + sizeof(unsigned) * bins * 2 + sizeof(float) * 32;
    const size_t acc_bytes = sizeof(double) * bins * 32;
    const size_t uni = ((exact_bytes > acc_bytes ? exact_bytes : acc_bytes) + 15) & ~size_t(15);
    const size_t per_warp_al = ((uni + sizeof(float) * 2 * bins + 15) & ~size_t(15)) + sizeof(double) * 2 * kOriAxis;
    unsigned char* wbase = sm_raw + warp * per_warp_al;
    double* acc = reinterpret_cast<double*>(wbase);
    double* node = reinterpret_cast<double*>(wbase);
    unsigned* cnt = reinterpret_cast<unsigned*>(node + bins * a.depth);
    unsigned* mask = cnt + bins;
    float* vals = reinterpret_cast<float*>(mask + bins);
    float* hist = reinterpret_cast<float*>(wbase + uni);
    float* hist2 = hist + bins;
    // per-axis window-weight factors exp(-d^2 / denom) for x and y
    double* wx = reinterpret_cast<double*>(wbase + ((uni + sizeof(float) * 2 * bins + 15) & ~size_t(15)));
    double* wy = wx + kOriAxis;
    // peaks go straight to global: angles[k][bins], counts[k] (K4b emits them)
    float* ang = a.angles;
    int* ncopy = a.counts;
    const long long n = a.n_host >= 0 ? a.n_host : (long long)*a.n_dev;
    // persistent: each warp claims keypoints one at a time from a global
    // ticket (a keypoint's window area scales with sigma^2, so fixed groups
    // would leave warps waiting for the slowest one)
    for (;;) {
        unsigned kt = 0;
        if (lane == 0) kt = atomicAdd(a.scan.ticket, 1u);
        const long long k = (long long)__shfl_sync(0xffffffffu, kt, 0);
        if (k >= n) break;
        const DevKeypoint kp = a.kps[k];
        if (kp.octave < 0) {   // a rejected candidate slot
            if (lane == 0) ncopy[k] = 0;
            continue;
        }
        const PyramidDesc& p = a.pyr;
        const OctaveDesc& od = p.oct[kp.octave];
        const double to_input = ldexp(1.0, kp.octave) * (p.upsampled ? 0.5 : 1.0);
        const double cx = kp.x / to_input, cy = kp.y / to_input;
        const double sigma_rel = kp.sigma / to_input;
        const int lvl = nearest_level(p, sigma_rel);
        const float* __restrict__ img = od.gauss + (long long)kp.image * p.gauss_img_stride(kp.octave) +
                                        (long long)lvl * od.level_stride;
        const int radius = (int)llround(3.0 * 1.5 * sigma_rel);
        const double denom = 2.0 * (1.5 * sigma_rel) * (1.5 * sigma_rel);
        const int x0 = (int)llround(cx), y0 = (int)llround(cy);
        const int ya = max(y0 - radius, 1), yb = min(y0 + radius, od.h - 2);
        const int xa = max(x0 - radius, 1), xb = min(x0 + radius, od.w - 2);
        const int nx = xb - xa + 1, ny = yb - ya + 1;
        const int npx = (nx > 0 && ny > 0) ? nx * ny : 0;

        const bool sep = nx <= kOriAxis && ny <= kOriAxis;
        if (sep) {
            for (int j = lane; j < nx; j += 32) {
                const double d = D_SUB((double)(xa + j), cx);
                wx[j] = dsift_exp_mid(D_DIV(-D_MUL(d, d), denom));
            }
            for (int j = lane; j < ny; j += 32) {
                const double d = D_SUB((double)(ya + j), cy);
                wy[j] = dsift_exp_mid(D_DIV(-D_MUL(d, d), denom));
            }
            __syncwarp();
        }
        // one window pixel q (row-major, orient.cpp:40-58): its bin and leaf value
        // q / nx without an integer division: exact for q < 2^20 (the window
        // is at most a few thousand pixels)
        const float inv_nx = 1.0f / (float)max(nx, 1);
        bool nan_seen = false;
        auto pixel = [&](int q, int& bin, float& val) {
            bin = -1;
            val = 0.0f;
            if (q < npx) {
                const int qy = (int)(((float)q + 0.5f) * inv_nx);
                const int x = xa + (q - qy * nx), y = ya + qy;
                DSIFT_BOUND(x >= 1 && x <= od.w - 2 && y >= 1 && y <= od.h - 2, 301);
                DSIFT_BOUND(!sep || (x - xa < nx && y - ya < ny && nx <= kOriAxis && ny <= kOriAxis), 302);
                const float* r0 = img + (long long)y * od.pitch;
                const float gx = F_SUB(__ldg(r0 + x + 1), __ldg(r0 + x - 1));
                const float gy = F_SUB(__ldg(r0 + od.pitch + x), __ldg(r0 - od.pitch + x));
                const float mag = F_SQRT(F_ADD(F_MUL(gx, gx), F_MUL(gy, gy)));
                const unsigned am = __activemask();   // the lanes of both votes below
                float theta = dsift_atan2f_mask(gy, gx, am, atan_tab);
                theta = (theta < 0.0f) ? F_ADD(theta, (float)kTwoPi) : theta;
                nan_seen |= isnan(theta);   // the reference's int(NaN) bin is out of range -> it throws
                theta = isnan(theta) ? 0.0f : theta;
                bin = (int)ds_div_2pi((double)F_MUL(theta, (float)bins));
                bin = (bin >= bins) ? bin - bins : bin;
                // float(exp(-(ddx^2 + ddy^2) / denom)) (orient.cpp:54-55) from the
                // per-axis factors, certified (|arg| <= 9: |P - D| <= 2^-48 D), else
                // evaluated as the reference does — warp-uniformly: the reference's
                // evaluation equals the certified product wherever that is proven
                float wgt;
                const bool wok = sep && ds_separable_weight<45>(D_MUL(wx[x - xa], wy[y - ya]), wgt);
                if (__any_sync(am, !wok)) {
                    const double ddx = D_SUB((double)x, cx), ddy = D_SUB((double)y, cy);
                    const double arg = D_DIV(-D_ADD(D_MUL(ddx, ddx), D_MUL(ddy, ddy)), denom);
                    wgt = (float)dsift_exp_mid(arg);
                }
                val = F_MUL(mag, wgt);
            }
        };

        // Certified pass: each lane sums its pixels' leaves per bin in FP64
        // (lane-private slots, no serialisation), the bins are folded over the
        // 32 lanes in a fixed order, and each bin's float is proven equal to
        // the reference's pairwise tree (detsum.cpp:19-31) by the exact-span or
        // rounding-interval test of the descriptor kernels.  Any unproven bin
        // sends the keypoint through the exact binary-counter pass below.
        for (int bb = 0; bb < bins; ++bb) acc[bb * 32 + lane] = 0.0;
        int emin = 1 << 20;   // lowest biased exponent of this lane's nonzero leaves
        for (int base = 0; base < npx; base += 32) {
            int bin;
            float val;
            pixel(base + lane, bin, val);
            if (bin >= 0) {
                DSIFT_BOUND(bin < bins, 303);
                double* slot = acc + bin * 32 + lane;
                *slot = *slot + (double)val;
                if (val > 0.0f) {
                    const int e = (int)((__float_as_uint(val) >> 23) & 0xffu);
                    emin = min(emin, e ? e : -22);
                }
            }
        }
        if (nan_seen) atomicOr(a.err, kErrHistogramRange);
#pragma unroll
        for (int d = 16; d; d >>= 1) emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, d));
        __syncwarp();
        bool ok = true;
        {
            const int steps = (npx + 31) / 32;
            const double e = (double)(steps + 32 + a.depth + 64) * 0x1p-53;
            for (int bb = lane; bb < bins; bb += 32) {
                double sum = 0.0;
                for (int l = 0; l < 32; ++l) sum = sum + acc[bb * 32 + l];
                const int top = (int)((__double_as_longlong(sum) >> 52) & 0x7ff) - 1023;
                float res;
                if (sum == 0.0 || top - (emin - 150) <= 52) {   // every partial sum exact
                    res = __double2float_rn(sum);
                } else {
                    res = __double2float_rn(sum * (1.0 - e));
                    ok = ok && (res == __double2float_rn(sum * (1.0 + e)));
                }
                hist[bb] = res;
            }
        }
        if (!__all_sync(0xffffffffu, ok)) {
            // exact pass: bins fed in scan order through binary-counter trees
            __syncwarp();
            for (int bb = lane; bb < bins; bb += 32) {
                cnt[bb] = 0;
                mask[bb] = 0;
            }
            __syncwarp();
            for (int base = 0; base < npx; base += 32) {
                int bin;
                float val;
                pixel(base + lane, bin, val);
                const unsigned grp = __match_any_sync(0xffffffffu, bin);
                if (bin >= 0 && lane == __ffs(grp) - 1) mask[bin] = grp;
                vals[lane] = val;
                __syncwarp();
                for (int bb = lane; bb < bins; bb += 32) {
                    unsigned m = mask[bb];
                    if (!m) continue;
                    mask[bb] = 0;
                    while (m) {
                        const int l = __ffs(m) - 1;
                        m &= m - 1;
                        tree_push_smem(node + bb * a.depth, &cnt[bb], (double)vals[l]);
                    }
                }
                __syncwarp();
            }
            for (int bb = lane; bb < bins; bb += 32)
                hist[bb] = (float)tree_result_smem(node + bb * a.depth, cnt[bb]);
        }
        __syncwarp();
        if (a.hist_out)
            for (int bb = lane; bb < bins; bb += 32) a.hist_out[k * bins + bb] = hist[bb];

        // smooth_histogram_circular, 2 passes (orient.cpp:62-75)
        float* cur = hist;
        float* nxt = hist2;
        for (int pass = 0; pass < 2; ++pass) {
            for (int bb = lane; bb < bins; bb += 32) {
                const double prev = cur[(bb + bins - 1) % bins], mid = cur[bb], succ = cur[(bb + 1) % bins];
                nxt[bb] = (float)(0.25 * prev + 0.5 * mid + 0.25 * succ);
            }
            __syncwarp();
            float* tmpp = cur;
            cur = nxt;
            nxt = tmpp;
        }
        // peaks (orient.cpp:77-113)
        float mx = 0.0f;
        for (int bb = lane; bb < bins; bb += 32) mx = fmaxf(mx, cur[bb]);
#pragma unroll
        for (int d = 16; d; d >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        int total = 0;
        if (mx > 0.0f) {
            const float gate = a.peak_ratio * mx;
            for (int chunk = 0; chunk < bins; chunk += 32) {
                const int bb = chunk + lane;
                bool pk = false;
                float angf = 0.0f;
                if (bb < bins) {
                    const float h0 = cur[bb], hm = cur[(bb + bins - 1) % bins], hp = cur[(bb + 1) % bins];
                    if (h0 > hm && h0 > hp && h0 >= gate) {
                        pk = true;
                        const double den = (double)hm - 2.0 * h0 + hp;
                        const double delta = den != 0.0 ? 0.5 * ((double)hm - hp) / den : 0.0;
                        double angle = (bb + delta) * kTwoPi / bins;
                        if (angle < 0.0) angle += kTwoPi;
                        if (angle >= kTwoPi) angle -= kTwoPi;
                        angf = (float)angle;
                        if (angf == 0.0f) angf = 0.0f;
                        if (angf >= (float)kTwoPi) angf = 0.0f;
                    }
                }
                const unsigned pm = __ballot_sync(0xffffffffu, pk);
                if (pk) ang[k * bins + total + __popc(pm & ((1u << lane) - 1u))] = angf;
                total += __popc(pm);
            }
        }
        if (total == 0) {
            if (lane == 0) ang[k * bins] = 0.0f;
            total = 1;
        }
        if (lane == 0) ncopy[k] = total;
        __syncwarp();
    }
}

// K4b: oriented copies in keypoint order (the reference's flattened
// per-candidate slots, io.cpp:117-125).  Tiles of 256 keypoints: a block scan
// of the copy counts plus a decoupled look-back over ticket-ordered tiles --
// uniform, tiny tiles, so the look-back never waits on heavy work.
__global__ void __launch_bounds__(256)
orient_emit_kernel(const __grid_constant__ OrientArgs a) {
    __shared__ unsigned ticket_s;
    __shared__ unsigned long long off_s;
    __shared__ int warp_tot[8];
    const long long n = a.n_host >= 0 ? a.n_host : (long long)*a.n_dev;
    const unsigned n_tiles = (unsigned)((n + 255) / 256);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        const unsigned t = scan_ticket(a.emit_scan, &ticket_s);
        if (t >= n_tiles) break;
        const long long k = (long long)t * 256 + threadIdx.x;
        const int c = k < n ? a.counts[k] : 0;
        int incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        int warp_off = 0, tile_total = 0;
        for (int wq = 0; wq < 8; ++wq) {
            if (wq < warp) warp_off += warp_tot[wq];
            tile_total += warp_tot[wq];
        }
        const unsigned long long off = scan_exclusive(a.emit_scan, t, (unsigned long long)tile_total, n_tiles, &off_s);
        if (threadIdx.x == 0 && (long long)(off + tile_total) > a.cap) atomicOr(a.err, kErrOrientedCapacity);
        if (c > 0) {
            const DevKeypoint kp = a.kps[k];
            const long long dst0 = (long long)off + warp_off + (incl - c);
            for (int i = 0; i < c; ++i) {
                if (dst0 + i >= a.cap) break;
                DevKeypoint cp = kp;
                cp.angle = a.angles[k * a.bins + i];
                a.out[dst0 + i] = cp;
            }
        }
        __syncthreads();
    }
}


size_t orient_smem_bytes(int bins, int depth) {
    const size_t exact_bytes = sizeof(double) * bins * depth + sizeof(unsigned) * bins * 2 + sizeof(float) * 32;
    const size_t acc_bytes = sizeof(double) * bins * 32;
    const size_t uni = ((exact_bytes > acc_bytes ? exact_bytes : acc_bytes) + 15) & ~size_t(15);
    const size_t per_warp_al = ((uni + sizeof(float) * 2 * bins + 15) & ~size_t(15)) + sizeof(double) * 2 * kOriAxis;
    return kOriWarps * per_warp_al;
}

cudaError_t launch_orient(const OrientArgs& a, cudaStream_t st) {
    if (a.n_tiles == 0) return cudaSuccess;
    const size_t smem = orient_smem_bytes(a.bins, a.depth);
    cudaError_t e = cudaFuncSetAttribute(orient_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, orient_kernel, kOriWarps * 32, smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<long long>((long long)a.n_tiles, (long long)sms * std::max(1, per_sm));
    orient_kernel<<<std::max(1u, grid), kOriWarps * 32, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const long long nk = (long long)a.n_tiles * kOriTile;
    const int grid2 = (int)std::max<long long>(1, std::min<long long>((nk + 255) / 256, (long long)sms * 8));
    orient_emit_kernel<<<grid2, 256, 0, st>>>(a);
    return cudaGetLastError();
}

int orient_tile_size() { return kOriTile; }

}  // namespace dsift
