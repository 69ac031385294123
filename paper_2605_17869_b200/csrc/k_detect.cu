// k_detect.cu — K2+K3: scale-space extrema, Taylor refinement, contrast and
// edge rejection, deterministic compaction (reference: detect.cpp:11-172).
//
// One launch covers every (image, octave, 32x32 tile) of the batch.  A tile
// stages all s+2 DoG levels (+1-pixel halo) in shared memory once, tests the
// strict 26-neighbour extremum on levels 1..s with the float pre-gate
// |v| > 0.5f*ct/s (detect.cpp:35-36), refines each candidate in place with the
// reference's FP64 Cramer solve (no FMA contraction: this file is compiled
// with -fmad=false) and emits accepted keypoints through a warp-shuffle block
// scan plus a decoupled look-back over ticket-ordered tiles.  Output order is
// (image, octave, tile, thread, level, row) — fixed by construction, no
// atomics on order; canonical order is restored later by the sort (K7).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_scan.cuh"
#include "dsift_tma.cuh"

namespace dsift {

DSIFT_BOUNDS_UNIT(detect)

constexpr int kDetTile = 32;
constexpr int kDetThreads = 256;
constexpr int kDetHalo = kDetTile + 2;
constexpr int kDetPitch = 36;   // staged row pitch (floats): 16-byte aligned rows

// refine_extremum (detect.cpp:73-156), bit-exact FP64 restatement.
__device__ bool refine_candidate(const DetectArgs& a, int b, int o, int x, int y, int i,
                                 DevKeypoint* kp) {
    const OctaveDesc& od = a.pyr.oct[o];
    const int s = a.pyr.s, w = od.w, h = od.h, pitch = od.pitch;
    const float* __restrict__ dogb = od.dog + (long long)b * a.pyr.dog_img_stride(o);
    const long long ls = od.level_stride;
#define DAT(L, X, Y) ((double)__ldg(dogb + (long long)(L) * ls + (long long)(Y) * pitch + (X)))
    double dx = 0, dy = 0, ds = 0, gx = 0, gy = 0, gs = 0, dxx = 0, dyy = 0, dxy = 0;
    bool converged = false;
    for (int it = 0; it < a.max_iters; ++it) {
        const double v = DAT(i, x, y);
        gx = 0.5 * (DAT(i, x + 1, y) - DAT(i, x - 1, y));
        gy = 0.5 * (DAT(i, x, y + 1) - DAT(i, x, y - 1));
        gs = 0.5 * (DAT(i + 1, x, y) - DAT(i - 1, x, y));
        dxx = DAT(i, x + 1, y) + DAT(i, x - 1, y) - 2.0 * v;
        dyy = DAT(i, x, y + 1) + DAT(i, x, y - 1) - 2.0 * v;
        const double dss = DAT(i + 1, x, y) + DAT(i - 1, x, y) - 2.0 * v;
        dxy = 0.25 * (DAT(i, x + 1, y + 1) - DAT(i, x - 1, y + 1) - DAT(i, x + 1, y - 1) +
                      DAT(i, x - 1, y - 1));
        const double dxs = 0.25 * (DAT(i + 1, x + 1, y) - DAT(i + 1, x - 1, y) -
                                   DAT(i - 1, x + 1, y) + DAT(i - 1, x - 1, y));
        const double dys = 0.25 * (DAT(i + 1, x, y + 1) - DAT(i + 1, x, y - 1) -
                                   DAT(i - 1, x, y + 1) + DAT(i - 1, x, y - 1));
        const double det = dxx * (dyy * dss - dys * dys) - dxy * (dxy * dss - dys * dxs) +
                           dxs * (dxy * dys - dyy * dxs);
        if (fabs(det) < 1e-12) return false;
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
            converged = true;
            break;
        }
        if (dx > 0.5) ++x; else if (dx < -0.5) --x;
        if (dy > 0.5) ++y; else if (dy < -0.5) --y;
        if (ds > 0.5) ++i; else if (ds < -0.5) --i;
        if (x < 1 || x >= w - 1 || y < 1 || y >= h - 1 || i < 1 || i > s) return false;
    }
    if (!converged) return false;
    const double value = DAT(i, x, y) + 0.5 * (gx * dx + gy * dy + gs * ds);
#undef DAT
    if (fabs(value) < a.contrast_gate) return false;
    const double tr = dxx + dyy;
    const double det2 = dxx * dyy - dxy * dxy;
    const double r = a.edge_r;
    if (det2 <= 0.0 || tr * tr * r >= det2 * (r + 1.0) * (r + 1.0)) return false;
    const double to_input = ldexp(1.0, o) * (a.pyr.upsampled ? 0.5 : 1.0);
    kp->x = (float)((x + dx) * to_input);
    kp->y = (float)((y + dy) * to_input);
    kp->sigma = (float)(a.pyr.sigma0 * pow(2.0, o + (i + ds) / s) * (a.pyr.upsampled ? 0.5 : 1.0));
    kp->angle = 0.0f;
    kp->response = (float)fabs(value);
    kp->octave = o;
    kp->interval = i;
    kp->image = b;
    return true;
}

// K2a: one CTA per (image, octave, 32x32 tile) in a fixed tile order; every
// thread records which of its (level, row) positions are extrema as a 12-bit
// mask and the tile publishes its count.  No tile ever waits on another.
// kS > 0: intervals known at compile time (the level loop unrolls and the
// sliding window lives in renamed registers); kS = 0: any s.
template <int kS>
__global__ void __launch_bounds__(kDetThreads, 5)   // 5 CTAs/SM: swept 3 / 4 / 5 / 6 -> 2.80 / 2.57 / 2.49 / 2.82 ms
detect_count_kernel(const __grid_constant__ DetectArgs a) {
    extern __shared__ __align__(128) float lv_raw[];
    // [s+2][34][kDetPitch], 128-byte aligned (TMA destination)
    // 128-byte aligned TMA destination, offset from the array itself so every
    // access stays in the shared window (LDS, not generic LD)
    float* lv_s = lv_raw + (((128u - (smem_u32(lv_raw) & 127u)) & 127u) >> 2);
    __shared__ int warp_tot[kDetThreads / 32];
    const unsigned t = blockIdx.x;
    const int b = (int)(t / a.tiles_per_image);
    const int rr = (int)(t % a.tiles_per_image);
    int o = 0;
    while (o + 1 < a.pyr.n_oct && a.oct_tile_base[o + 1] <= rr) ++o;
    const OctaveDesc& od = a.pyr.oct[o];
    const int tile = rr - a.oct_tile_base[o];
    const int xs = 1 + (tile % od.tiles_x) * kDetTile;
    const int ys = 1 + (tile / od.tiles_x) * kDetTile;
    const int s = kS > 0 ? kS : a.pyr.s, w = od.w, h = od.h;
    const int nlev = s + 2;
    const int lane = threadIdx.x & 31;

    if ((a.tma_mask >> o) & 1u) {
        // one TMA box {36, 34, s+2} of the DoG stack: 34 rows (tile + halo) x
        // 36 columns from xs - 1 of each level; out-of-image elements arrive
        // as zeros, exactly like the copy path below
        __shared__ __align__(8) uint64_t bar;
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            mbar_arrive_expect_tx(&bar, (unsigned)(sizeof(float) * kDetPitch * kDetHalo * nlev));
            tma_load_3d(lv_s, &a.dog_maps[o], xs - 1, ys - 1, b * nlev, &bar);
        }
        __syncthreads();
        mbar_wait(&bar, 0);
    } else {
        // stage s+2 DoG levels (+1 halo) with asynchronous 4-byte copies: every
        // load is in flight at once (a load->store chain per row serialises on
        // memory latency); out-of-image positions are zero-filled
        const float* __restrict__ dogb = od.dog + (long long)b * a.pyr.dog_img_stride(o);
        // a staged row = 32 aligned floats (8 x 16 B, xs - 1 = 32k) + 2 halo floats
        for (int idx = threadIdx.x; idx < nlev * kDetHalo * 10; idx += kDetThreads) {
            const int r = idx / 10, q = idx - r * 10;
            const int l = r / kDetHalo, yy = ys - 1 + (r - l * kDetHalo);
            const int xx = xs - 1 + (q < 8 ? 4 * q : 24 + q);   // q = 8, 9 -> columns 32, 33
            const int cols = q < 8 ? 4 : 1;
            const int nin = yy < h ? max(0, min(cols, w - xx)) : 0;
            const float* g = dogb + (nin ? (long long)l * od.level_stride + (long long)yy * od.pitch + xx : 0);
            const unsigned sa = (unsigned)__cvta_generic_to_shared(lv_s + r * kDetPitch + (xx - (xs - 1)));
            if (q < 8)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(4 * nin));
            else
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(g), "r"(4 * nin));
        }
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
    }

    // strictly_extremal (detect.cpp:11-28), branch-free: thread (lane, g) owns
    // column lane and the 4 rows 4g..4g+3 of the tile.  Per level it keeps the
    // max / min of each 3-pixel row segment of rows 4g-1..4g+4; a candidate's
    // 26-neighbour max is max(its level's 8 neighbours, the 3x3 of the levels
    // above and below), v > that (is_max) or v < the min (fmaxf/fminf ignore a
    // NaN neighbour exactly like the reference's failed comparisons).
    const int lx = lane, g = threadIdx.x >> 5;
    float hx[3][6], hn[3][6];         // row-segment max / min of levels i-1, i, i+1
    float cc[4], cl[4], cr[4];        // level i: centre, left, right of rows 4g..4g+3
    auto load_level = [&](int l, float (&mx)[6], float (&mn)[6], bool keep_centre) {
        const float* base = lv_s + (l * kDetHalo + 4 * g) * kDetPitch + lx;
        DSIFT_BOUND(l < nlev && 4 * g + 6 <= kDetHalo && lx + 3 <= kDetPitch, 201);
#pragma unroll
        for (int r = 0; r < 6; ++r) {
            const float a0 = base[r * kDetPitch], a1 = base[r * kDetPitch + 1], a2 = base[r * kDetPitch + 2];
            mx[r] = fmaxf(fmaxf(a0, a1), a2);
            mn[r] = fminf(fminf(a0, a1), a2);
            if (keep_centre && r >= 1 && r <= 4) {
                cl[r - 1] = a0;
                cc[r - 1] = a1;
                cr[r - 1] = a2;
            }
        }
    };
    unsigned hits = 0;
    load_level(0, hx[0], hn[0], false);
    load_level(1, hx[1], hn[1], true);
    const int x = xs + lx;
#pragma unroll (kS > 0 ? kS : 1)
    for (int i = 1; i <= s; ++i) {
        load_level(i + 1, hx[2], hn[2], false);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = q + 1;   // row in the 6-row window
            const float v = cc[q];
            const float m8 = fmaxf(fmaxf(hx[1][r - 1], hx[1][r + 1]), fmaxf(cl[q], cr[q]));
            const float n8 = fminf(fminf(hn[1][r - 1], hn[1][r + 1]), fminf(cl[q], cr[q]));
            const float mo = fmaxf(fmaxf(fmaxf(hx[0][r - 1], hx[0][r]), hx[0][r + 1]),
                                   fmaxf(fmaxf(hx[2][r - 1], hx[2][r]), hx[2][r + 1]));
            const float no = fminf(fminf(fminf(hn[0][r - 1], hn[0][r]), hn[0][r + 1]),
                                   fminf(fminf(hn[2][r - 1], hn[2][r]), hn[2][r + 1]));
            const bool ext = (v > 0.0f) ? (v > fmaxf(m8, mo)) : (v < fminf(n8, no));
            const int y = ys + 4 * g + q;
            // float pre-gate |v| > 0.5 * ct / s (detect.cpp:35); interior pixels only
            const bool hit = ext && (fabsf(v) > a.pre_gate) && x <= w - 2 && y <= h - 2;
            hits |= (hit ? 1u : 0u) << ((i - 1) * 4 + q);
        }
        if (i < s) {   // slide the level window: i -> i-1, i+1 -> i (+ its centres)
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                hx[0][r] = hx[1][r];
                hn[0][r] = hn[1][r];
                hx[1][r] = hx[2][r];
                hn[1][r] = hn[2][r];
            }
            const float* base = lv_s + ((i + 1) * kDetHalo + 4 * g) * kDetPitch + lx;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                cl[q] = base[(q + 1) * kDetPitch];
                cc[q] = base[(q + 1) * kDetPitch + 1];
                cr[q] = base[(q + 1) * kDetPitch + 2];
            }
        }
    }
    a.hit_masks[(size_t)t * kDetThreads + threadIdx.x] = hits;
    int cnt = __popc(hits);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if (lane == 0) warp_tot[g] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int wq = 0; wq < kDetThreads / 32; ++wq) tot += warp_tot[wq];
        a.tile_counts[t] = (unsigned)tot;
    }
}

// K2b (after the device-wide scan of the tile counts, k_sort.cu): candidates
// of tile t go to [tile_offsets[t], +count) in (thread, level,
// row) order -- the same deterministic order as a single-pass look-back.  One
// warp per tile (8 tiles per CTA): lane j replays count-kernel threads 8j..8j+7.
__global__ void __launch_bounds__(256)
detect_emit_kernel(const __grid_constant__ DetectArgs a) {
    const int lane = threadIdx.x & 31;
    const unsigned t = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (t >= a.n_tiles) return;
    const unsigned cnt_t = a.tile_counts[t];
    const unsigned long long tile_off = a.tile_offsets[t];
    if (t == a.n_tiles - 1 && lane == 0) {
        const unsigned long long total = tile_off + cnt_t;
        if ((long long)total > a.cap) atomicOr(a.err, kErrCandidateCapacity);
        *a.scan.total = min(total, (unsigned long long)a.cap);   // never more than was written
    }
    if (cnt_t == 0) return;
    const int b = (int)(t / a.tiles_per_image);
    const int rr = (int)(t % a.tiles_per_image);
    int o = 0;
    while (o + 1 < a.pyr.n_oct && a.oct_tile_base[o + 1] <= rr) ++o;
    const OctaveDesc& od = a.pyr.oct[o];
    const int tile = rr - a.oct_tile_base[o];
    const int xs = 1 + (tile % od.tiles_x) * kDetTile;
    const int ys = 1 + (tile / od.tiles_x) * kDetTile;
    const uint4* mp = reinterpret_cast<const uint4*>(a.hit_masks + (size_t)t * kDetThreads) + 2 * lane;
    const uint4 ma = mp[0], mb = mp[1];
    const unsigned mw[8] = {ma.x, ma.y, ma.z, ma.w, mb.x, mb.y, mb.z, mb.w};   // count threads 8j..8j+7
    int count = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) count += __popc(mw[k]);
    int incl = count;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int nb = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += nb;
    }
    unsigned long long slot = tile_off + (incl - count);
    const float* __restrict__ dogb = od.dog + (long long)b * a.pyr.dog_img_stride(o);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int th = lane * 8 + k;                 // the count kernel's thread index
        const int lx = th & 31, g = th >> 5;
        unsigned hits = mw[k];
        while (hits) {
            const int bit = __ffs(hits) - 1;
            hits &= hits - 1;
            const int i = 1 + (bit >> 2), q = bit & 3;
            const int x = xs + lx, y = ys + 4 * g + q;
            if ((long long)slot < a.cap) {
                const float v = __ldg(dogb + (long long)i * od.level_stride + (long long)y * od.pitch + x);
                DevCandidate c = {b, o, i, y, x, v > 0.0f ? 1 : 0};
                a.cand_out[slot] = c;
            }
            ++slot;
        }
    }
}

// K3 as its own pass: one thread per candidate (every lane busy, refinement
// runs once), tiles of 256 candidates in ticket order; survivors are
// compacted with a block scan + decoupled look-back, so they keep the
// candidate order (detect.cpp:158-172) and the orientation stage only sees
// real keypoints.  keep[c] (optional, stage API) records each verdict.
__global__ void __launch_bounds__(256)
refine_kernel(const __grid_constant__ DetectArgs a, const DevCandidate* __restrict__ cand,
              const unsigned long long* n_cand, int* keep) {
    __shared__ unsigned ticket_s;
    __shared__ unsigned long long off_s;
    __shared__ int warp_tot[8];
    const long long n = (long long)*n_cand;
    const unsigned n_tiles = (unsigned)((n + 255) / 256);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        const unsigned t = scan_ticket(a.scan, &ticket_s);
        if (t >= n_tiles) break;
        const long long c = (long long)t * 256 + threadIdx.x;
        DevKeypoint kp;
        bool ok = false;
        if (c < n) {
            const DevCandidate e = cand[c];
            ok = refine_candidate(a, e.image, e.octave, e.col, e.row, e.interval, &kp);
            if (keep) keep[c] = ok ? 1 : 0;
        }
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        if (lane == 0) warp_tot[warp] = __popc(m);
        __syncthreads();
        int warp_off = 0, tile_total = 0;
        for (int wq = 0; wq < 8; ++wq) {
            if (wq < warp) warp_off += warp_tot[wq];
            tile_total += warp_tot[wq];
        }
        const unsigned long long off = scan_exclusive(a.scan, t, (unsigned long long)tile_total, n_tiles, &off_s);
        if (ok) {
            const unsigned long long slot = off + warp_off + __popc(m & ((1u << lane) - 1u));
            if ((long long)slot < a.cap) a.out[slot] = kp;
        }
        if (threadIdx.x == 0 && (long long)(off + tile_total) > a.cap) atomicOr(a.err, kErrKeypointCapacity);
        __syncthreads();
    }
}

cudaError_t launch_refine(const DetectArgs& a, const DevCandidate* cand, const unsigned long long* n_cand,
                          long long cap, int* keep, cudaStream_t st) {
    const int grid = (int)std::max<long long>(1, std::min<long long>((cap + 255) / 256, 148 * 8));
    refine_kernel<<<grid, 256, 0, st>>>(a, cand, n_cand, keep);
    return cudaGetLastError();
}

cudaError_t launch_detect(const DetectArgs& a, cudaStream_t st) {
    if (a.n_tiles == 0) return cudaSuccess;
    const size_t smem = sizeof(float) * (size_t)(a.pyr.s + 2) * kDetHalo * kDetPitch + 128;
    void (*fn)(DetectArgs) = a.pyr.s == 3 ? detect_count_kernel<3> : detect_count_kernel<0>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<a.n_tiles, kDetThreads, smem, st>>>(a);
    e = launch_scan_u32(a.tile_counts, a.tile_offsets, (long long)a.n_tiles, a.scan_state, nullptr, st);
    if (e != cudaSuccess) return e;
    detect_emit_kernel<<<(a.n_tiles + 7) / 8, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace dsift
