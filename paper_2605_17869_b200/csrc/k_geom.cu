// k_geom.cu — MAGSAC-lite homography estimation on the device
// (reference: geom.cpp:104-161 dlt_homography, :181-320 magsac_lite,
// linalg.cpp:9-93 jacobi_eigen_sym).
//
// The host draws the hypothesis samples from the seeded SplitMix64 stream
// (geom.cpp:193-232, sequential by definition).  The device then
//   G1  one warp per hypothesis: normalized 4-point DLT (Hartley scaling,
//       A^T A, cyclic Jacobi sweeps with the rotations' row updates spread
//       over the lanes, smallest eigenvector), det / inverse checks;
//   G2  one CTA per hypothesis: the soft truncated-quadratic terms of every
//       correspondence and their detsum tree sum (detsum.cpp:19-71);
//   G3  one CTA: the winner (score descending, iteration ascending), the soft
//       inliers of the winner (ordered compaction), the weighted DLT refit
//       (order-defining sums sequential, elementwise work parallel, A^T A
//       entries owned by 45 threads in the reference's row order, Jacobi on
//       one warp) and the final inlier mask.
// Every floating-point expression is the reference's, evaluated in the same
// order in IEEE binary64 (no contraction: built with -fmad=false); std::hypot
// is glibc's algorithm (ds_hypot).  Results are bit-identical to the
// reference (tests/test_geom.py).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_math.cuh"

namespace dsift {

namespace {

constexpr int kG2Threads = 128;
constexpr int kG3Threads = 256;

// Homography::det (geom.cpp:22-25)
__device__ __forceinline__ double h_det(const double* h) {
    return h[0] * (h[4] * h[8] - h[5] * h[7]) - h[1] * (h[3] * h[8] - h[5] * h[6]) +
           h[2] * (h[3] * h[7] - h[4] * h[6]);
}

// Homography::normalize (geom.cpp:40-51)
__device__ __forceinline__ void h_normalize(double* h) {
    if (fabs(h[8]) > 1e-12) {
        const double inv = 1.0 / h[8];
        for (int i = 0; i < 9; ++i) h[i] *= inv;
        return;
    }
    double norm = 0.0;
    for (int i = 0; i < 9; ++i) norm += h[i] * h[i];
    norm = ds_sqrt_d(norm);
    if (norm > 0.0)
        for (int i = 0; i < 9; ++i) h[i] /= norm;
}

// Homography::inverse (geom.cpp:27-38); false where the reference throws
__device__ __forceinline__ bool h_inverse(const double* h, double* inv) {
    const double d = h_det(h);
    if (fabs(d) < 1e-15) return false;
    inv[0] = (h[4] * h[8] - h[5] * h[7]) / d;
    inv[1] = (h[2] * h[7] - h[1] * h[8]) / d;
    inv[2] = (h[1] * h[5] - h[2] * h[4]) / d;
    inv[3] = (h[5] * h[6] - h[3] * h[8]) / d;
    inv[4] = (h[0] * h[8] - h[2] * h[6]) / d;
    inv[5] = (h[2] * h[3] - h[0] * h[5]) / d;
    inv[6] = (h[3] * h[7] - h[4] * h[6]) / d;
    inv[7] = (h[1] * h[6] - h[0] * h[7]) / d;
    inv[8] = (h[0] * h[4] - h[1] * h[3]) / d;
    h_normalize(inv);
    return true;
}

// symmetric_error_sq (geom.cpp:167-179)
__device__ __forceinline__ double sym_err_sq(const double* h, const double* hi, double x1, double y1, double x2,
                                             double y2) {
    const double wf = h[6] * x1 + h[7] * y1 + h[8];
    const double wb = hi[6] * x2 + hi[7] * y2 + hi[8];
    if (fabs(wf) < 1e-12 || fabs(wb) < 1e-12) return __longlong_as_double(0x7ff0000000000000LL);
    const double fx = (h[0] * x1 + h[1] * y1 + h[2]) / wf - x2;
    const double fy = (h[3] * x1 + h[4] * y1 + h[5]) / wf - y2;
    const double bx = (hi[0] * x2 + hi[1] * y2 + hi[2]) / wb - x1;
    const double by = (hi[3] * x2 + hi[4] * y2 + hi[5]) / wb - y1;
    return fx * fx + fy * fy + bx * bx + by * by;
}

// std::max(0.0, 1.0 - r2 / tau_sq) (geom.cpp:254)
__device__ __forceinline__ double soft_term(double r2, double tau_sq) {
    const double t = 1.0 - r2 / tau_sq;
    return (0.0 < t) ? t : 0.0;
}

// jacobi_eigen_sym on a 9x9 row-major symmetric matrix (linalg.cpp:9-93),
// one warp: every lane forms the rotation scalars (same operations, same
// values), lane k < 9 then updates row / column k of A and lane 16 + k row k
// of V.  Within one rotation no lane reads an element another lane writes
// (A(k,p), A(k,q) belong to lane k; lane p owns the 2x2 block), so the result
// is the reference's sequential sweep.  Writes the eigenvector of the smallest
// eigenvalue (row 8 of the result, sign-normalized) to hn.  a, v: shared [81].
__device__ void jacobi9_smallest_warp(double* a, double* v, double* hn) {
    const int n = 9;
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < 81; i += 32) v[i] = (i % 10 == 0) ? 1.0 : 0.0;
    __syncwarp();
    double norm = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) norm += a[i * n + j] * a[i * n + j];
    norm = ds_sqrt_d(norm);
    const double tol = norm > 0.0 ? norm * 1e-15 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
        if (ds_sqrt_d(2.0 * off) <= tol) break;
        for (int p = 0; p < n - 1; ++p) {
            for (int q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (apq == 0.0) continue;
                const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + ds_sqrt_d(theta * theta + 1.0));
                const double c = 1.0 / ds_sqrt_d(t * t + 1.0);
                const double s = t * c;
                const double tau = s / (1.0 + c);
                const double app = a[p * n + p], aqq = a[q * n + q];
                double akp = 0.0, akq = 0.0, vkp = 0.0, vkq = 0.0;
                const int k = lane & 15;
                if (lane < 9 && k != p && k != q) {
                    akp = a[k * n + p];
                    akq = a[k * n + q];
                } else if (lane >= 16 && k < 9) {
                    vkp = v[k * n + p];
                    vkq = v[k * n + q];
                }
                __syncwarp();
                if (lane < 9) {
                    if (k == p) {
                        a[p * n + p] = app - t * apq;
                        a[q * n + q] = aqq + t * apq;
                        a[p * n + q] = 0.0;
                        a[q * n + p] = 0.0;
                    } else if (k != q) {
                        const double nkp = akp - s * (akq + tau * akp);
                        const double nkq = akq + s * (akp - tau * akq);
                        a[k * n + p] = nkp;
                        a[p * n + k] = nkp;
                        a[k * n + q] = nkq;
                        a[q * n + k] = nkq;
                    }
                } else if (lane >= 16 && k < 9) {
                    v[k * n + p] = vkp - s * (vkq + tau * vkp);
                    v[k * n + q] = vkq + s * (vkp - tau * vkq);
                }
                __syncwarp();
            }
        }
    }
    // stable descending order of the diagonal (std::stable_sort): the last
    // entry is the smallest, ties resolved toward the higher original index
    int order[9];
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int k = 1; k < n; ++k) {
        const int key = order[k];
        int j = k - 1;
        while (j >= 0 && a[key * n + key] > a[order[j] * n + order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = key;
    }
    const int col = order[n - 1];
    int arg = 0;
    double best = -1.0;
    for (int r = 0; r < n; ++r) {
        const double m = fabs(v[r * n + col]);
        if (m > best) {
            best = m;
            arg = r;
        }
    }
    const double sign = v[arg * n + col] < 0.0 ? -1.0 : 1.0;
    if (lane < n) hn[lane] = sign * v[lane * n + col];
    __syncwarp();
}

struct NormT {
    double scale, cx, cy;
};

// hartley_normalize (geom.cpp:68-94) over already-gathered coordinates; false
// where the reference throws (coincident points).  xs / ys are normalized in
// place.
__device__ bool hartley(double* xs, double* ys, int n, NormT& t) {
    double sx = 0.0, sy = 0.0;
    for (int i = 0; i < n; ++i) {
        sx += xs[i];
        sy += ys[i];
    }
    t.cx = sx / (double)n;
    t.cy = sy / (double)n;
    double mean_dist = 0.0;
    for (int i = 0; i < n; ++i) mean_dist += ds_hypot(xs[i] - t.cx, ys[i] - t.cy);
    mean_dist /= (double)n;
    if (mean_dist < 1e-12) return false;
    t.scale = ds_sqrt_d(2.0) / mean_dist;
    for (int i = 0; i < n; ++i) {
        xs[i] = (xs[i] - t.cx) * t.scale;
        ys[i] = (ys[i] - t.cy) * t.scale;
    }
    return true;
}

// three_collinear (geom.cpp:96-106)
__device__ bool three_collinear(const double* xs, const double* ys, int n) {
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j)
            for (int k = j + 1; k < n; ++k) {
                const double area = (xs[j] - xs[i]) * (ys[k] - ys[i]) - (xs[k] - xs[i]) * (ys[j] - ys[i]);
                if (fabs(area) < 1e-9) return true;
            }
    return false;
}

// The two DLT rows of correspondence (x, y) -> (u, v) with weight w (geom.cpp:130-131).
__device__ __forceinline__ void dlt_rows(double w, double x, double y, double u, double v, double (&r1)[9],
                                         double (&r2)[9]) {
    r1[0] = 0; r1[1] = 0; r1[2] = 0;
    r1[3] = -w * x; r1[4] = -w * y; r1[5] = -w;
    r1[6] = w * v * x; r1[7] = w * v * y; r1[8] = w * v;
    r2[0] = w * x; r2[1] = w * y; r2[2] = w;
    r2[3] = 0; r2[4] = 0; r2[5] = 0;
    r2[6] = -w * u * x; r2[7] = -w * u * y; r2[8] = -w * u;
}

// Denormalize + normalize + finiteness (geom.cpp:137-160) from hn.
__device__ bool dlt_finish(const double* hn, const NormT& ts, const NormT& td, double* out) {
    const double tsrc[9] = {ts.scale, 0, -ts.scale * ts.cx, 0, ts.scale, -ts.scale * ts.cy, 0, 0, 1};
    const double tdi[9] = {1.0 / td.scale, 0, td.cx, 0, 1.0 / td.scale, td.cy, 0, 0, 1};
    double m1[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += tdi[r * 3 + k] * hn[k * 3 + c];
            m1[r * 3 + c] = acc;
        }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
            for (int k = 0; k < 3; ++k) acc += m1[r * 3 + k] * tsrc[k * 3 + c];
            out[r * 3 + c] = acc;
        }
    h_normalize(out);
    for (int i = 0; i < 9; ++i)
        if (!isfinite(out[i])) return false;
    return true;
}

// G1: minimal-sample model of every hypothesis (geom.cpp:236-252), one warp
// per hypothesis: lane 0 normalizes the 4 points, the lanes own A^T A
// entries, the warp runs the Jacobi sweeps, lane 0 denormalizes and checks.
constexpr int kG1Warps = 4;
__global__ void __launch_bounds__(32 * kG1Warps) magsac_hyp_kernel(const double* __restrict__ m,
                                                                   const int4* __restrict__ samples, int iters,
                                                                   double* __restrict__ models,
                                                                   unsigned char* __restrict__ valid) {
    __shared__ double sa[kG1Warps][81], sv[kG1Warps][81], shn[kG1Warps][9], spts[kG1Warps][16];
    __shared__ NormT sts[kG1Warps], std_[kG1Warps];
    __shared__ int sok[kG1Warps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it = blockIdx.x * kG1Warps + w;
    if (it >= iters) return;   // warp-uniform
    double* a = sa[w];
    double* pts = spts[w];   // sx[4], sy[4], dx[4], dy[4], normalized
    if (lane == 0) {
        int ok = 0;
        const int4 s = samples[it];
        if (s.x >= 0) {
            const int idx[4] = {s.x, s.y, s.z, s.w};
            for (int k = 0; k < 4; ++k) {
                pts[k] = m[4 * idx[k] + 0];
                pts[4 + k] = m[4 * idx[k] + 1];
                pts[8 + k] = m[4 * idx[k] + 2];
                pts[12 + k] = m[4 * idx[k] + 3];
            }
            NormT ts, td;
            ok = hartley(pts, pts + 4, 4, ts) && hartley(pts + 8, pts + 12, 4, td) &&
                 !three_collinear(pts, pts + 4, 4) && !three_collinear(pts + 8, pts + 12, 4);
            sts[w] = ts;
            std_[w] = td;
        }
        sok[w] = ok;
    }
    __syncwarp();
    if (!sok[w]) {
        if (lane == 0) valid[it] = 0;
        return;
    }
    for (int e = lane; e < 45; e += 32) {   // entry (p, q), q >= p: rows in the reference's order
        int p = 0, r = e;
        while (r >= 9 - p) {
            r -= 9 - p;
            ++p;
        }
        const int q = p + r;
        double acc = 0.0;
        for (int i = 0; i < 4; ++i) {
            double r1[9], r2[9];
            dlt_rows(1.0, pts[i], pts[4 + i], pts[8 + i], pts[12 + i], r1, r2);
            acc += r1[p] * r1[q];
            acc += r2[p] * r2[q];
        }
        a[p * 9 + q] = acc;
        a[q * 9 + p] = acc;
    }
    __syncwarp();
    jacobi9_smallest_warp(a, sv[w], shn[w]);
    if (lane == 0) {
        double h[9], hi[9];
        bool ok = dlt_finish(shn[w], sts[w], std_[w], h);
        if (ok) {
            const double det = h_det(h);
            ok = isfinite(det) && det != 0.0 && h_inverse(h, hi);
        }
        if (ok)
            for (int i = 0; i < 9; ++i) {
                models[18 * it + i] = h[i];
                models[18 * it + 9 + i] = hi[i];
            }
        valid[it] = ok ? 1 : 0;
    }
}

// Binary counter over aligned 2^level blocks (the detsum tree; see dsift_tree.cuh).
struct LevelCounter {
    double node[40];
    unsigned long long count;
    __device__ void push(double x, int level) {
        unsigned long long c = count >> level;
        int j = level;
        while (c & 1ull) {
            x = node[j] + x;
            c >>= 1;
            ++j;
        }
        node[j] = x;
        count += 1ull << level;
    }
    __device__ double result() const {
        double r = 0.0;
        bool have = false;
        for (int j = 0; (count >> j) != 0ull; ++j)
            if ((count >> j) & 1ull) {
                r = have ? node[j] + r : node[j];
                have = true;
            }
        return r;
    }
};

// G2: score of every valid hypothesis (geom.cpp:253-258).  Each warp sums
// aligned 32-term blocks with the xor butterfly (exactly the tree's top of a
// complete 32-leaf subtree); thread 0 feeds the block sums, then the partial
// tail, into the counter in leaf order.
__global__ void __launch_bounds__(kG2Threads) magsac_score_kernel(const double* __restrict__ m, long long n,
                                                                  const double* __restrict__ models,
                                                                  const unsigned char* __restrict__ valid,
                                                                  double tau_sq, double* __restrict__ scores,
                                                                  double* __restrict__ block_sums) {
    const int it = blockIdx.x;
    if (!valid[it]) {
        if (threadIdx.x == 0) scores[it] = -1.0;
        return;
    }
    __shared__ double h[18];
    __shared__ double tail[32];
    if (threadIdx.x < 18) h[threadIdx.x] = models[18 * it + threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long nfull = n >> 5;
    double* bs = block_sums + (long long)it * ((n >> 5) + 1);
    for (long long b = warp; b <= nfull; b += kG2Threads / 32) {
        const long long i = (b << 5) + lane;
        double t = 0.0;
        if (i < n) t = soft_term(sym_err_sq(h, h + 9, m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]), tau_sq);
        if (b < nfull) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) t = t + __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) bs[b] = t;
        } else if (i < n) {
            tail[lane] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        LevelCounter tc;
        tc.count = 0ull;
        for (long long b = 0; b < nfull; ++b) tc.push(bs[b], 5);
        const int rem = (int)(n & 31);
        for (int k = 0; k < rem; ++k) tc.push(tail[k], 0);
        scores[it] = tc.result();
    }
}

// Weighted normalized DLT of n correspondences (geom.cpp:108-161) by one CTA
// of kG3Threads: the order-defining sums (centroids, mean distances) are
// sequential loops of one thread each; everything elementwise is parallel;
// A^T A entries are owned by 45 threads; the Jacobi sweeps run on warp 0.
// x1..y2: global scratch holding the raw coordinates (normalized in place);
// hs, ht: scratch [n].  Returns (to every thread) whether the reference
// would have returned a model; out = H on success.
struct DltShared {
    double ata[81], jv[81], hn[9];
    NormT ts, td;
    double sum[4];
    int ok;
};
__device__ bool dlt_cta(DltShared& S, double* x1, double* y1, double* x2, double* y2, const double* w, int n,
                        double* hs, double* ht, double* out) {
    const int tid = threadIdx.x;
    if (tid == 0) S.ok = 1;
    if (tid == 0 || tid == 32) {   // hartley_normalize (geom.cpp:68-94): centroid sums
        const double* xs = tid == 0 ? x1 : x2;
        const double* ys = tid == 0 ? y1 : y2;
        double sx = 0.0, sy = 0.0;
        for (int i = 0; i < n; ++i) {
            sx += xs[i];
            sy += ys[i];
        }
        NormT& t = tid == 0 ? S.ts : S.td;
        t.cx = sx / (double)n;
        t.cy = sy / (double)n;
    }
    __syncthreads();
    for (int i = tid; i < n; i += kG3Threads) {
        hs[i] = ds_hypot(x1[i] - S.ts.cx, y1[i] - S.ts.cy);
        ht[i] = ds_hypot(x2[i] - S.td.cx, y2[i] - S.td.cy);
    }
    __syncthreads();
    if (tid == 0 || tid == 32) {
        const double* hh = tid == 0 ? hs : ht;
        NormT& t = tid == 0 ? S.ts : S.td;
        double mean_dist = 0.0;
        for (int i = 0; i < n; ++i) mean_dist += hh[i];
        mean_dist /= (double)n;
        if (mean_dist < 1e-12) atomicAnd(&S.ok, 0);
        t.scale = ds_sqrt_d(2.0) / mean_dist;
    }
    __syncthreads();
    if (!S.ok) return false;
    for (int i = tid; i < n; i += kG3Threads) {
        x1[i] = (x1[i] - S.ts.cx) * S.ts.scale;
        y1[i] = (y1[i] - S.ts.cy) * S.ts.scale;
        x2[i] = (x2[i] - S.td.cx) * S.td.scale;
        y2[i] = (y2[i] - S.td.cy) * S.td.scale;
    }
    __syncthreads();
    if (tid == 0 && n == 4 && (three_collinear(x1, y1, 4) || three_collinear(x2, y2, 4))) S.ok = 0;
    if (tid < 45) {
        int p = 0, e = tid;
        while (e >= 9 - p) {
            e -= 9 - p;
            ++p;
        }
        const int q = p + e;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
            double r1[9], rr[9];
            dlt_rows(w ? w[i] : 1.0, x1[i], y1[i], x2[i], y2[i], r1, rr);
            acc += r1[p] * r1[q];
            acc += rr[p] * rr[q];
        }
        S.ata[p * 9 + q] = acc;
        S.ata[q * 9 + p] = acc;
    }
    __syncthreads();
    if (!S.ok) return false;
    if (tid < 32) {
        jacobi9_smallest_warp(S.ata, S.jv, S.hn);
        if (tid == 0) S.ok = dlt_finish(S.hn, S.ts, S.td, out);
    }
    __syncthreads();
    return S.ok != 0;
}

// G3: winner, soft inliers, weighted refit, final mask (geom.cpp:261-319).
// out_i: [0] success, [1] best iteration; out_d: [0] score, [1..9] H.
// scratch (device): r2, x1, y1, x2, y2, w, hs, ht — 8 n doubles.
__global__ void __launch_bounds__(kG3Threads) magsac_final_kernel(const double* __restrict__ m, long long n, int iters,
                                                                  const double* __restrict__ models,
                                                                  const unsigned char* __restrict__ valid,
                                                                  const double* __restrict__ scores, double tau_sq,
                                                                  double* __restrict__ scratch,
                                                                  unsigned char* __restrict__ mask,
                                                                  int* __restrict__ out_i, double* __restrict__ out_d) {
    __shared__ DltShared D;
    __shared__ double h[9], hi[9], refit[9], refit_inv[9];
    __shared__ double wsc[kG3Threads / 32];
    __shared__ int wix[kG3Threads / 32], cnt[kG3Threads];
    __shared__ int best_s, ok_s, nin_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* r2 = scratch;
    double* x1 = r2 + n;
    double* y1 = x1 + n;
    double* x2 = y1 + n;
    double* y2 = x2 + n;
    double* wt = y2 + n;
    double* hs = wt + n;
    double* ht = hs + n;
    // winner: highest score, lowest iteration on ties (geom.cpp:263-268)
    double bs = 0.0;
    int bi = -1;
    for (int it = tid; it < iters; it += kG3Threads)
        if (valid[it] && (bi < 0 || scores[it] > bs)) {
            bs = scores[it];
            bi = it;
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double os = __shfl_down_sync(0xffffffffu, bs, o);
        const int oi = __shfl_down_sync(0xffffffffu, bi, o);
        if (oi >= 0 && (bi < 0 || os > bs || (os == bs && oi < bi))) {
            bs = os;
            bi = oi;
        }
    }
    if (lane == 0) {
        wsc[warp] = bs;
        wix[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
        int best = -1;
        double b = 0.0;
        for (int k = 0; k < kG3Threads / 32; ++k)
            if (wix[k] >= 0 && (best < 0 || wsc[k] > b || (wsc[k] == b && wix[k] < best))) {
                b = wsc[k];
                best = wix[k];
            }
        best_s = best;
        out_i[0] = 0;
        out_i[1] = best;
        out_d[0] = 0.0;
        int ok = 0;
        if (best >= 0) {
            for (int i = 0; i < 9; ++i) h[i] = models[18 * best + i];
            ok = h_inverse(h, hi) ? 1 : 0;   // the winner's inverse, as the reference recomputes it
        }
        ok_s = ok;
    }
    __syncthreads();
    if (!ok_s) {
        for (long long i = tid; i < n; i += kG3Threads) mask[i] = 0;
        return;
    }
    // soft inliers in index order (geom.cpp:276-283): per-thread contiguous chunks
    const long long chunk = (n + kG3Threads - 1) / kG3Threads;
    const long long c0 = tid * chunk, c1 = min(n, c0 + chunk);
    int c = 0;
    for (long long i = c0; i < c1; ++i) {
        const double e = sym_err_sq(h, hi, m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]);
        r2[i] = e;
        c += e < tau_sq;
    }
    cnt[tid] = c;
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < kG3Threads; ++k) {
            const int v = cnt[k];
            cnt[k] = acc;
            acc += v;
        }
        nin_s = acc;
    }
    __syncthreads();
    {
        int k = cnt[tid];
        for (long long i = c0; i < c1; ++i)
            if (r2[i] < tau_sq) {
                x1[k] = m[4 * i];
                y1[k] = m[4 * i + 1];
                x2[k] = m[4 * i + 2];
                y2[k] = m[4 * i + 3];
                wt[k] = 1.0 - r2[i] / tau_sq;
                ++k;
            }
    }
    __syncthreads();
    const int nin = nin_s;
    bool ok = nin >= 4 && dlt_cta(D, x1, y1, x2, y2, wt, nin, hs, ht, refit);
    if (ok) {
        if (tid == 0) {
            ok_s = h_inverse(refit, refit_inv) ? 1 : 0;
            if (ok_s) {
                out_i[0] = 1;
                out_d[0] = scores[best_s];
                for (int i = 0; i < 9; ++i) out_d[1 + i] = refit[i];
            }
        }
        __syncthreads();
        ok = ok_s != 0;
    }
    for (long long i = tid; i < n; i += kG3Threads) {
        unsigned char v = 0;
        if (ok) v = sym_err_sq(refit, refit_inv, m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]) < tau_sq;
        mask[i] = v;
    }
}

// Standalone weighted DLT (geom.cpp:108-161) for the C ABI: one CTA, the
// refit's code path.  status: 1 ok, 0 where the reference throws.
// scratch: x1, y1, x2, y2, hs, ht — 6 n doubles.
__global__ void __launch_bounds__(kG3Threads) dlt_kernel(const double* __restrict__ m, const double* __restrict__ w,
                                                         int n, double* __restrict__ scratch, int* __restrict__ status,
                                                         double* __restrict__ out) {
    __shared__ DltShared D;
    double* x1 = scratch;
    double* y1 = x1 + n;
    double* x2 = y1 + n;
    double* y2 = x2 + n;
    for (int i = threadIdx.x; i < n; i += kG3Threads) {
        x1[i] = m[4 * i];
        y1[i] = m[4 * i + 1];
        x2[i] = m[4 * i + 2];
        y2[i] = m[4 * i + 3];
    }
    __syncthreads();
    const bool ok = dlt_cta(D, x1, y1, x2, y2, w, n, y2 + n, y2 + 2 * (long long)n, out);
    if (threadIdx.x == 0) *status = ok ? 1 : 0;
}

}  // namespace

size_t magsac_scratch_bytes(long long n, int iters) {
    return sizeof(double) * 18 * (size_t)iters + (size_t)iters + 256 + sizeof(double) * (size_t)iters +
           sizeof(double) * (size_t)iters * (size_t)((n >> 5) + 1) + sizeof(double) * 8 * (size_t)n + 2048;
}

cudaError_t launch_magsac(const double* m, long long n, const int4* samples, int iters, double tau_sq, void* scratch,
                          unsigned char* mask, int* out_i, double* out_d, cudaStream_t st) {
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    double* models = reinterpret_cast<double*>(take(sizeof(double) * 18 * (size_t)iters));
    unsigned char* valid = reinterpret_cast<unsigned char*>(take((size_t)iters));
    double* scores = reinterpret_cast<double*>(take(sizeof(double) * (size_t)iters));
    double* bsums = reinterpret_cast<double*>(take(sizeof(double) * (size_t)iters * (size_t)((n >> 5) + 1)));
    double* fscr = reinterpret_cast<double*>(take(sizeof(double) * 8 * (size_t)n));
    magsac_hyp_kernel<<<(iters + kG1Warps - 1) / kG1Warps, 32 * kG1Warps, 0, st>>>(m, samples, iters, models, valid);
    magsac_score_kernel<<<iters, kG2Threads, 0, st>>>(m, n, models, valid, tau_sq, scores, bsums);
    magsac_final_kernel<<<1, kG3Threads, 0, st>>>(m, n, iters, models, valid, scores, tau_sq, fscr, mask, out_i,
                                                  out_d);
    return cudaGetLastError();
}

size_t dlt_scratch_bytes(long long n) { return sizeof(double) * 6 * (size_t)n + 256; }

cudaError_t launch_dlt(const double* m, const double* w, int n, void* scratch, int* status, double* out,
                       cudaStream_t st) {
    dlt_kernel<<<1, kG3Threads, 0, st>>>(m, w, n, static_cast<double*>(scratch), status, out);
    return cudaGetLastError();
}

}  // namespace dsift
