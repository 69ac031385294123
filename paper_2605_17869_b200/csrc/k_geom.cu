// k_geom.cu — MAGSAC-lite homography estimation on the device
// (reference: geom.cpp:104-161 dlt_homography, :181-320 magsac_lite,
// linalg.cpp:9-93 jacobi_eigen_sym).
//
// The host draws the hypothesis samples from the seeded SplitMix64 stream
// (geom.cpp:193-232, sequential by definition).  The device then
//   G1  one thread per hypothesis: normalized 4-point DLT (Hartley scaling,
//       A^T A, cyclic Jacobi, smallest eigenvector), det / inverse checks;
//   G2  one CTA per hypothesis: the soft truncated-quadratic terms of every
//       correspondence and their detsum tree sum (detsum.cpp:19-71);
//   G3  one CTA: the winner (score descending, iteration ascending), the soft
//       inliers of the winner, the weighted DLT refit (A^T A entries owned by
//       45 threads, each summed in the reference's row order) and the final
//       inlier mask.
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

// jacobi_eigen_sym on a 9x9 row-major symmetric matrix (linalg.cpp:9-93);
// writes the eigenvector of the smallest eigenvalue (row 8 of the result,
// sign-normalized) to hn.  One thread; a and v are scratch [81].
__device__ void jacobi9_smallest(double* a, double* v, double* hn) {
    const int n = 9;
    for (int i = 0; i < 81; ++i) v[i] = 0.0;
    for (int i = 0; i < n; ++i) v[i * n + i] = 1.0;
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
                a[p * n + p] = app - t * apq;
                a[q * n + q] = aqq + t * apq;
                a[p * n + q] = 0.0;
                a[q * n + p] = 0.0;
                for (int k = 0; k < n; ++k) {
                    if (k == p || k == q) continue;
                    const double akp = a[k * n + p], akq = a[k * n + q];
                    a[k * n + p] = akp - s * (akq + tau * akp);
                    a[p * n + k] = a[k * n + p];
                    a[k * n + q] = akq + s * (akp - tau * akq);
                    a[q * n + k] = a[k * n + q];
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = v[k * n + p], vkq = v[k * n + q];
                    v[k * n + p] = vkp - s * (vkq + tau * vkp);
                    v[k * n + q] = vkq + s * (vkp - tau * vkq);
                }
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
    for (int r = 0; r < n; ++r) hn[r] = sign * v[r * n + col];
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

// One A^T A row update (geom.cpp:122-126): ata[p][q] += row[p] * row[q], q >= p.
__device__ __forceinline__ void ata_add_row(double* ata, const double (&row)[9]) {
    for (int p = 0; p < 9; ++p)
        for (int q = p; q < 9; ++q) ata[p * 9 + q] += row[p] * row[q];
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

// G1: minimal-sample model of every hypothesis (geom.cpp:236-252).
__global__ void __launch_bounds__(64) magsac_hyp_kernel(const double* __restrict__ m, const int4* __restrict__ samples,
                                                        int iters, double* __restrict__ models,
                                                        unsigned char* __restrict__ valid) {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= iters) return;
    valid[it] = 0;
    const int4 s = samples[it];
    if (s.x < 0) return;
    const int idx[4] = {s.x, s.y, s.z, s.w};
    double sx[4], sy[4], dx[4], dy[4];
    for (int k = 0; k < 4; ++k) {
        sx[k] = m[4 * idx[k] + 0];
        sy[k] = m[4 * idx[k] + 1];
        dx[k] = m[4 * idx[k] + 2];
        dy[k] = m[4 * idx[k] + 3];
    }
    // copies of the raw target coordinates (rows use the normalized ones)
    NormT ts, td;
    if (!hartley(sx, sy, 4, ts) || !hartley(dx, dy, 4, td)) return;
    if (three_collinear(sx, sy, 4) || three_collinear(dx, dy, 4)) return;
    double a[81], v[81];
    for (int i = 0; i < 81; ++i) a[i] = 0.0;
    for (int i = 0; i < 4; ++i) {
        double r1[9], r2[9];
        dlt_rows(1.0, sx[i], sy[i], dx[i], dy[i], r1, r2);
        ata_add_row(a, r1);
        ata_add_row(a, r2);
    }
    for (int p = 0; p < 9; ++p)
        for (int q = 0; q < p; ++q) a[p * 9 + q] = a[q * 9 + p];
    double hn[9], h[9], hi[9];
    jacobi9_smallest(a, v, hn);
    if (!dlt_finish(hn, ts, td, h)) return;
    const double det = h_det(h);
    if (!isfinite(det) || det == 0.0) return;
    if (!h_inverse(h, hi)) return;
    for (int i = 0; i < 9; ++i) {
        models[18 * it + i] = h[i];
        models[18 * it + 9 + i] = hi[i];
    }
    valid[it] = 1;
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

struct G3Shared {
    double h[9], hi[9], refit[9], refit_inv[9];
    NormT ts, td;
    int best;
    int n_in;
    int ok;
};

// G3: winner, soft inliers, weighted refit, final mask (geom.cpp:261-319).
// out: [0] status (1 = success), [1] best iteration, then score (double) and
// h[9] in out_d.  Scratch (device, 7 n doubles): r2, inlier x1 y1 x2 y2, w.
__global__ void __launch_bounds__(kG3Threads) magsac_final_kernel(const double* __restrict__ m, long long n, int iters,
                                                                  const double* __restrict__ models,
                                                                  const unsigned char* __restrict__ valid,
                                                                  const double* __restrict__ scores, double tau_sq,
                                                                  double* __restrict__ scratch,
                                                                  unsigned char* __restrict__ mask,
                                                                  int* __restrict__ out_i, double* __restrict__ out_d) {
    __shared__ G3Shared S;
    __shared__ double ata[81];
    __shared__ double jv[81];
    __shared__ double hn[9];
    const int tid = threadIdx.x;
    double* r2 = scratch;
    double* ix1 = scratch + n;
    double* iy1 = ix1 + n;
    double* ix2 = iy1 + n;
    double* iy2 = ix2 + n;
    double* iw = iy2 + n;
    if (tid == 0) {
        int best = -1;
        for (int it = 0; it < iters; ++it) {
            if (!valid[it]) continue;
            if (best < 0 || scores[it] > scores[best]) best = it;
        }
        S.best = best;
        S.ok = 0;
        out_i[0] = 0;
        out_i[1] = best;
        out_d[0] = 0.0;
        if (best >= 0) {
            for (int i = 0; i < 9; ++i) S.h[i] = models[18 * best + i];
            // the winner's inverse is recomputed as the reference does (geom.cpp:270-274)
            S.ok = h_inverse(S.h, S.hi) ? 1 : 0;
        }
    }
    __syncthreads();
    if (!S.ok) {
        for (long long i = tid; i < n; i += kG3Threads) mask[i] = 0;
        return;
    }
    for (long long i = tid; i < n; i += kG3Threads)
        r2[i] = sym_err_sq(S.h, S.hi, m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]);
    __syncthreads();
    if (tid == 0) {   // ordered compaction of the soft inliers (geom.cpp:276-283)
        int k = 0;
        for (long long i = 0; i < n; ++i)
            if (r2[i] < tau_sq) {
                ix1[k] = m[4 * i];
                iy1[k] = m[4 * i + 1];
                ix2[k] = m[4 * i + 2];
                iy2[k] = m[4 * i + 3];
                iw[k] = 1.0 - r2[i] / tau_sq;
                ++k;
            }
        S.n_in = k;
        S.ok = k >= 4;
    }
    __syncthreads();
    if (!S.ok) {
        for (long long i = tid; i < n; i += kG3Threads) mask[i] = 0;
        return;
    }
    const int nin = S.n_in;
    // Hartley normalization of both sides: sequential sums (threads 0 and 32)
    if (tid == 0 || tid == 32) {
        double* xs = tid == 0 ? ix1 : ix2;
        double* ys = tid == 0 ? iy1 : iy2;
        NormT t;
        const bool ok = hartley(xs, ys, nin, t);
        if (tid == 0) S.ts = t; else S.td = t;
        if (!ok) atomicAnd(&S.ok, 0);
    }
    __syncthreads();
    if (!S.ok) {
        for (long long i = tid; i < n; i += kG3Threads) mask[i] = 0;
        return;
    }
    if (nin == 4 && tid == 0) {   // geom.cpp:116-118 (only for a 4-point refit)
        if (three_collinear(ix1, iy1, 4) || three_collinear(ix2, iy2, 4)) S.ok = 0;
    }
    // A^T A: thread e < 45 owns entry (p, q), q >= p, summed over the rows in order
    if (tid < 45) {
        int p = 0, e = tid;
        while (e >= 9 - p) {
            e -= 9 - p;
            ++p;
        }
        const int q = p + e;
        double acc = 0.0;
        for (int i = 0; i < nin; ++i) {
            double r1[9], rr[9];
            dlt_rows(iw[i], ix1[i], iy1[i], ix2[i], iy2[i], r1, rr);
            acc += r1[p] * r1[q];
            acc += rr[p] * rr[q];
        }
        ata[p * 9 + q] = acc;
        ata[q * 9 + p] = acc;
    }
    __syncthreads();
    if (tid == 0 && S.ok) {
        jacobi9_smallest(ata, jv, hn);
        bool ok = dlt_finish(hn, S.ts, S.td, S.refit);
        if (ok) ok = h_inverse(S.refit, S.refit_inv);
        S.ok = ok;
        if (ok) {
            out_i[0] = 1;
            out_d[0] = scores[S.best];
            for (int i = 0; i < 9; ++i) out_d[1 + i] = S.refit[i];
        }
    }
    __syncthreads();
    for (long long i = tid; i < n; i += kG3Threads) {
        unsigned char v = 0;
        if (S.ok) v = sym_err_sq(S.refit, S.refit_inv, m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]) < tau_sq;
        mask[i] = v;
    }
}

// Standalone weighted DLT (geom.cpp:108-161) for the C ABI: one CTA, the same
// code path as the refit.  status: 1 ok, 0 degenerate.
__global__ void __launch_bounds__(kG3Threads) dlt_kernel(const double* __restrict__ m, const double* __restrict__ w,
                                                         int n, double* __restrict__ scratch, int* __restrict__ status,
                                                         double* __restrict__ out) {
    __shared__ double ata[81];
    __shared__ double jv[81];
    __shared__ double hn[9];
    __shared__ NormT ts, td;
    __shared__ int ok;
    const int tid = threadIdx.x;
    double* x1 = scratch;
    double* y1 = x1 + n;
    double* x2 = y1 + n;
    double* y2 = x2 + n;
    if (tid == 0) ok = 1;
    for (int i = tid; i < n; i += kG3Threads) {
        x1[i] = m[4 * i];
        y1[i] = m[4 * i + 1];
        x2[i] = m[4 * i + 2];
        y2[i] = m[4 * i + 3];
    }
    __syncthreads();
    if (tid == 0 || tid == 32) {
        NormT t;
        const bool good = tid == 0 ? hartley(x1, y1, n, t) : hartley(x2, y2, n, t);
        if (tid == 0) ts = t; else td = t;
        if (!good) atomicAnd(&ok, 0);
    }
    __syncthreads();
    if (tid == 0 && ok && n == 4 && (three_collinear(x1, y1, 4) || three_collinear(x2, y2, 4))) ok = 0;
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
        ata[p * 9 + q] = acc;
        ata[q * 9 + p] = acc;
    }
    __syncthreads();
    if (tid == 0) {
        int good = ok;
        if (good) {
            jacobi9_smallest(ata, jv, hn);
            good = dlt_finish(hn, ts, td, out);
        }
        *status = good;
    }
}

}  // namespace

size_t magsac_scratch_bytes(long long n, int iters) {
    return sizeof(double) * 18 * (size_t)iters + (size_t)iters + 256 + sizeof(double) * (size_t)iters +
           sizeof(double) * (size_t)iters * (size_t)((n >> 5) + 1) + sizeof(double) * 7 * (size_t)n + 1024;
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
    double* fscr = reinterpret_cast<double*>(take(sizeof(double) * 6 * (size_t)n));
    magsac_hyp_kernel<<<(iters + 63) / 64, 64, 0, st>>>(m, samples, iters, models, valid);
    magsac_score_kernel<<<iters, kG2Threads, 0, st>>>(m, n, models, valid, tau_sq, scores, bsums);
    magsac_final_kernel<<<1, kG3Threads, 0, st>>>(m, n, iters, models, valid, scores, tau_sq, fscr, mask, out_i,
                                                  out_d);
    return cudaGetLastError();
}

size_t dlt_scratch_bytes(long long n) { return sizeof(double) * 4 * (size_t)n + 256; }

cudaError_t launch_dlt(const double* m, const double* w, int n, void* scratch, int* status, double* out,
                       cudaStream_t st) {
    dlt_kernel<<<1, kG3Threads, 0, st>>>(m, w, n, static_cast<double*>(scratch), status, out);
    return cudaGetLastError();
}

}  // namespace dsift
