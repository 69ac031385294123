// k_match.cu — symmetric ratio-test matching on device descriptors
// (reference: match.cpp:19-119 ratio_match, tree_dot, scan_row).
//
// Every distance is the reference's float expression
//     sq = (|a|^2 + |b|^2) - 2 * tree_dot(a, b);  sq = max(sq, 0);  d = sqrtf(sq)
// where tree_dot rounds each of the 128 products to float and sums them with
// detsum's pairwise tree in double (detsum.cpp:19-31; 128 leaves = one complete
// dyadic tree), rounded to float once.  A thread owns a 2x2 block of (a, b)
// pairs of a 32x32 tile and builds each tree as eight-leaf subtrees folded by
// a register binary counter (the same tree).  The matrix is reduced both ways
// into (d1, index, d2) partials per tile, merged in index order with the
// reference's strict-< first-index-wins rule (scan_row, match.cpp:44-66).
#include <cuda_runtime.h>

#include "dsift_common.cuh"
#include "dsift_kernels.cuh"
#include "dsift_math.cuh"

namespace dsift {

constexpr int kMT = 32;        // tile edge (rows of A and of B)
constexpr int kDim = 128;

struct Top2 {
    float d1, d2;
    int idx;
};

// the ordered merge of two scan_row states: `l` covers lower indices than `r`
__device__ __forceinline__ Top2 top2_merge(const Top2& l, const Top2& r) {
    Top2 o;
    if (r.d1 < l.d1) {   // strict: an equal distance keeps the earlier index
        o.d1 = r.d1;
        o.idx = r.idx;
        o.d2 = (l.d1 < r.d2) ? l.d1 : r.d2;
    } else {
        o.d1 = l.d1;
        o.idx = l.idx;
        o.d2 = (r.d1 < l.d2) ? r.d1 : l.d2;
    }
    return o;
}

// |row|^2 as tree_dot(row, row): warp per row, lane holds leaves 4L..4L+3;
// the xor butterfly is the upper levels of the same dyadic tree.
__global__ void sqnorm_kernel(const float* __restrict__ d, long long n, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((long long)gridDim.x * blockDim.x) >> 5) {
        const float4 v = reinterpret_cast<const float4*>(d + r * kDim)[lane];
        double s = ((double)F_MUL(v.x, v.x) + (double)F_MUL(v.y, v.y)) +
                   ((double)F_MUL(v.z, v.z) + (double)F_MUL(v.w, v.w));
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) s = s + __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[r] = (float)s;
    }
}

// One 32x32 tile of the distance matrix and its row / column partials.
// row_part[i][tile_b] = scan of a_i over b in the tile (A->B), col_part[j][tile_a]
// = scan of b_j over a in the tile (B->A; the distance is symmetric).
__global__ void __launch_bounds__(256)
match_tile_kernel(const float* __restrict__ A, long long na, const float* __restrict__ B, long long nb,
                  const float* __restrict__ nA, const float* __restrict__ nB, Top2* __restrict__ row_part,
                  Top2* __restrict__ col_part, int tiles_a, int tiles_b) {
    __shared__ __align__(16) float sa[kMT][kDim + 4];
    __shared__ __align__(16) float sb[kMT][kDim + 4];
    __shared__ float dist[kMT][kMT + 1];
    const int ta = blockIdx.y, tb = blockIdx.x;
    const long long a0 = (long long)ta * kMT, b0 = (long long)tb * kMT;
    for (int i = threadIdx.x; i < kMT * kDim / 4; i += 256) {
        const int r = i / (kDim / 4), c = i - r * (kDim / 4);
        float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
        if (a0 + r < na) va = reinterpret_cast<const float4*>(A + (a0 + r) * kDim)[c];
        if (b0 + r < nb) vb = reinterpret_cast<const float4*>(B + (b0 + r) * kDim)[c];
        *reinterpret_cast<float4*>(&sa[r][4 * c]) = va;
        *reinterpret_cast<float4*>(&sb[r][4 * c]) = vb;
    }
    __syncthreads();
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // rows 2ty..2ty+1 of A, 2tx..2tx+1 of B
    double cnt[4][4];   // per pair: binary counter over the 16 eight-leaf subtrees (levels 4-7)
    double fin[4];
#pragma unroll
    for (int c = 0; c < kDim / 8; ++c) {
        float av[2][8], bv[2][8];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const float4 x0 = *reinterpret_cast<const float4*>(&sa[2 * ty + q][8 * c]);
            const float4 x1 = *reinterpret_cast<const float4*>(&sa[2 * ty + q][8 * c + 4]);
            const float4 y0 = *reinterpret_cast<const float4*>(&sb[2 * tx + q][8 * c]);
            const float4 y1 = *reinterpret_cast<const float4*>(&sb[2 * tx + q][8 * c + 4]);
            av[q][0] = x0.x; av[q][1] = x0.y; av[q][2] = x0.z; av[q][3] = x0.w;
            av[q][4] = x1.x; av[q][5] = x1.y; av[q][6] = x1.z; av[q][7] = x1.w;
            bv[q][0] = y0.x; bv[q][1] = y0.y; bv[q][2] = y0.z; bv[q][3] = y0.w;
            bv[q][4] = y1.x; bv[q][5] = y1.y; bv[q][6] = y1.z; bv[q][7] = y1.w;
        }
        // c is a compile-time constant here: the counter's merges are static
        const bool t1 = (c & 1) != 0, t2 = (c & 3) == 3, t3 = (c & 7) == 7, t4 = (c & 15) == 15;
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int qa = p >> 1, qb = p & 1;
            double l[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) l[k] = (double)F_MUL(av[qa][k], bv[qb][k]);   // float products (match.cpp:22)
            double x = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));   // levels 1-3
            if (t1) x = cnt[p][0] + x;   // earlier (left) subtree + this one
            if (t2) x = cnt[p][1] + x;
            if (t3) x = cnt[p][2] + x;
            if (t4) x = cnt[p][3] + x;
            if (!t1) cnt[p][0] = x;
            else if (!t2) cnt[p][1] = x;
            else if (!t3) cnt[p][2] = x;
            else if (!t4) cnt[p][3] = x;
            else fin[p] = x;
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int r = 2 * ty + (p >> 1), q = 2 * tx + (p & 1);
        const long long i = a0 + r, j = b0 + q;
        float d = __int_as_float(0x7fc00000);   // outside the sets: never a candidate
        if (i < na && j < nb) {
            const float dot = (float)fin[p];
            float sq = F_SUB(F_ADD(nA[i], nB[j]), F_MUL(2.0f, dot));   // match.cpp:51
            if (sq < 0.0f) sq = 0.0f;
            d = F_SQRT(sq);
        }
        dist[r][q] = d;
    }
    __syncthreads();
    // row scans (A->B) by threads 0..31, column scans (B->A) by threads 32..63
    if (threadIdx.x < 2 * kMT) {
        const bool rows = threadIdx.x < kMT;
        const int t = threadIdx.x & (kMT - 1);
        Top2 s{__int_as_float(0x7f800000), __int_as_float(0x7f800000), -1};
        for (int k = 0; k < kMT; ++k) {   // increasing index: scan_row's order
            const float d = rows ? dist[t][k] : dist[k][t];
            const int idx = (int)((rows ? b0 : a0) + k);
            if (d < s.d1) {
                s.d2 = s.d1;
                s.d1 = d;
                s.idx = idx;
            } else if (d < s.d2) {
                s.d2 = d;
            }
        }
        if (rows) {
            if (a0 + t < na) row_part[(a0 + t) * tiles_b + tb] = s;
        } else {
            if (b0 + t < nb) col_part[(b0 + t) * tiles_a + ta] = s;
        }
    }
}

// Merge each row's tile partials in tile order, then the ratio test
// (match.cpp:96-108): best[i] = index if d1 < ratio * d2, else -1.
__global__ void match_reduce_kernel(const Top2* __restrict__ part, long long n, int tiles, float ratio,
                                    int* __restrict__ best, float* __restrict__ dist) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        Top2 s = part[i * tiles];
        for (int t = 1; t < tiles; ++t) s = top2_merge(s, part[i * tiles + t]);
        const bool pass = s.idx >= 0 && s.d1 < F_MUL(ratio, s.d2);
        best[i] = pass ? s.idx : -1;
        if (dist) dist[i] = pass ? s.d1 : 0.0f;
    }
}

size_t match_scratch_bytes(long long na, long long nb) {
    const long long ta = (na + kMT - 1) / kMT, tb = (nb + kMT - 1) / kMT;
    return sizeof(float) * (size_t)(na + nb) + sizeof(Top2) * (size_t)(na * tb + nb * ta) +
           sizeof(int) * (size_t)(na + nb) + sizeof(float) * (size_t)na + 1024;
}

cudaError_t launch_ratio_match(const float* A, long long na, const float* B, long long nb, float ratio, void* scratch,
                               int* best_a, int* best_b, float* dist_a, cudaStream_t st) {
    const int ta = (int)((na + kMT - 1) / kMT), tb = (int)((nb + kMT - 1) / kMT);
    char* p = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    float* nA = reinterpret_cast<float*>(take(sizeof(float) * na));
    float* nB = reinterpret_cast<float*>(take(sizeof(float) * nb));
    Top2* rp = reinterpret_cast<Top2*>(take(sizeof(Top2) * (size_t)na * tb));
    Top2* cp = reinterpret_cast<Top2*>(take(sizeof(Top2) * (size_t)nb * ta));
    sqnorm_kernel<<<(int)std::min<long long>((na * 32 + 255) / 256, 148LL * 16), 256, 0, st>>>(A, na, nA);
    sqnorm_kernel<<<(int)std::min<long long>((nb * 32 + 255) / 256, 148LL * 16), 256, 0, st>>>(B, nb, nB);
    match_tile_kernel<<<dim3(tb, ta), 256, 0, st>>>(A, na, B, nb, nA, nB, rp, cp, ta, tb);
    match_reduce_kernel<<<(int)std::max<long long>(1, std::min<long long>((na + 255) / 256, 148LL * 8)), 256, 0, st>>>(
        rp, na, tb, ratio, best_a, dist_a);
    match_reduce_kernel<<<(int)std::max<long long>(1, std::min<long long>((nb + 255) / 256, 148LL * 8)), 256, 0, st>>>(
        cp, nb, ta, ratio, best_b, nullptr);
    return cudaGetLastError();
}

}  // namespace dsift
