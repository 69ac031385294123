// tests/native/libm_check.cpp — test helper: compares the product's libm
// restatements (paper_2605_17869_b200/csrc/dsift_math.cuh, compiled here as
// host code with -ffp-contract=off) against the live host glibc.  The same
// header is compiled into the CUDA kernels, so host-twin == glibc plus
// device == host-twin (checked in tests/test_gpu_parity.py) gives device ==
// glibc, the function the reference calls.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../paper_2605_17869_b200/csrc/dsift_math.cuh"

namespace {
struct Rng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uni() { return double(next() >> 11) * (1.0 / 9007199254740992.0); }
};

float bitsf(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
uint32_t fbits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}
uint64_t dbits(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
}
}  // namespace

extern "C" {

// mode 0: arbitrary finite float bit patterns (both signs, all exponents)
// mode 1: pipeline-shaped gradients: differences of two [0,1] floats, and
//         0.5f * difference (describe.cpp:84-85, orient.cpp:46-47)
// mode 2: special values (0, +-0, inf, nan, x == 1)
int64_t lc_atan2f_mismatch(uint64_t seed, int64_t n, int mode, float* first_bad /*[3]*/) {
    Rng r{seed};
    int64_t bad = 0;
    const float specials[] = {0.0f, -0.0f, 1.0f, -1.0f, INFINITY, -INFINITY, NAN, 1e-30f, 3e38f,
                              1e-45f, 0.5f, 2.4375f, 0.4375f, 1.1875f, 0.6875f};
    const int ns = sizeof(specials) / sizeof(float);
    for (int64_t i = 0; i < n; ++i) {
        float y, x;
        if (mode == 0) {
            do {
                y = bitsf(uint32_t(r.next()));
            } while (!std::isfinite(y));
            do {
                x = bitsf(uint32_t(r.next()));
            } while (!std::isfinite(x));
        } else if (mode == 1) {
            const float a = float(r.uni()), b = float(r.uni()), c = float(r.uni()),
                        d = float(r.uni());
            // scale the dynamic range like real pyramid levels (smooth areas -> tiny diffs)
            const float s = std::ldexp(1.0f, -int(r.next() % 20));
            y = (a - b) * s;
            x = (c - d) * s;
            if (r.next() & 1) {
                y = 0.5f * y;
                x = 0.5f * x;
            }
        } else {
            y = specials[r.next() % ns];
            x = specials[r.next() % ns];
        }
        const float ref = atan2f(y, x);
        const float got = dsift_atan2f(y, x);
        if (fbits(ref) != fbits(got) && !(std::isnan(ref) && std::isnan(got))) {
            if (bad == 0 && first_bad) {
                first_bad[0] = y;
                first_bad[1] = x;
                first_bad[2] = got;
            }
            ++bad;
        }
    }
    return bad;
}

// exp over [lo, hi] uniformly; mode 1 = arguments shaped like the pipeline's
// Gaussian weights: -(a^2 + b^2) / denom (orient.cpp:55, describe.cpp:97-98).
int64_t lc_exp_mismatch(uint64_t seed, int64_t n, double lo, double hi, int mode,
                        double* first_bad) {
    Rng r{seed};
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        double x;
        if (mode == 0) {
            x = lo + (hi - lo) * r.uni();
        } else {
            const double bw = 2.0 + 20.0 * r.uni();
            const int u = int(r.next() % 161) - 80, v = int(r.next() % 161) - 80;
            const double uu = u / bw, vv = v / bw;
            x = -(uu * uu + vv * vv) / 8.0;
        }
        const double ref = std::exp(x);
        // the branch-free window-weight variant must agree wherever it is used
        const double got = (x > -512.0 && x < 512.0 && (i & 1)) ? dsift_exp_mid(x) : dsift_exp(x);
        if (dbits(ref) != dbits(got)) {
            if (bad == 0 && first_bad) {
                first_bad[0] = x;
                first_bad[1] = got;
            }
            ++bad;
        }
    }
    return bad;
}

// cos/sin of float angles in [0, 2pi): returns double mismatches; *float_bad
// counts angles whose (float)(cx + cos*u) style sample coordinate would move
// (here: results that differ after rounding to float).
int64_t lc_sincos_mismatch(uint64_t seed, int64_t n, int64_t* float_bad) {
    // half float angles in [0, 2pi), half arbitrary doubles in [-8, 8)
    Rng r{seed};
    int64_t bad = 0, fb = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = (i & 1) ? double(float(r.uni() * 6.283185307179586)) : r.uni() * 16.0 - 8.0;
        double s, c;
        dsift_sincos(a, &s, &c);
        const double rs = std::sin(a), rc = std::cos(a);
        if (dbits(rs) != dbits(s) || dbits(rc) != dbits(c)) {
            ++bad;
            if (float(rs) != float(s) || float(rc) != float(c)) ++fb;
        }
    }
    if (float_bad) *float_bad = fb;
    return bad;
}

// Exhaustive: every float angle in [0, 2pi] (the domain describe.cpp:51-52
// feeds), split over `threads` host threads.
int64_t lc_sincos_exhaustive(int threads) {
    const uint32_t hi = fbits(6.2831855f);
    std::vector<int64_t> bad(threads, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (uint64_t u = t; u <= hi; u += threads) {
                const double a = bitsf(uint32_t(u));
                double s, c;
                dsift_sincos(a, &s, &c);
                if (dbits(std::sin(a)) != dbits(s) || dbits(std::cos(a)) != dbits(c)) ++bad[t];
            }
        });
    for (auto& th : pool) th.join();
    int64_t b = 0;
    for (int64_t x : bad) b += x;
    return b;
}

void lc_atan2f_batch(const float* y, const float* x, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = dsift_atan2f(y[i], x[i]);
}
void lc_exp_batch(const double* x, int64_t n, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = dsift_exp(x[i]);
}
void lc_sincos_batch(const double* a, int64_t n, double* s, double* c) {
    for (int64_t i = 0; i < n; ++i) dsift_sincos(a[i], &s[i], &c[i]);
}

}  // extern "C"

extern "C" {
// Exhaustive: ds_div_2pi(t) == t / (2pi) (IEEE) for every float t in [0, tmax].
int64_t lc_div2pi_mismatch(float tmax) {
    int64_t bad = 0;
    for (uint32_t u = 0;; ++u) {
        float t;
        std::memcpy(&t, &u, 4);
        if (!(t <= tmax)) break;
        const double td = (double)t;
        if (ds_div_2pi(td) != td / 6.283185307179586476925286766559) ++bad;
    }
    return bad;
}
}

extern "C" {
// ds_hypot vs glibc hypot: mode 0 pixel-scale coordinates (Hartley
// normalization inputs), mode 1 arbitrary finite doubles, mode 2 specials.
int64_t lc_hypot_mismatch(uint64_t seed, int64_t n, int mode, double* first_bad /*[3]*/) {
    Rng r{seed};
    int64_t bad = 0;
    const double specials[] = {0.0, -0.0, 1.0, -1.0, INFINITY, -INFINITY, NAN, 1e-320, 1.7e308,
                               0x1p-511, 0x1p511, 0x1p-600, 3.0, 4.0};
    const int ns = sizeof(specials) / sizeof(double);
    for (int64_t i = 0; i < n; ++i) {
        double x, y;
        if (mode == 0) {
            x = (r.uni() - 0.5) * 6000.0;
            y = (r.uni() - 0.5) * 6000.0;
            if (i % 3 == 1) y *= 1e-4;
            if (i % 7 == 2) x = y * (1.0 + r.uni() * 1e-9);
        } else if (mode == 1) {
            do {
                uint64_t u = r.next();
                std::memcpy(&x, &u, 8);
            } while (!std::isfinite(x));
            do {
                uint64_t u = r.next();
                std::memcpy(&y, &u, 8);
            } while (!std::isfinite(y));
        } else {
            x = specials[i % ns];
            y = specials[(i / ns) % ns];
        }
        const double g = std::hypot(x, y), m = ds_hypot(x, y);
        if (dbits(g) != dbits(m) && !(std::isnan(g) && std::isnan(m))) {
            if (bad == 0 && first_bad) {
                first_bad[0] = x;
                first_bad[1] = y;
                first_bad[2] = m;
            }
            ++bad;
        }
    }
    return bad;
}
}
