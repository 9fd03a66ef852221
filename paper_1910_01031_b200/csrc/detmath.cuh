// detmath.cuh -- counter-based RNG and deterministic elementary functions (device).
//
// Included only by translation units compiled with --fmad=false, so every double
// expression below is evaluated as written with IEEE round-to-nearest and no FMA
// contraction. The functions use only +,-,*,/,sqrt,floor and bit manipulation, which
// makes them reproducible bit-for-bit by any IEEE implementation of the same
// definition -- in particular by the CPU checker in oracle/.
#pragma once

#include <cstdint>

namespace dcg {
namespace det {

// stream_seed (rng.hpp:25-40): three splitmix64 rounds over (master, tag, index)
__host__ __device__ inline uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__host__ __device__ inline uint64_t stream_key(uint64_t master, uint64_t tag, uint64_t index) {
    uint64_t s = splitmix(master ^ 0x8000000000000000ull);
    s = splitmix(s ^ tag);
    return splitmix(s ^ (index + 0x51ed2700a1b4c2d3ull));
}

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of the 4x32 bijection.
__device__ __forceinline__ uint4 philox(uint4 c, uint64_t key) {
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
    return c;
}

__device__ __forceinline__ double ln_det(double x) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    int e = static_cast<int>((b >> 52) & 0x7ff) - 1023;
    double m = __longlong_as_double(
        static_cast<long long>((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
    if (m > 1.41421356237309514547e+00) {
        m = m * 0.5;
        e = e + 1;
    }
    const double f = m - 1.0;
    const double s = f / (2.0 + f);
    const double z = s * s;
    double q = 1.0 / 27.0;
    q = q * z + 1.0 / 25.0;
    q = q * z + 1.0 / 23.0;
    q = q * z + 1.0 / 21.0;
    q = q * z + 1.0 / 19.0;
    q = q * z + 1.0 / 17.0;
    q = q * z + 1.0 / 15.0;
    q = q * z + 1.0 / 13.0;
    q = q * z + 1.0 / 11.0;
    q = q * z + 1.0 / 9.0;
    q = q * z + 1.0 / 7.0;
    q = q * z + 1.0 / 5.0;
    q = q * z + 1.0 / 3.0;
    const double two_s = 2.0 * s;
    const double lm = two_s + two_s * (z * q);
    const double de = static_cast<double>(e);
    return de * 6.93147180369123816490e-01 + (de * 1.90821492927058770002e-10 + lm);
}

__device__ __forceinline__ double exp_det(double x) {
    if (x < -708.0) return 0.0;
    if (x > 709.0) return __longlong_as_double(0x7ff0000000000000ll);
    const double kf = floor(x * 1.44269504088896338700e+00 + 0.5);
    const double r = (x - kf * 6.93147180369123816490e-01) - kf * 1.90821492927058770002e-10;
    double p = 1.0 / 6227020800.0;
    p = p * r + 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    const int k = static_cast<int>(kf);
    const int k1 = k / 2, k2 = k - k1;
    const double s1 = __longlong_as_double(static_cast<long long>(k1 + 1023) << 52);
    const double s2 = __longlong_as_double(static_cast<long long>(k2 + 1023) << 52);
    return (p * s1) * s2;
}

__device__ __forceinline__ void sincos2pi_det(double u, double* sn, double* cs) {
    const double t = 4.0 * u;
    const double q = floor(t + 0.5);
    const double r = t - q;
    const double x = r * 1.57079632679489655800e+00;
    const double x2 = x * x;
    double ps = -1.0 / 355687428096000.0;
    ps = ps * x2 + 1.0 / 1307674368000.0;
    ps = ps * x2 - 1.0 / 6227020800.0;
    ps = ps * x2 + 1.0 / 39916800.0;
    ps = ps * x2 - 1.0 / 362880.0;
    ps = ps * x2 + 1.0 / 5040.0;
    ps = ps * x2 - 1.0 / 120.0;
    ps = ps * x2 + 1.0 / 6.0;
    const double s = x - x * x2 * ps;
    double pc = 1.0 / 6402373705728000.0;
    pc = pc * x2 - 1.0 / 20922789888000.0;
    pc = pc * x2 + 1.0 / 87178291200.0;
    pc = pc * x2 - 1.0 / 479001600.0;
    pc = pc * x2 + 1.0 / 3628800.0;
    pc = pc * x2 - 1.0 / 40320.0;
    pc = pc * x2 + 1.0 / 720.0;
    pc = pc * x2 - 1.0 / 24.0;
    pc = pc * x2 + 0.5;
    const double c = 1.0 - x2 * pc;
    switch (static_cast<int>(q) & 3) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
    }
}

// Pair p of draw `draw` on `substream`: normals 2p (cos) and 2p+1 (sin), Box-Muller on
// two 53-bit uniforms, u1 in (0,1], u2 in [0,1).
__device__ __forceinline__ void normal_pair(uint64_t key, uint32_t substream, uint64_t draw,
                                            uint32_t p, double* z0, double* z1) {
    const uint4 x = philox(make_uint4(p, substream, static_cast<uint32_t>(draw),
                                      static_cast<uint32_t>(draw >> 32)),
                           key);
    const uint64_t a = (static_cast<uint64_t>(x.x >> 5) << 26) | (x.y >> 6);
    const uint64_t b = (static_cast<uint64_t>(x.z >> 5) << 26) | (x.w >> 6);
    const double u1 = static_cast<double>(a + 1) * 1.1102230246251565404e-16; // 2^-53
    const double u2 = static_cast<double>(b) * 1.1102230246251565404e-16;
    const double r = sqrt(-2.0 * ln_det(u1));
    double sn, cs;
    sincos2pi_det(u2, &sn, &cs);
    *z0 = r * cs;
    *z1 = r * sn;
}

// coarse-grid offsets of one draw: counter {0xFFFFFFFF, substream, draw}, multiply-shift
__device__ __forceinline__ void draw_offsets(uint64_t key, uint32_t substream, uint64_t draw,
                                             int c, int* oj, int* ok) {
    const uint4 x = philox(make_uint4(0xFFFFFFFFu, substream, static_cast<uint32_t>(draw),
                                      static_cast<uint32_t>(draw >> 32)),
                           key);
    *oj = static_cast<int>(__umulhi(x.x, static_cast<uint32_t>(c)));
    *ok = static_cast<int>(__umulhi(x.y, static_cast<uint32_t>(c)));
}

// Catmull-Rom cubic (stochastic.hpp:81-87)
__device__ __forceinline__ double catmull(double fm1, double f0, double f1, double f2, double t) {
    const double a = 2.0 * f0;
    const double b = f1 - fm1;
    const double c = 2.0 * fm1 - 5.0 * f0 + 4.0 * f1 - f2;
    const double d = -fm1 + 3.0 * f0 - 3.0 * f1 + f2;
    return 0.5 * (a + t * (b + t * (c + t * d)));
}

__host__ __device__ __forceinline__ int wrapi(int a, int n) {
    int r = a % n;
    return r < 0 ? r + n : r;
}

// wrap for operands within one period of the range, a in [-n, 2n): no integer division
__host__ __device__ __forceinline__ int wrap1(int a, int n) {
    return a < 0 ? a + n : (a >= n ? a - n : a);
}

// wrap1 with a (rarely taken) exact fallback for tiny periods
__host__ __device__ __forceinline__ int wrapf(int a, int n) {
    const int r = wrap1(a, n);
    return (r < 0 || r >= n) ? wrapi(r, n) : r;
}

} // namespace det
} // namespace dcg
