// host_ops.cpp -- host-side steps of the SIR comparison (SPEC.md iewpf_filter, standard PF
// weights + residual resampling). The log-likelihoods come from the device
// (dc_pf_loglik); what is left is O(N_e) scalar work in a fixed order, so every rank of a
// multi-GPU run computes identical weights and indices from the all-gathered values.
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/driftcast_gpu.h"

namespace {

uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// stream_seed (rng.hpp:35-40)
uint64_t stream_key(uint64_t master, uint64_t tag, uint64_t index) {
    uint64_t s = splitmix(master ^ 0x8000000000000000ull);
    s = splitmix(s ^ tag);
    return splitmix(s ^ (index + 0x51ed2700a1b4c2d3ull));
}

// Philox4x32-10, the same bijection as the device generator (csrc/detmath.cuh)
void philox(uint32_t c[4], uint64_t key) {
    uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
        const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
        const uint32_t lo0 = static_cast<uint32_t>(p0), hi0 = static_cast<uint32_t>(p0 >> 32);
        const uint32_t lo1 = static_cast<uint32_t>(p1), hi1 = static_cast<uint32_t>(p1 >> 32);
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
    }
}

constexpr uint64_t kTagResample = 7;  // StreamTag::resample (rng.hpp:24)

// uniform in [0,1) of residual draw s at cycle: counter {s, 0, cycle lo, cycle hi}
double resample_uniform(uint64_t key, uint64_t cycle, uint32_t s) {
    uint32_t c[4] = {s, 0u, static_cast<uint32_t>(cycle), static_cast<uint32_t>(cycle >> 32)};
    philox(c, key);
    const uint64_t a = (static_cast<uint64_t>(c[0] >> 5) << 26) | (c[1] >> 6);
    return static_cast<double>(a) * 1.1102230246251565404e-16;  // 2^-53
}

} // namespace

extern "C" {

// standard_pf_weights: w_i proportional to exp(loglik_i), normalised.
// Evaluated as exp(loglik_i - max) / sum_k exp(loglik_k - max), sums in index order.
// Collapse: every exp(loglik_i) underflows in double (max < log of the smallest
// subnormal), reported with the max log-weight.
dc_status dc_pf_weights(const double* loglik, int32_t n, double* w_out, double* max_loglik) {
    if (n <= 0 || !loglik || !w_out) return DC_EINVAL;
    double mx = -INFINITY;
    for (int i = 0; i < n; ++i)
        if (loglik[i] > mx) mx = loglik[i];
    if (max_loglik) *max_loglik = mx;
    if (!std::isfinite(mx)) return DC_ECOLLAPSE;
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        w_out[i] = std::exp(loglik[i] - mx);
        s += w_out[i];
    }
    for (int i = 0; i < n; ++i) w_out[i] = w_out[i] / s;
    if (mx < -745.13321910194122) return DC_ECOLLAPSE;  // exp(mx) == 0 in double
    return DC_OK;
}

// residual_resample: floor(N w_i) copies of particle i, then the
// remaining R slots by multinomial draws on the residuals N w_i - floor(N w_i) (inverse
// CDF over the ascending cumulative sum). Counts within 1e-12 of an integer are taken as
// that integer, so exactly representable shares (uniform, 1/2, ...) are deterministic
// even when N w_i rounds to 0.999...9. Output: the index multiset in ascending order.
dc_status dc_residual_resample(const double* w, int32_t n, uint64_t seed, uint64_t cycle,
                               int32_t* idx_out) {
    if (n <= 0 || !w || !idx_out) return DC_EINVAL;
    std::vector<int64_t> cnt(n, 0);
    std::vector<double> res(n, 0.0);
    int64_t used = 0;
    for (int i = 0; i < n; ++i) {
        if (!(w[i] >= 0.0) || !std::isfinite(w[i])) return DC_EINVAL;
        const double x = static_cast<double>(n) * w[i];
        const double f = std::floor(x + 1e-12);
        cnt[i] = static_cast<int64_t>(f);
        res[i] = x - f > 0.0 ? x - f : 0.0;
        used += cnt[i];
    }
    if (used > n) return DC_EINVAL;  // weights do not sum to 1
    const int64_t R = n - used;
    if (R > 0) {
        std::vector<double> cum(n);
        double s = 0.0;
        for (int i = 0; i < n; ++i) {
            s += res[i];
            cum[i] = s;
        }
        if (!(s > 0.0)) return DC_EINVAL;
        const uint64_t key = stream_key(seed, kTagResample, 0);
        for (int64_t r = 0; r < R; ++r) {
            const double u = resample_uniform(key, cycle, static_cast<uint32_t>(r)) * s;
            int lo = 0, hi = n - 1;  // first i with cum[i] > u
            while (lo < hi) {
                const int mid = (lo + hi) / 2;
                if (cum[mid] > u) hi = mid;
                else lo = mid + 1;
            }
            cnt[lo] += 1;
        }
    }
    int k = 0;
    for (int i = 0; i < n; ++i)
        for (int64_t c = 0; c < cnt[i]; ++c) idx_out[k++] = i;
    return DC_OK;
}

} // extern "C"
