// experiment.cu -- the twin-experiment operators either side of the hot path (SURVEY.md
// §8(f)), on sm_100a, compiled --fmad=false like the other fp64 units:
//   obs_noise        eps ~ N(0, diag(r_hu, r_hv)) per (platform, observation index),
//                    counter-based (stream_seed(seed, obs_noise, platform))
//   observe_drifters observe_drifter: minimal-image displacement / dt_obs
//                    times H_eq, + eps
//   pf_loglik        standard particle-filter log-likelihood -1/2 d^T R^-1 d of every member
//                    with the eta-compensated innovations, obs-id order
//   resample_gather  member m <- member idx[m] (fields, time, drifter copies) after
//                    residual resampling
//   forecast_error   E_d and RMSE_d of the drifter forecast (PAPER.md:1919-1926,
//                    SPEC.md:674-682), members summed in id order
#include <cuda_runtime.h>
#include <cstdint>

#include "dc_internal.h"
#include "detmath.cuh"
#include "experiment_kernels.h"

namespace dcg {

namespace {

constexpr uint64_t kTagObsNoise = 4;  // StreamTag::obs_noise (rng.hpp:21)

__global__ void obs_noise_kernel(uint64_t seed, int kind, const int* __restrict__ ids, int n,
                                 uint64_t obs_index, double sr_hu, double sr_hv, double* eps) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t platform =
        (static_cast<uint64_t>(static_cast<uint32_t>(kind)) << 32) | static_cast<uint32_t>(ids[i]);
    const uint64_t key = det::stream_key(seed, kTagObsNoise, platform);
    double z0, z1;
    det::normal_pair(key, 0u, obs_index, 0u, &z0, &z1);
    eps[2 * i] = sr_hu * z0;
    eps[2 * i + 1] = sr_hv * z1;
}

// minimal periodic image of a displacement between two wrapped positions
__device__ __forceinline__ double min_image(double d, double len) {
    if (d > 0.5 * len) return d - len;
    if (d < -0.5 * len) return d + len;
    return d;
}

__global__ void observe_drifters_kernel(SweParams sp, const double* __restrict__ prev,
                                        const double* __restrict__ cur, int n, double dt_obs,
                                        const double* __restrict__ eps, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lx = sp.nx * sp.dx, ly = sp.ny * sp.dy;
    const double ddx = min_image(cur[2 * i] - prev[2 * i], lx);
    const double ddy = min_image(cur[2 * i + 1] - prev[2 * i + 1], ly);
    double yh = ddx / dt_obs * sp.h_eq;
    double yv = ddy / dt_obs * sp.h_eq;
    if (eps) {
        yh = yh + eps[2 * i];
        yv = yv + eps[2 * i + 1];
    }
    y[2 * i] = yh;
    y[2 * i + 1] = yv;
}

// one CTA per member: q_o = d0*d0/r_hu + d1*d1/r_hv with d the innovation of
// innovations_kernel, then phi = sum_o q_o from 0.0 in id order
__global__ void pf_loglik_kernel(SweParams sp, const float* __restrict__ eta,
                                 const float* __restrict__ hu, const float* __restrict__ hv,
                                 const double* __restrict__ obs, const int* __restrict__ cells,
                                 int n_obs, double r_hu, double r_hv, double* q, double* loglik,
                                 const int* err) {
    const int m = blockIdx.x;
    if (err[m]) {
        if (threadIdx.x == 0) loglik[m] = -__longlong_as_double(0x7ff0000000000000ll);
        return;
    }
    const size_t mbase = static_cast<size_t>(m) * sp.mstride;
    double* qm = q + static_cast<size_t>(m) * n_obs;
    for (int o = threadIdx.x; o < n_obs; o += blockDim.x) {
        const int j = cells[2 * o], k = cells[2 * o + 1];
        const size_t c = mbase + static_cast<size_t>(k) * sp.pitch + j;
        const double h = sp.h_eq + static_cast<double>(eta[c]);
        const double d0 = obs[4 * o + 2] * h / sp.h_eq - static_cast<double>(hu[c]);
        const double d1 = obs[4 * o + 3] * h / sp.h_eq - static_cast<double>(hv[c]);
        qm[o] = d0 * d0 / r_hu + d1 * d1 / r_hv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int o = 0; o < n_obs; ++o) s += qm[o];
        loglik[m] = -0.5 * s;
    }
}

// fields: out member m, row k <- in member idx[m], row k (grid: rows, members)
__global__ void resample_fields_kernel(SweParams sp, const int* __restrict__ idx,
                                       const float* __restrict__ ie, const float* __restrict__ iu,
                                       const float* __restrict__ iv, float* oe, float* ou,
                                       float* ov) {
    const int m = blockIdx.y, k = blockIdx.x;
    const size_t src = static_cast<size_t>(idx[m]) * sp.mstride + static_cast<size_t>(k) * sp.pitch;
    const size_t dst = static_cast<size_t>(m) * sp.mstride + static_cast<size_t>(k) * sp.pitch;
    for (int j = threadIdx.x; j < sp.nx; j += blockDim.x) {
        oe[dst + j] = ie[src + j];
        ou[dst + j] = iu[src + j];
        ov[dst + j] = iv[src + j];
    }
}

// per-member scalars and drifter copies; reads the pre-resampling copies
__global__ void resample_members_kernel(int M, int n_d, const int* __restrict__ idx,
                                        const double* __restrict__ t_in, double* t_out,
                                        const double* __restrict__ pos_in, double* pos_out,
                                        const int* __restrict__ wind_in, int* wind_out,
                                        const int* __restrict__ err_old, int* err, int* err_pos,
                                        int* err_sub) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M) {
        t_out[i] = t_in[idx[i]];
        err[i] = err_old[idx[i]];
        err_pos[i] = err_old[M + idx[i]];
        err_sub[i] = err_old[2 * M + idx[i]];
    }
    if (n_d > 0 && i < M * n_d * 2) {
        const int m = i / (n_d * 2), r = i - m * n_d * 2;
        const size_t src = static_cast<size_t>(idx[m]) * n_d * 2 + r;
        pos_out[i] = pos_in[src];
        wind_out[i] = wind_in[src];
    }
}

// one CTA per drifter: E_d = mean_i |x_i - truth|^2 and the ensemble mean of the
// unwrapped positions (x + wind * L), then RMSE_d = mean_i |x_i - mean|^2, distances by
// the minimal periodic image. The per-member terms are computed in parallel, a chunk of
// kFeThreads members at a time; thread 0 folds each chunk in member-id order, so the sums
// are the sequential ones (bitwise equal to the oracle and to any member partition).
constexpr int kFeThreads = 128;

__global__ void __launch_bounds__(kFeThreads)
forecast_error_kernel(SweParams sp, int M, int n_d, const double* __restrict__ pos,
                      const int* __restrict__ wind, const double* __restrict__ truth,
                      double* ed, double* rd) {
    __shared__ double t_e[kFeThreads], t_x[kFeThreads], t_y[kFeThreads];
    __shared__ double s_mean[2];
    const int d = blockIdx.x;
    const int t = threadIdx.x;
    const double lx = sp.nx * sp.dx, ly = sp.ny * sp.dy;
    const double tx = truth[2 * d], ty = truth[2 * d + 1];
    double se = 0.0, sx = 0.0, sy = 0.0;
    for (int m0 = 0; m0 < M; m0 += kFeThreads) {
        const int m = m0 + t;
        if (m < M) {
            const size_t q = (static_cast<size_t>(m) * n_d + d) * 2;
            const double ex = min_image(pos[q] - tx, lx), ey = min_image(pos[q + 1] - ty, ly);
            t_e[t] = ex * ex + ey * ey;
            t_x[t] = pos[q] + wind[q] * lx;
            t_y[t] = pos[q + 1] + wind[q + 1] * ly;
        }
        __syncthreads();
        if (t == 0) {
            const int n = min(kFeThreads, M - m0);
            for (int i = 0; i < n; ++i) {
                se = se + t_e[i];
                sx = sx + t_x[i];
                sy = sy + t_y[i];
            }
        }
        __syncthreads();
    }
    if (t == 0) {
        const double mx = sx / M, my = sy / M;
        // wrap the mean into the domain for the minimal-image spread
        double wx = fmod(mx, lx), wy = fmod(my, ly);
        if (wx < 0.0) wx += lx;
        if (wy < 0.0) wy += ly;
        s_mean[0] = wx;
        s_mean[1] = wy;
    }
    __syncthreads();
    const double wx = s_mean[0], wy = s_mean[1];
    double sr = 0.0;
    for (int m0 = 0; m0 < M; m0 += kFeThreads) {
        const int m = m0 + t;
        if (m < M) {
            const size_t q = (static_cast<size_t>(m) * n_d + d) * 2;
            const double ex = min_image(pos[q] - wx, lx), ey = min_image(pos[q + 1] - wy, ly);
            t_e[t] = ex * ex + ey * ey;
        }
        __syncthreads();
        if (t == 0) {
            const int n = min(kFeThreads, M - m0);
            for (int i = 0; i < n; ++i) sr = sr + t_e[i];
        }
        __syncthreads();
    }
    if (t == 0) {
        ed[d] = se / M;
        rd[d] = sr / M;
    }
}

} // namespace

void launch_obs_noise(cudaStream_t s, uint64_t seed, int kind, const int* ids, int n,
                      uint64_t obs_index, double sr_hu, double sr_hv, double* eps) {
    KScope ks(s, "obs_noise", 20.0 * n);
    obs_noise_kernel<<<(n + 127) / 128, 128, 0, s>>>(seed, kind, ids, n, obs_index, sr_hu, sr_hv,
                                                     eps);
}

void launch_observe_drifters(cudaStream_t s, const SweParams& sp, const double* prev,
                             const double* cur, int n, double dt_obs, const double* eps, double* y) {
    KScope ks(s, "observe_drifters", 64.0 * n);
    observe_drifters_kernel<<<(n + 127) / 128, 128, 0, s>>>(sp, prev, cur, n, dt_obs, eps, y);
}

void launch_pf_loglik(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                      const float* hv, const double* obs, const int* cells, int n_obs, double r_hu,
                      double r_hv, double* q, double* loglik, const int* err, int M) {
    KScope ks(s, "pf_loglik", (12.0 + 16.0) * n_obs * M);
    pf_loglik_kernel<<<M, 128, 0, s>>>(sp, eta, hu, hv, obs, cells, n_obs, r_hu, r_hv, q, loglik,
                                       err);
}

void launch_resample(cudaStream_t s, const SweParams& sp, int M, const int* idx, const float* ie,
                     const float* iu, const float* iv, float* oe, float* ou, float* ov,
                     const double* t_in, double* t_out, int n_d, const double* pos_in,
                     double* pos_out, const int* wind_in, int* wind_out, const int* err_old,
                     int* err, int* err_pos, int* err_sub) {
    {
        KScope ks(s, "resample_fields", 24.0 * sp.nx * sp.ny * M);
        resample_fields_kernel<<<dim3(sp.ny, M), 128, 0, s>>>(sp, idx, ie, iu, iv, oe, ou, ov);
    }
    KScope ks(s, "resample_members", (16.0 + 48.0 * n_d) * M);
    const int n = (M * n_d * 2 > M) ? M * n_d * 2 : M;
    resample_members_kernel<<<(n + 127) / 128, 128, 0, s>>>(M, n_d, idx, t_in, t_out, pos_in,
                                                            pos_out, wind_in, wind_out, err_old,
                                                            err, err_pos, err_sub);
}

void launch_forecast_error(cudaStream_t s, const SweParams& sp, int M, int n_d, const double* pos,
                           const int* wind, const double* truth, double* ed, double* rd) {
    KScope ks(s, "forecast_error", 24.0 * n_d * M + 32.0 * n_d);
    forecast_error_kernel<<<n_d, kFeThreads, 0, s>>>(sp, M, n_d, pos, wind, truth, ed, rd);
}

} // namespace dcg
