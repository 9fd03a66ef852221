// experiment_kernels.h -- launchers of experiment.cu (private).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "dc_internal.h"

namespace dcg {

void launch_obs_noise(cudaStream_t s, uint64_t seed, int kind, const int* ids, int n,
                      uint64_t obs_index, double sr_hu, double sr_hv, double* eps);
void launch_observe_drifters(cudaStream_t s, const SweParams& sp, const double* prev,
                             const double* cur, int n, double dt_obs, const double* eps, double* y);
void launch_pf_loglik(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                      const float* hv, const double* obs, const int* cells, int n_obs, double r_hu,
                      double r_hv, double* q, double* loglik, const int* err, int M);
// err_old: [3][M] err, err_pos, err_sub before resampling (a slot takes its source's flags)
void launch_resample(cudaStream_t s, const SweParams& sp, int M, const int* idx, const float* ie,
                     const float* iu, const float* iv, float* oe, float* ou, float* ov,
                     const double* t_in, double* t_out, int n_d, const double* pos_in,
                     double* pos_out, const int* wind_in, int* wind_out,
                     const int* err_old, int* err, int* err_pos, int* err_sub);
void launch_forecast_error(cudaStream_t s, const SweParams& sp, int M, int n_d, const double* pos,
                           const int* wind, const double* truth, double* ed, double* rd);

} // namespace dcg
