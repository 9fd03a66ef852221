// iewpf_kernels.h -- launchers of iewpf.cu (private).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "dc_internal.h"

namespace dcg {

void launch_obs_locate(cudaStream_t s, const SweParams& sp, const double* obs, int n_obs,
                       int* cells, int* bad);
void launch_innovations(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                        const float* hv, const double* obs, const int* cells, int n_obs,
                        const double* S, double log_ne, double* d, double* sd, double* scal,
                        const int* err, int M);
void launch_pull_windows(cudaStream_t s, const ErrParams& ep, const double* sd, int n_obs,
                         double* win, const int* err, int M);
void launch_tile_lists(cudaStream_t s, const SweParams& sp, const ErrParams& ep, const int* cells,
                       int n_obs, int* lists, int* counts, int* n_tiles_out, int* tiles_x_out);
// pull_tables (member-independent interpolation tables of every (tile, covering obs),
// tabs: n_tiles x n_obs x pull_table_bytes()) + pull_apply
size_t pull_table_bytes();
void launch_pull_apply(cudaStream_t s, const CUtensorMap* smap, const SweParams& sp,
                       const ErrParams& ep, const double* win,
                       const int* cells, int n_obs, const int* lists, const int* counts,
                       int n_tiles, int tiles_x, void* tabs, float* eta, float* hu, float* hv,
                       int* err, int* err_pos, int M, double entries, double touched_cells);
void launch_perp_pair(cudaStream_t s, const ErrParams& ep, uint64_t seed, int64_t member_base,
                      uint64_t cycle, double ratio, double* xi, double* nu, int* foffs,
                      double* scal, const int* err, int M);
void launch_gather_cz(cudaStream_t s, int M, const double* scal, double* cz);
// errors (E_BETA / E_ALPHA) go to aerr; launch_merge_err folds them into err after the
// pull chain joined, so an earlier-stage error keeps precedence
void launch_barrier_alpha(cudaStream_t s, const double* cz_all, int n_total, int M, double n_psi,
                          int one_stage, double* scal, double* wb, int* aerr);
void launch_merge_err(cudaStream_t s, int M, const int* aerr, int* err);
void launch_local_blocks(cudaStream_t s, const ErrParams& ep, const double* xi, const double* nu,
                         const double* scal, const double* wb, const int* cells, int n_obs,
                         const int* order, const int* level_start, int n_levels,
                         const int* foffs, const double* usig, double* z, const int* err,
                         const int* aerr, int M, int one_stage);
void launch_drifters(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                     const float* hv, int M, int n_d, double dt, double* pos, int* wind, int* err,
                     int* err_pos);
void launch_observe_mooring(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                            const float* hv, int m, const double* xy, int n, double* y, int* bad);

} // namespace dcg
