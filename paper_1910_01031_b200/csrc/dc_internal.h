// dc_internal.h -- private structures shared by the CUDA translation units and the
// C-ABI implementation (api.cu). Not part of the public boundary.
#pragma once
#include <atomic>
#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/driftcast_gpu.h"

namespace dcg {

// device-side error codes (first error per member wins, atomicCAS from 0)
enum DevErr : int {
    E_NONE = 0,
    E_DRY_CELL = 2,      // "flux_rhs: dry cell at (j,k)"           (swe.hpp:324-331)
    E_NONFINITE = 3,     // "model_step: non-finite value after substep k" (swe.hpp:416-418)
    E_RUNAWAY = 4,       // "model_step: substep count exploded"   (swe.hpp:255-256)
    E_DRY_FACE = 12,     // "flux_rhs: dry reconstructed face value" (swe.hpp:374-375)
    E_DRY_ADD = 22,      // "add_q_half: perturbation dried a cell" (stochastic.hpp:159)
    E_DRY_DRIFTER = 32,  // "advect_drifters: dry cell at (j,k)"
    E_ALPHA = 42,        // "solve_alpha: ..."
    E_BETA = 52,         // "sync_target_beta: ..."
};

// Constants of the shallow-water stencil, derived exactly as the reference's Stepper
// derives them (double, then one rounding to float): swe.hpp:277-278,340-344,356-357,380-382.
// the stage kernel's column window: 2 columns per thread, a 2-column halo on each side
#ifndef DC_SWE_COLS
#define DC_SWE_COLS 256
#endif
constexpr int kSweCols = DC_SWE_COLS;
constexpr int kSweOut = kSweCols - 4;

struct SweParams {
    // state layout: every member holds (ny+4) x pitch floats per field -- the ny x nx
    // cells inside a 2-cell periodic ghost frame (stage kernels read it through TMA);
    // field pointers address cell (0, 0), cell (k, j) of member m is at
    // m*mstride + k*pitch + j, k in [-2, ny+2), j in [-2, nx+2)
    int nx, ny, pitch, M;
    size_t mstride;       // (ny + 4) * pitch
    int by, strips;       // rows per CTA strip, strips per member (uniform strips)
    const int2* units;    // optional CTA row units {m, y0 | y1 << 16}: big strips first,
    int n_units;          // short ones last so the final wave drains quickly (api.cu)
    int ctas_per_member;  // stage-2 CTAs of one member (set per launch by launch_stage)
    int tiles_x;          // 252-column tiles per row (set per launch)
    int grid_units;       // row units of the launch (grid y, continued in z past 65535)
    int end_mode;         // stage 2: fused substep end (0 off, 1 flag only, 2 + graph cond)
    unsigned long long end_cond;  // cudaGraphConditionalHandle of the step's while node
    float H, g, theta, cf_x, cf_y, inv_g, idx, idy, fH;
    float half_theta, fH_4;  // theta / 2, fH / 4 (exact scalings, swe.cu reconP / seg_tend)
    double dx, dy, courant, model_dt, h_eq, gd;
    float neg_zero;       // -0.0f, opaque to ptxas (packed-product addend, swe.cu)
};

// Per-member control block for the device-side CFL substep loop (swe.hpp:244-259).
struct StepCtl {
    double* t;          // simulation time
    double* t_end;      // t + model_dt of the step in progress
    double* remaining;  // seconds left in the step
    double* dt;         // dt of the substep about to run
    int* sub;           // substep index within the step
    int* active;        // 1 while remaining > 0
    int* err;           // DevErr
    int* err_pos;       // k*nx+j of the first dry cell found (atomicMin)
    int* err_sub;       // substep index of a non-finite failure
    unsigned* mx;       // [M][4]: max|u|+c bits, max|v|+c bits, ordered min h, spare
    int* any_active;    // loop condition (host-visible in the fallback path)
    unsigned* mdone;    // [M] stage-2 CTAs of the member finished this substep (fused end)
    int* n_active;      // members still stepping (fused end: the last one ends the loop)
    unsigned* step_max; // max substeps of a member in the step in progress
    unsigned long long* iters;  // [0] += substep-loop iterations per step (max over members),
                                // [1] += member-substeps (cell-updates / cells), counted as
                                // members retire from a step
};

struct ErrParams {
    int c, nxc, nyc;
    double dxc, dyc;
    double inv_c;         // 1.0 / c_omega (stochastic.hpp:96)
    double cx, cy;        // g*H/(f*2*dx), g*H/(f*2*dy)  (stochastic.hpp:127-128)
    double cxc, cyc;      // same at coarse spacing (stochastic.hpp:181-182)
    double w[25];         // SOAR weights w[(db+2)*5 + (da+2)] (stochastic.hpp:54-57)
    double h_eq;
};

// Opt a kernel in to `bytes` of dynamic shared memory on the current device, once per
// (kernel, device): the attribute is per device, so a process driving several GPUs needs
// it on each of them.
template <class F>
inline void smem_opt_in(F* func, size_t bytes) {
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_relaxed) & bit) return;
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    done.fetch_or(bit);
}

// ---- device allocations (guard.cu): plain cudaMalloc, or guard-banded with DC_GUARD=1 ----
cudaError_t dmalloc_impl(void** p, size_t bytes, const char* file, int line);
cudaError_t dfree(void* p);
int check_guards(std::string* msg);
template <class T>
inline cudaError_t dmalloc_t(T** p, size_t bytes, const char* file, int line) {
    return dmalloc_impl(reinterpret_cast<void**>(p), bytes, file, line);
}
#define DMALLOC(pp, bytes) dcg::dmalloc_t((pp), (bytes), __FILE__, __LINE__)

// ---- kernel profiler (kprof.cu; dc_profile_begin / dc_profile_end) ----
// A launcher declares `KScope ks(stream, "kernel", algorithmic_bytes);` before its launch:
// inside an open profile window (and outside stream capture) the kernel is bracketed by
// CUDA events on its stream; otherwise the scope costs one pointer test.
struct KScope {
    KScope(cudaStream_t s, const char* name, double bytes);
    ~KScope();
    KScope(const KScope&) = delete;
    KScope& operator=(const KScope&) = delete;
    cudaStream_t s;
    int rec;
};
bool kprof_active();
void kprof_begin();
int kprof_end(dc_kernel_time* out, int cap);

// stochastic.cu launchers
void launch_philox_noise(cudaStream_t s, const ErrParams& ep, int M, uint64_t seed, uint64_t tag,
                         int64_t member_base, uint32_t substream, uint64_t draw, double* xi,
                         int* offsets, const int* err);
// philox_noise + coarse_soar in one pass (xi stays on chip); needs (16+4)*nxc*8 B of
// shared memory (nxc <= 1280)
void launch_philox_soar(cudaStream_t s, const ErrParams& ep, int M, uint64_t seed, uint64_t tag,
                        int64_t member_base, uint32_t substream, uint64_t draw, double* corr,
                        int* offsets, const int* err);
void launch_coarse_soar(cudaStream_t s, const ErrParams& ep, int M, const double* in,
                        double* out, const int* err);
// smap: the model state set's TMA map with box {tile::TX + 4, tile::TY, 3} (api.cu qmap)
void launch_q_half_apply(cudaStream_t s, const CUtensorMap* smap, const SweParams& sp,
                         const ErrParams& ep, const double* corr, const int* offsets,
                         double scale, float* eta, float* hu, float* hv, int* err,
                         int* err_pos, int M, unsigned* mx = nullptr,
                         const char* prof_name = "q_half_apply");

// swe.cu launchers
void launch_cfl_scan(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                     const float* hv, StepCtl ctl);
void launch_step_begin(cudaStream_t s, const SweParams& sp, StepCtl ctl,
                       unsigned long long cond_handle = 0, int use_cond = 0);
void launch_reset_stats(cudaStream_t s, const SweParams& sp, StepCtl ctl);
int swe_stage_occupancy();
// TMA map of a state set (3 fields field_stride floats apart, origin = storage row -2 of
// member 0, column -2); box {box_cols, box_rows, 3} (0: the stage kernels' {256, 3})
bool make_state_map(CUtensorMap* map, const float* origin, const SweParams& sp,
                    size_t field_stride, int box_cols = 0, int box_rows = 0);
// refresh the ghost frame of a state set (f0 = field 0 at cell (0, 0))
void launch_fix_ghosts(cudaStream_t s, const SweParams& sp, float* f0, size_t field_stride);
// One SSP-RK2 stage over every member. maps: [0] the input state set, [1] the psi^n set
// (stage 2). end_mode of a stage-2 launch:
// 0 = none; 1 = each member's last stage-2 CTA runs the member's substep end (loop flag
// read by the host); 2 = same, and the CTA that retires the last active member clears
// the graph's while condition (cond_handle)
void launch_stage(cudaStream_t s, const SweParams& sp, bool exact, int stage,
                  const CUtensorMap* maps, const float* ie, const float* iu, const float* iv,
                  float* oe, float* ou, float* ov, StepCtl ctl,
                  unsigned long long cond_handle = 0, int end_mode = 0);
void launch_selftest_math(cudaStream_t s, unsigned long long* counts);
void launch_cfl_public(cudaStream_t s, const SweParams& sp, const float* eta, const float* hu,
                       const float* hv, unsigned long long* gmax, int* dry_pos);
void launch_flux_rhs(cudaStream_t s, const SweParams& sp, bool exact, int m,
                     const CUtensorMap* maps, const float* eta, const float* hu, const float* hv,
                     float* re, float* ru, float* rv, StepCtl ctl);

} // namespace dcg
