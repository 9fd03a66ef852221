// iewpf_host.h -- device buffers of the observation / drifter / IEWPF stages.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

#include "dc_internal.h"

namespace dcg {

struct IewpfBuffers {
    int cap_obs = 0;          // capacity (observations)
    int n_obs = 0;
    double* obs = nullptr;    // [n_obs][4] x, y, y_hu, y_hv
    int* cells = nullptr;     // [n_obs][2] containing cell (j,k)
    double* d = nullptr;      // [M][n_obs][2] innovations
    double* sd = nullptr;     // [M][n_obs][2] S*d
    double* win = nullptr;    // [M][n_obs][121] pull windows (SOAR(SOAR(dipole)))
    int* tile_lists = nullptr;// [n_tiles][cap_obs] int4 {obs id, oj | ok << 16, ao, bo}, ascending id
    int* tile_count = nullptr;// [n_tiles]
    void* tabs = nullptr;     // [n_tiles][cap_obs] interpolation tables of the pull
    double* nu = nullptr;     // [M][nr]
    double* scal = nullptr;   // [M][8]: c, phi, gamma, zeta, alpha, xx, nn, nx
    double* cz = nullptr;     // [M][2] local (c, zeta)
    double* cz_all = nullptr; // [cap_total][2]
    int cap_total = 0;
    double* wb = nullptr;     // [2] w_target, beta
    double* S = nullptr;      // [4]
    double* usig = nullptr;   // [49*49]
    int* foffs = nullptr;     // [M][2] filter-grid offsets
    double* z = nullptr;      // [M][nr] posterior coarse field
    int* bad = nullptr;       // locate failure flag
    int n_total = 0;
    uint64_t cycle = 0;
    int one_stage = 0;        // dc_iewpf_set_mode
    bool pending = false;     // dc_iewpf_begin done, dc_iewpf_finish not yet: the obs /
                              // cells / S d buffers belong to that analysis
    double S_host[4] = {0, 0, 0, 0};
    std::vector<double> usig_host;
    bool usig_valid = false;
    // pinned host staging ring for observation uploads: a slot is reused only after the
    // event recorded behind its H2D copy completed, so an upload never drains the stream
    static constexpr int kStageSlots = 4;
    unsigned char* stage = nullptr;  // kStageSlots x stage_bytes
    size_t stage_bytes = 0;          // per slot
    cudaEvent_t stage_ev[kStageSlots] = {nullptr, nullptr, nullptr, nullptr};
    int stage_next = 0;
    // local-block schedule: observation ids ordered by dependency level
    int* lb_order = nullptr;  // [cap_obs]
    int* lb_start = nullptr;  // [cap_obs + 1] first position of each level in lb_order
    int lb_levels = 0;
    std::vector<double> lb_xy;  // observation positions the schedule was built for
    std::vector<int> lb_host;   // host copy of order + start, uploaded from the pinned
    bool lb_dirty = false;      // staging slot of the next upload_obs when dirty
    // pull footprint of the current observation set (algorithmic bytes of the pull, kprof):
    // (tile, covering obs) entries and the cells of the tiles at least one obs touches
    double pull_entries = 0.0, pull_cells = 0.0;
    // drifters
    int n_d = 0;
    double* dpos = nullptr;   // [M][n_d][2]
    int* dwind = nullptr;     // [M][n_d][2]
    // the pull chain (pull_windows -> tile_lists -> pull_tables -> pull_apply) runs on a
    // second stream, concurrently with perp_pair, the barrier exchange, barrier_alpha,
    // local_blocks and coarse_soar, which never touch the state; the posterior waits for it
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool join_pending = false;
    int* aerr = nullptr;      // [M] barrier / alpha errors, merged into err after the join
                              // (so a pull error keeps its precedence, as in the reference)
};

// persistent scratch of forecast_error (per-drifter E_d, RMSE_d): device truth and results,
// pinned host copies; grown on demand, never freed per call
struct FeScratch {
    int cap = 0;
    double* d_truth = nullptr;  // [cap][2]
    double* d_out = nullptr;    // [2][cap] E_d, RMSE_d
    double* h_io = nullptr;     // pinned [4][cap]: truth in, E_d / RMSE_d out
};

// pinned readback slots (dc_readback_enqueue / dc_readback_wait): one cycle's outputs
// copied device -> host behind the cycle's work, read by the host while later cycles run
struct ReadbackSlot {
    bool used = false;       // enqueued and not yet waited for
    bool has_diag = false, has_drift = false, has_fe = false;
    int n_d = 0;
    size_t cap = 0;          // bytes of buf
    unsigned char* buf = nullptr;  // pinned: err[M] | scal[M*8] | wb[2] | pos | wind | truth | fe
    cudaEvent_t ev = nullptr;
};
constexpr int kReadbackSlots = 2;

inline void readback_free(ReadbackSlot* r) {
    for (int i = 0; i < kReadbackSlots; ++i) {
        if (r[i].buf) cudaFreeHost(r[i].buf);
        if (r[i].ev) cudaEventDestroy(r[i].ev);
        r[i] = ReadbackSlot{};
    }
}

inline void fe_free(FeScratch& f) {
    if (f.d_truth) dcg::dfree(f.d_truth);
    if (f.d_out) dcg::dfree(f.d_out);
    if (f.h_io) cudaFreeHost(f.h_io);
    f = FeScratch{};
}

inline void iewpf_free(IewpfBuffers& b) {
    void* ps[] = {b.obs, b.cells, b.d, b.sd, b.win, b.tile_lists, b.tile_count, b.tabs, b.nu, b.scal,
                  b.cz, b.cz_all, b.wb, b.S, b.usig, b.foffs, b.dpos, b.dwind, b.z, b.bad,
                  b.lb_order, b.lb_start, b.aerr};
    for (void* p : ps)
        if (p) dcg::dfree(p);
    if (b.aux) {
        cudaStreamSynchronize(b.aux);
        cudaStreamDestroy(b.aux);
    }
    if (b.ev_fork) cudaEventDestroy(b.ev_fork);
    if (b.ev_join) cudaEventDestroy(b.ev_join);
    if (b.stage) cudaFreeHost(b.stage);
    for (cudaEvent_t e : b.stage_ev)
        if (e) cudaEventDestroy(e);
    b = IewpfBuffers{};
}

} // namespace dcg
