// iewpf_host.h -- device buffers of the observation / drifter / IEWPF stages.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>

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
    double S_host[4] = {0, 0, 0, 0};
    std::vector<double> usig_host;
    bool usig_valid = false;
    void* stage = nullptr;    // pinned host staging
    size_t stage_bytes = 0;
    // local-block schedule: observation ids ordered by dependency level
    int* lb_order = nullptr;  // [cap_obs]
    int* lb_start = nullptr;  // [cap_obs + 1] first position of each level in lb_order
    int lb_levels = 0;
    std::vector<double> lb_xy;  // observation positions the schedule was built for
    std::vector<int> lb_host;   // host copy of order + start (source of the async upload)
    // drifters
    int n_d = 0;
    double* dpos = nullptr;   // [M][n_d][2]
    int* dwind = nullptr;     // [M][n_d][2]
};

inline void iewpf_free(IewpfBuffers& b) {
    void* ps[] = {b.obs, b.cells, b.d, b.sd, b.win, b.tile_lists, b.tile_count, b.nu, b.scal,
                  b.cz, b.cz_all, b.wb, b.S, b.usig, b.foffs, b.dpos, b.dwind, b.z, b.bad,
                  b.lb_order, b.lb_start};
    for (void* p : ps)
        if (p) cudaFree(p);
    if (b.stage) cudaFreeHost(b.stage);
    b = IewpfBuffers{};
}

} // namespace dcg
