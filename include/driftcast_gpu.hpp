// driftcast_gpu.hpp -- header-only C++ face of the C ABI (driftcast_gpu.h) shaped like
// the reference operator surface (proj/include/driftcast/*.hpp), for the existing C++
// driver. Status codes become the reference's exception types:
//   DC_EINVAL -> std::invalid_argument, DC_EDRY -> DryCellError (swe.hpp:32-34),
//   DC_ENONFINITE / DC_ERUNAWAY -> std::runtime_error (swe.hpp:255-256, 416-418).
// When the reference headers are on the include path, driftcast::DryCellError itself is
// thrown, so existing catch sites keep working unchanged.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "driftcast_gpu.h"

#if defined(__has_include)
#if __has_include("driftcast/swe.hpp")
#include "driftcast/swe.hpp"
#define DRIFTCAST_GPU_HAVE_REFERENCE 1
#endif
#endif

namespace driftcast {
namespace gpu {

#ifdef DRIFTCAST_GPU_HAVE_REFERENCE
using DryCellError = ::driftcast::DryCellError;
#else
struct DryCellError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#endif

inline void throw_status(dc_status st, const std::string& msg) {
    switch (st) {
    case DC_OK: return;
    case DC_EINVAL: throw std::invalid_argument(msg);
    case DC_EDRY: throw DryCellError(msg);
    case DC_ENONFINITE:
    case DC_ERUNAWAY:
    case DC_EIO:        // snapshot / file I/O (state.hpp:71-116 throws runtime_error)
    case DC_ECOLLAPSE:  // standard PF weights: "ensemble collapse"
    case DC_ENCCL:      // multi-GPU communicator
        throw std::runtime_error(msg);
    default: throw std::runtime_error("driftcast_gpu: " + msg);
    }
}

/// Paper defaults (§5): 500x300 double jet, dx=dy=2220 m, c_Omega=5,
/// L0 = 3/4 coarse spacing, q0 = 2.5e-4, Courant 0.8, theta 1.3, model dt 60 s.
inline dc_config default_config() {
    dc_config c{};
    c.nx = 500;
    c.ny = 300;
    c.dx = c.dy = 2220.0;
    c.g = 9.806;
    c.f = 1.405e-4;
    c.h_eq = 230.0;
    c.courant = 0.8;
    c.limiter_theta = 1.3;
    c.model_dt = 60.0;
    c.q0 = 2.5e-4;
    c.c_omega = 5;
    c.l0 = 0.75 * c.c_omega * c.dx;
    c.c_soar = 2;
    c.seed = 1;
    c.exact_fp = 1;
    return c;
}

/// Precomputed IEWPF operators.
struct FilterOperators {
    double hqht[4];
    double S[4];
    std::vector<double> block, usig;  // 49x49 row-major
};

inline FilterOperators precompute_filter_operators(const dc_config& cfg, double r_hu = 1.0,
                                                   double r_hv = 1.0) {
    FilterOperators f;
    throw_status(dc_precompute_S(&cfg, r_hu, r_hv, f.hqht, f.S), "precompute_S failed");
    f.block.resize(49 * 49);
    f.usig.resize(49 * 49);
    throw_status(dc_precompute_local_svd(&cfg, f.S, f.block.data(), f.usig.data()),
                 "precompute_local_svd failed");
    return f;
}

/// An ensemble of particles resident on one GPU: the batched counterpart of
/// std::vector<OceanState> + Stepper + NoiseStream per particle.
class Ensemble {
public:
    Ensemble(const dc_config& cfg, int n_members, std::int64_t member_base = 0, int device = 0,
             void* stream = nullptr)
        : cfg_(cfg), n_(n_members) {
        dc_status st = dc_create(&cfg, n_members, member_base, device, stream, &ctx_);
        if (st) throw_status(st, "dc_create failed");
    }
    ~Ensemble() {
        if (ctx_) dc_destroy(ctx_);
    }
    Ensemble(const Ensemble&) = delete;
    Ensemble& operator=(const Ensemble&) = delete;
    Ensemble(Ensemble&& o) noexcept : cfg_(o.cfg_), n_(o.n_), ctx_(o.ctx_) { o.ctx_ = nullptr; }

    int size() const { return n_; }
    const dc_config& config() const { return cfg_; }
    dc_ctx* handle() { return ctx_; }

    // init_double_jet (swe.hpp:459-500) broadcast to every particle
    void init_double_jet() { check(dc_init_double_jet(ctx_)); }
    // Stepper::model_step (swe.hpp:244-259) on every particle, n times
    void model_step(int n = 1) { check(dc_step(ctx_, n)); }
    // perturb_state (stochastic.hpp:164-173), counter-based noise
    void perturb_state() { check(dc_perturb(ctx_, DC_NOISE_PHILOX, nullptr, nullptr)); }
    // perturb_state with injected offsets [n][2] and xi [n][nxc*nyc]
    void perturb_state(const std::int32_t* offsets, const double* xi) {
        check(dc_perturb(ctx_, DC_NOISE_INJECTED, offsets, xi));
    }
    // advect_drifters
    void set_drifters(const std::vector<double>& pos_xy, int n_drifters) {
        check(dc_drifters_set(ctx_, pos_xy.data(), n_drifters));
    }
    void advect_drifters(double dt) { check(dc_drifters_advect(ctx_, dt)); }
    // iewpf_assimilate, single-context (no collective)
    void iewpf_assimilate(const std::vector<dc_obs>& obs, const FilterOperators& f,
                          std::uint64_t cycle) {
        check(dc_iewpf_assimilate(ctx_, obs.data(), static_cast<int>(obs.size()), f.S,
                                  f.usig.data(), cycle));
    }
    // the analysis split at its barrier (multi-GPU drivers that run their own collective):
    // begin -> exchange every rank's (c_i, zeta_i) [n_total][2] -> finish
    void iewpf_begin(const std::vector<dc_obs>& obs, const FilterOperators& f,
                     std::uint64_t cycle, int n_total, double* cz_out, bool cz_on_device) {
        check(dc_iewpf_begin(ctx_, obs.data(), static_cast<int>(obs.size()), f.S, f.usig.data(),
                             cycle, n_total, cz_out, cz_on_device ? 1 : 0));
    }
    void iewpf_finish(const double* cz_all, bool cz_on_device) {
        check(dc_iewpf_finish(ctx_, cz_all, cz_on_device ? 1 : 0));
    }
    // the original one-stage IEWPF instead of the two-stage default
    void set_one_stage(bool one_stage) {
        check(dc_iewpf_set_mode(ctx_, one_stage ? DC_IEWPF_ONE_STAGE : DC_IEWPF_TWO_STAGE));
    }
    // multi-GPU (one process per GPU): join the ranks' NCCL communicator; afterwards
    // iewpf_assimilate / da_cycle exchange (c_i, zeta_i) at the barrier and forecast
    // statistics gather every rank's drifters to rank 0
    void comm_attach(const std::uint8_t* nccl_id, int rank, int world, std::int64_t n_total) {
        check(dc_comm_attach(ctx_, nccl_id, rank, world, n_total));
    }
    void comm_detach() { check(dc_comm_detach(ctx_)); }
    // one DA cycle
    void da_cycle(int n_steps, const std::vector<dc_obs>& obs, const FilterOperators& f,
                  std::uint64_t cycle) {
        check(dc_da_cycle(ctx_, n_steps, obs.data(), static_cast<int>(obs.size()), f.S,
                          f.usig.data(), cycle));
    }
    // innovation of every member: d[m][o][2] (synchronous)
    std::vector<double> innovations(const std::vector<dc_obs>& obs) {
        std::vector<double> d(static_cast<size_t>(n_) * obs.size() * 2);
        check(dc_innovations(ctx_, obs.data(), static_cast<int>(obs.size()), d.data()));
        return d;
    }
    // observe_mooring without noise on member m: y[o][2]
    std::vector<double> observe_mooring(int m, const std::vector<double>& xy) {
        std::vector<double> y(xy.size());
        check(dc_observe_mooring(ctx_, m, xy.data(), static_cast<int>(xy.size() / 2), y.data()));
        return y;
    }
    // Stepper::flux_rhs (swe.hpp:229-239) of member m, Field2D layout
    void flux_rhs(int m, std::vector<float>& de, std::vector<float>& du, std::vector<float>& dv) {
        const size_t n = static_cast<size_t>(cfg_.nx) * cfg_.ny;
        de.resize(n);
        du.resize(n);
        dv.resize(n);
        check(dc_flux_rhs(ctx_, m, de.data(), du.data(), dv.data()));
    }
    // Stepper::cfl_dt (swe.hpp:212-226) of every member
    std::vector<double> cfl_dt() {
        std::vector<double> dt(n_);
        check(dc_cfl_dt(ctx_, dt.data()));
        return dt;
    }
    // pipelined per-cycle outputs: enqueue behind the queued work, read while the next
    // cycle runs (slot 0 or 1); truth_xy [n_d][2] enables the forecast statistics
    void readback_enqueue(int slot, const std::vector<double>* truth_xy) {
        int what = DC_READBACK_DIAG | DC_READBACK_DRIFTERS;
        if (truth_xy) what |= DC_READBACK_FORECAST_ERROR;
        check(dc_readback_enqueue(ctx_, slot, what, truth_xy ? truth_xy->data() : nullptr));
    }
    struct Readback {
        std::vector<dc_particle_diag> diag;
        double w_beta[2] = {0.0, 0.0};
        std::vector<double> pos;
        std::vector<std::int32_t> wind;
        double E = 0.0, RMSE = 0.0;
    };
    Readback readback_wait(int slot, int n_drifters) {
        Readback r;
        r.diag.resize(n_);
        r.pos.resize(static_cast<size_t>(n_) * n_drifters * 2);
        r.wind.resize(r.pos.size());
        r.E = r.RMSE = std::nan("");
        check(dc_readback_wait(ctx_, slot, r.diag.data(), r.w_beta, r.pos.data(), r.wind.data(),
                               &r.E, &r.RMSE));
        return r;
    }
    std::vector<dc_particle_diag> diagnostics(double* w_beta = nullptr) {
        std::vector<dc_particle_diag> d(n_);
        double wb[2];
        check(dc_iewpf_diagnostics(ctx_, d.data(), w_beta ? w_beta : wb));
        return d;
    }
    // OceanState of particle m, Field2D layout (field.hpp:48-50)
    void download(int m, std::vector<float>& eta, std::vector<float>& hu, std::vector<float>& hv,
                  double* t) {
        const size_t n = static_cast<size_t>(cfg_.nx) * cfg_.ny;
        eta.resize(n);
        hu.resize(n);
        hv.resize(n);
        check(dc_download_member(ctx_, m, eta.data(), hu.data(), hv.data(), t));
    }
    void upload(int m, const float* eta, const float* hu, const float* hv, double t) {
        check(dc_upload_member(ctx_, m, eta, hu, hv, t));
    }
    // snapshots / checkpoints (state.hpp:71-116)
    void save_snapshot(int m, const std::string& path) {
        check(dc_save_snapshot(ctx_, m, path.c_str()));
    }
    void load_snapshot(int m, const std::string& path) {
        check(dc_load_snapshot(ctx_, m, path.c_str()));
    }
    void checkpoint_save(const std::string& dir, std::uint64_t filter_cycle) {
        check(dc_checkpoint_save(ctx_, dir.c_str(), filter_cycle));
    }
    std::uint64_t checkpoint_load(const std::string& dir) {
        std::uint64_t c = 0;
        check(dc_checkpoint_load(ctx_, dir.c_str(), &c));
        return c;
    }

    // SIR comparison: log-likelihoods of this context's members
    std::vector<double> pf_loglik(const std::vector<dc_obs>& obs, double r_hu = 1.0,
                                  double r_hv = 1.0) {
        std::vector<double> ll(n_);
        check(dc_pf_loglik(ctx_, obs.data(), static_cast<std::int32_t>(obs.size()), r_hu, r_hv,
                           ll.data()));
        return ll;
    }
    void resample(const std::vector<std::int32_t>& idx) { check(dc_resample_members(ctx_, idx.data())); }

    // drifter forecast error: {E, RMSE}
    std::pair<double, double> forecast_error(const std::vector<double>& truth_xy) {
        double e = 0.0, r = 0.0;
        check(dc_forecast_error(ctx_, truth_xy.data(), &e, &r, nullptr, nullptr));
        return {e, r};
    }
    // multi-GPU forecast statistics: this rank's drifters into device buffers for a gather
    void drifters_to_device(double* d_pos, std::int32_t* d_wind) {
        check(dc_drifters_get_device(ctx_, d_pos, d_wind));
    }

    void sync() { check(dc_sync(ctx_)); }

private:
    void check(dc_status st) {
        if (st) throw_status(st, dc_last_error(ctx_, nullptr, nullptr, nullptr, nullptr));
    }
    dc_config cfg_;
    int n_;
    dc_ctx* ctx_ = nullptr;
};

// forecast_error over drifter ensembles gathered from every rank (member-id order, device
// buffers): {E, RMSE}, bitwise equal to one context holding every member
inline std::pair<double, double> forecast_error_gathered(const dc_config& cfg, int device,
                                                         void* stream, int n_members, int n_d,
                                                         const double* d_pos,
                                                         const std::int32_t* d_wind,
                                                         const std::vector<double>& truth_xy) {
    double e = 0.0, r = 0.0;
    const dc_status st = dc_forecast_error_gathered(&cfg, device, stream, n_members, n_d, d_pos,
                                                    d_wind, truth_xy.data(), &e, &r, nullptr,
                                                    nullptr);
    if (st) throw_status(st, "dc_forecast_error_gathered failed");
    return {e, r};
}

} // namespace gpu
} // namespace driftcast
