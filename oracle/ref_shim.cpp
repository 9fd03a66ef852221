// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/oracle_api.h).
//
// A thin extern "C" shim over the reference's own header-only operators, compiled
// unchanged from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libdcref.so (git-ignored; travels to the GPU box as a built artefact).
// Nothing here restates an algorithm: every entry point calls the reference operator
// named in its comment. It exists to (1) pin this repo's CPU restatement
// (oracle/dc_oracle.cpp) bit-for-bit, (2) generate tests/golden fixtures, and (3) serve
// as the reference CPU arm of bench.py.
//
// Build flags follow the reference Release build: -O3, no -march (so no FMA
// contraction; proj/CMakeLists.txt:8-10, proj/tools/CMakeLists.txt:3).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <istream>
#include <limits>
#include <ostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

// Expose Stepper internals (load / cfl_from_loaded / rk2_loaded) so the shim can
// report the per-substep dt sequence that Stepper::model_step (swe.hpp:244-259)
// takes. Standard headers are included first, so only the reference's classes are
// affected.
#define private public
#include "driftcast/grid.hpp"
#include "driftcast/field.hpp"
#include "driftcast/rng.hpp"
#include "driftcast/state.hpp"
#include "driftcast/swe.hpp"
#include "driftcast/stochastic.hpp"
#undef private

#include "oracle_api.h"

using namespace driftcast;

namespace {

enum { RS_OK = 0, RS_EINVAL = 1, RS_EDRY = 2, RS_ERUNTIME = 3 };

void put_err(char* err, int errlen, const char* msg) {
    if (err && errlen > 0) {
        std::strncpy(err, msg, static_cast<size_t>(errlen) - 1);
        err[errlen - 1] = '\0';
    }
}

template <class F>
int guarded(char* err, int errlen, F&& fn) {
    try {
        fn();
        return RS_OK;
    } catch (const DryCellError& e) {
        put_err(err, errlen, e.what());
        return RS_EDRY;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return RS_EINVAL;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return RS_ERUNTIME;
    }
}

ModelGrid grid_of(const orc_params* p) { return ModelGrid(p->nx, p->ny, p->dx, p->dy); }
PhysParams phys_of(const orc_params* p) { return PhysParams(p->g, p->f, p->h_eq); }
SchemeParams scheme_of(const orc_params* p) {
    return SchemeParams(p->courant, p->limiter_theta, p->model_dt);
}
ErrorParams err_of(const orc_params* p) {
    if (p->q0 == 0.0) return ErrorParams(0.0, p->l0 > 0.0 ? p->l0 : 1.0);
    return ErrorParams(p->q0, p->l0);
}

OceanState state_in(const ModelGrid& g, const float* eta, const float* hu, const float* hv,
                    double t) {
    OceanState s(g, t);
    const size_t n = static_cast<size_t>(g.nx) * g.ny;
    std::memcpy(s.eta.data(), eta, n * sizeof(float));
    std::memcpy(s.hu.data(), hu, n * sizeof(float));
    std::memcpy(s.hv.data(), hv, n * sizeof(float));
    return s;
}

void state_out(const OceanState& s, float* eta, float* hu, float* hv) {
    const size_t n = s.eta.size();
    std::memcpy(eta, s.eta.data(), n * sizeof(float));
    std::memcpy(hu, s.hu.data(), n * sizeof(float));
    std::memcpy(hv, s.hv.data(), n * sizeof(float));
}

} // namespace

extern "C" {

/// init_double_jet (swe.hpp:459-500) with default JetParams.
int ref_init_double_jet(const orc_params* p, float* eta, float* hu, float* hv, char* err,
                        int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        OceanState s = init_double_jet(g, phys_of(p));
        state_out(s, eta, hu, hv);
    });
}

/// save_snapshot (state.hpp:78-83) of one state to a file, the reference writer.
int ref_save_snapshot(const orc_params* p, const float* eta, const float* hu, const float* hv,
                      double t, const char* path, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        OceanState s = state_in(g, eta, hu, hv, t);
        save_snapshot(std::string(path), s);
    });
}

/// load_snapshot (state.hpp:110-114): fields out, *t; errors as the reference throws them.
int ref_load_snapshot(const orc_params* p, const char* path, float* eta, float* hu, float* hv,
                      double* t, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        OceanState s = load_snapshot(std::string(path));
        if (s.nx() != p->nx || s.ny() != p->ny)
            throw std::invalid_argument("ref_load_snapshot: extents differ from the params");
        state_out(s, eta, hu, hv);
        *t = s.t;
    });
}

/// n_steps calls of Stepper::model_step (swe.hpp:244-259) on one member.
int ref_model_step(const orc_params* p, float* eta, float* hu, float* hv, double* t,
                   int n_steps, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        Stepper st(g, phys_of(p), scheme_of(p));
        OceanState s = state_in(g, eta, hu, hv, *t);
        for (int i = 0; i < n_steps; ++i) st.model_step(s);
        state_out(s, eta, hu, hv);
        *t = s.t;
    });
}

/// The substep dt sequence of one Stepper::model_step, obtained by running the same
/// loop body (swe.hpp:248-257) through the exposed internals. Advances the state.
int ref_model_step_dts(const orc_params* p, float* eta, float* hu, float* hv, double* t,
                       double* dts, int max_dts, int* n_dts, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        Stepper st(g, phys_of(p), scheme_of(p));
        OceanState s = state_in(g, eta, hu, hv, *t);
        double remaining = st.scheme_.model_dt;
        const double t_end = s.t + st.scheme_.model_dt;
        int sub = 0;
        while (remaining > 0.0) {
            st.load(s);
            double dt = st.cfl_from_loaded();
            if (dt >= remaining) dt = remaining;
            st.rk2_loaded(s, dt, sub);
            remaining -= dt;
            if (sub < max_dts) dts[sub] = dt;
            ++sub;
        }
        s.t = t_end;
        *n_dts = sub;
        state_out(s, eta, hu, hv);
        *t = s.t;
    });
}

/// Stepper::flux_rhs (swe.hpp:229-239).
int ref_flux_rhs(const orc_params* p, const float* eta, const float* hu, const float* hv,
                 float* de, float* du, float* dv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        Stepper st(g, phys_of(p), scheme_of(p));
        OceanState s = state_in(g, eta, hu, hv, 0.0);
        FieldF a, b, c;
        st.flux_rhs(s, a, b, c);
        const size_t n = s.eta.size();
        std::memcpy(de, a.data(), n * sizeof(float));
        std::memcpy(du, b.data(), n * sizeof(float));
        std::memcpy(dv, c.data(), n * sizeof(float));
    });
}

/// Stepper::cfl_dt (swe.hpp:212-226), the public fp64 formula.
int ref_cfl_dt(const orc_params* p, const float* eta, const float* hu, const float* hv,
               double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        Stepper st(g, phys_of(p), scheme_of(p));
        OceanState s = state_in(g, eta, hu, hv, 0.0);
        *out = st.cfl_dt(s);
    });
}

/// n_draws calls of perturb_state (stochastic.hpp:164-173) with
/// NoiseStream(seed, tag, index) (rng.hpp:48-49). Also returns what each draw
/// consumed -- offsets (2 per draw) and xi (nxc*nyc per draw, b-outer/a-inner) -- by
/// replaying an identical copy of the stream through uniform_below / sample_xi.
int ref_perturb(const orc_params* p, uint64_t seed, uint64_t tag, uint64_t index,
                int n_draws, float* eta, float* hu, float* hv, int32_t* offsets_out,
                double* xi_out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        PhysParams ph = phys_of(p);
        CoarseGrid base(g, p->c_omega);
        ErrorParams ep = err_of(p);
        NoiseStream ns(seed, static_cast<StreamTag>(tag), index);
        NoiseStream replay = ns;
        OceanState s = state_in(g, eta, hu, hv, 0.0);
        const size_t nr = base.points();
        for (int d = 0; d < n_draws; ++d) {
            perturb_state(s, ns, ep, base, ph, g);
            if (ep.q0 == 0.0) continue;
            int oj = static_cast<int>(replay.uniform_below(base.c_omega));
            int ok = static_cast<int>(replay.uniform_below(base.c_omega));
            CoarseField xi = sample_xi(replay, CoarseGrid(g, base.c_omega, oj, ok));
            if (offsets_out) {
                offsets_out[2 * d] = oj;
                offsets_out[2 * d + 1] = ok;
            }
            if (xi_out) std::memcpy(xi_out + d * nr, xi.values.data(), nr * sizeof(double));
        }
        state_out(s, eta, hu, hv);
    });
}

/// add_q_half (stochastic.hpp:144-160) of a host-given coarse field on offset (oj,ok).
int ref_add_q_half(const orc_params* p, int oj, int ok, const double* coarse, double scale,
                   float* eta, float* hu, float* hv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid cg(g, p->c_omega, oj, ok);
        CoarseField cf(cg);
        std::memcpy(cf.values.data(), coarse, cg.points() * sizeof(double));
        OceanState s = state_in(g, eta, hu, hv, 0.0);
        add_q_half(s, cf, err_of(p), phys_of(p), g, scale);
        state_out(s, eta, hu, hv);
    });
}

/// apply_soar (stochastic.hpp:49-69).
int ref_apply_soar(const orc_params* p, int oj, int ok, const double* in, double* out,
                   char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid cg(g, p->c_omega, oj, ok);
        CoarseField cf(cg);
        std::memcpy(cf.values.data(), in, cg.points() * sizeof(double));
        CoarseField r = apply_soar(cf, err_of(p));
        std::memcpy(out, r.values.data(), cg.points() * sizeof(double));
    });
}

/// interpolate_bicubic (stochastic.hpp:93-118).
int ref_interpolate_bicubic(const orc_params* p, int oj, int ok, const double* coarse,
                            double* fine, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid cg(g, p->c_omega, oj, ok);
        CoarseField cf(cg);
        std::memcpy(cf.values.data(), coarse, cg.points() * sizeof(double));
        FieldD r = interpolate_bicubic(cf, g);
        std::memcpy(fine, r.data(), r.size() * sizeof(double));
    });
}

/// geostrophic_balance (stochastic.hpp:122-139).
int ref_geostrophic_balance(const orc_params* p, const double* deta, double* dhu,
                            double* dhv, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        FieldD e(g.nx, g.ny), u, v;
        std::memcpy(e.data(), deta, e.size() * sizeof(double));
        geostrophic_balance(e, phys_of(p), g, u, v);
        std::memcpy(dhu, u.data(), u.size() * sizeof(double));
        std::memcpy(dhv, v.data(), v.size() * sizeof(double));
    });
}

/// apply_q_half_T (stochastic.hpp:193-202) for observation cell (j,k). If align != 0
/// the coarse grid is first aligned with align_coarse_offset (grid.hpp:113-117);
/// otherwise (oj,ok) is used as given (and a non-co-located cell throws).
int ref_apply_q_half_T(const orc_params* p, double y_hu, double y_hv, int j, int k,
                       int align, int oj, int ok, double* out, int32_t* offsets_out,
                       char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid base(g, p->c_omega, align ? 0 : oj, align ? 0 : ok);
        CoarseGrid cg = align ? align_coarse_offset({j, k}, base, g) : base;
        CoarseField r = apply_q_half_T(y_hu, y_hv, {j, k}, cg, err_of(p), phys_of(p));
        std::memcpy(out, r.values.data(), cg.points() * sizeof(double));
        if (offsets_out) {
            offsets_out[0] = cg.offset_j;
            offsets_out[1] = cg.offset_k;
        }
    });
}

/// adjoint_geo_balance (stochastic.hpp:178-188) on offset (oj,ok).
int ref_adjoint_geo_balance(const orc_params* p, double y_hu, double y_hv, int a, int b,
                            int oj, int ok, double* out, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid cg(g, p->c_omega, oj, ok);
        CoarseField r = adjoint_geo_balance(y_hu, y_hv, a, b, phys_of(p), cg);
        std::memcpy(out, r.values.data(), cg.points() * sizeof(double));
    });
}

/// locate_cell (grid.hpp:55-69).
int ref_locate_cell(const orc_params* p, double x, double y, int32_t* j, int32_t* k,
                    char* err, int errlen) {
    return guarded(err, errlen, [&] {
        auto c = locate_cell(x, y, grid_of(p));
        *j = c.first;
        *k = c.second;
    });
}

/// align_coarse_offset (grid.hpp:113-117).
int ref_align_coarse_offset(const orc_params* p, int j, int k, int32_t* oj, int32_t* ok,
                            char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        CoarseGrid cg = align_coarse_offset({j, k}, CoarseGrid(g, p->c_omega), g);
        *oj = cg.offset_j;
        *ok = cg.offset_k;
    });
}

/// soar_kernel (stochastic.hpp:43-45).
double ref_soar_kernel(const orc_params* p, double dist) { return soar_kernel(dist, err_of(p)); }

/// stream_seed (rng.hpp:35-40).
uint64_t ref_stream_seed(uint64_t master, uint64_t tag, uint64_t index) {
    return stream_seed(master, static_cast<StreamTag>(tag), index);
}

/// n draws of NoiseStream::normal (rng.hpp:69-84) from NoiseStream(seed, tag, index).
void ref_noise_normals(uint64_t seed, uint64_t tag, uint64_t index, int n, double* out) {
    NoiseStream ns(seed, static_cast<StreamTag>(tag), index);
    for (int i = 0; i < n; ++i) out[i] = ns.normal();
}

/// n draws of NoiseStream::uniform_below(range) (rng.hpp:57-66).
void ref_noise_uniform_below(uint64_t seed, uint64_t tag, uint64_t index, uint64_t range,
                             int n, uint64_t* out) {
    NoiseStream ns(seed, static_cast<StreamTag>(tag), index);
    for (int i = 0; i < n; ++i) out[i] = ns.uniform_below(range);
}

/// Threaded ensemble forecast on the reference operators, the CPU baseline of
/// bench.py: n_members members (state arrays member-major, each row-major k*nx+j) are
/// strided over n_threads workers, each owning one Stepper (swe.hpp:435-436; the
/// SPEC.md:634 work-pool model). Per member, per step s: Stepper::model_step, then
/// perturb_state with that member's NoiseStream(seed, model_error, member_base+i)
/// when perturb_after[s] != 0 (stochastic.hpp:164). Returns wall seconds.
int ref_forecast_threads(const orc_params* p, int n_members, uint64_t member_base, int n_steps,
                         const uint8_t* perturb_after, int n_threads, float* eta, float* hu,
                         float* hv, double* elapsed_s, char* err, int errlen) {
    return guarded(err, errlen, [&] {
        ModelGrid g = grid_of(p);
        PhysParams ph = phys_of(p);
        SchemeParams sc = scheme_of(p);
        ErrorParams ep = err_of(p);
        CoarseGrid base(g, p->c_omega);
        const size_t n = static_cast<size_t>(g.nx) * g.ny;
        std::vector<OceanState> states;
        std::vector<NoiseStream> streams;
        states.reserve(n_members);
        for (int m = 0; m < n_members; ++m) {
            states.push_back(state_in(g, eta + m * n, hu + m * n, hv + m * n, 0.0));
            streams.emplace_back(p->seed, StreamTag::model_error, member_base + m);
        }
        std::atomic<int> failed{0};
        std::string first_err;
        auto t0 = std::chrono::steady_clock::now();
        auto worker = [&](int w) {
            Stepper st(g, ph, sc);
            try {
                for (int m = w; m < n_members; m += n_threads)
                    for (int s = 0; s < n_steps; ++s) {
                        st.model_step(states[m]);
                        if (perturb_after[s]) perturb_state(states[m], streams[m], ep, base, ph, g);
                    }
            } catch (const std::exception& e) {
                if (failed.fetch_add(1) == 0) first_err = e.what();
            }
        };
        std::vector<std::thread> pool;
        for (int w = 0; w < n_threads; ++w) pool.emplace_back(worker, w);
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        *elapsed_s = std::chrono::duration<double>(t1 - t0).count();
        if (failed.load()) throw std::runtime_error(first_err);
        for (int m = 0; m < n_members; ++m)
            state_out(states[m], eta + m * n, hu + m * n, hv + m * n);
    });
}

} // extern "C"
