// truth.cpp -- generate_truth on the GPU, host C++ over the C ABI.
//
// One-member context on the truth stream family (StreamTag truth_model_error, particle 0:
// SURVEY.md §8d), stepped with model error after every model step. Drifters (lattice,
// advected in the truth) and moorings start observing at the insertion time; every
// observation interval each platform writes one record:
//   drifters: observe_drifter, displacement since the previous record
//   moorings: observe_mooring
// plus eps ~ N(0, R) from the obs_noise streams (observation index = record count).
// Output: dir/observations.txt (SPEC.md:401 grammar) and dir/truth_<t>.dcst snapshots.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/driftcast_gpu.h"

namespace {

std::vector<double> lattice(int nx_p, int ny_p, double lx, double ly) {
    std::vector<double> xy;
    for (int b = 0; b < ny_p; ++b)
        for (int a = 0; a < nx_p; ++a) {
            xy.push_back((a + 0.5) / nx_p * lx);
            xy.push_back((b + 0.5) / ny_p * ly);
        }
    return xy;
}

long long steps_of(double seconds, double dt) { return std::llround(seconds / dt); }

} // namespace

extern "C" {

dc_status dc_generate_truth(const dc_config* cfg, const dc_truth_plan* plan, const char* dir,
                            int32_t device, int64_t* n_records) {
    if (!cfg || !plan || !dir) return DC_EINVAL;
    if (n_records) *n_records = 0;
    const double dt = cfg->model_dt;
    const long long n_steps = steps_of(plan->duration, dt);
    const long long ins = steps_of(plan->insert_time, dt);
    const long long every = steps_of(plan->obs_interval, dt);
    const long long snap = plan->snapshot_interval > 0 ? steps_of(plan->snapshot_interval, dt) : 0;
    if (n_steps < 0 || ins < 0 || every <= 0 ||
        std::fabs(every * dt - plan->obs_interval) > 1e-9 * plan->obs_interval)
        return DC_EINVAL;  // cadence must be a multiple of model_dt (SPEC.md ExperimentPlan)
    dc_ctx* ctx = nullptr;
    dc_status st = dc_create(cfg, 1, 0, device, nullptr, &ctx);
    if (st) return st;
    auto fail = [&](dc_status s) {
        dc_destroy(ctx);
        return s;
    };
    if ((st = dc_set_model_error_tag(ctx, 3))) return fail(st);
    if ((st = dc_init_double_jet(ctx))) return fail(st);
    const std::string d(dir);
    auto snapshot = [&](long long step) {
        return dc_save_snapshot(ctx, 0, (d + "/truth_" + std::to_string(step * (long long)dt) +
                                         ".dcst").c_str());
    };
    if ((st = snapshot(0))) return fail(st);
    const double lx = cfg->nx * cfg->dx, ly = cfg->ny * cfg->dy;
    const int nd = plan->drifters_x * plan->drifters_y;
    const int nm = plan->moorings_x * plan->moorings_y;
    const std::vector<double> moor = lattice(plan->moorings_x, plan->moorings_y, lx, ly);
    std::vector<double> prev, cur(2 * static_cast<size_t>(nd)), y, eps;
    std::vector<int32_t> ids, wind(2 * static_cast<size_t>(nd));
    std::vector<dc_obs_record> recs;
    uint64_t obs_index = 0;
    bool drifting = false;
    const std::string obs_path = d + "/observations.txt";
    if ((st = dc_obs_file_write(obs_path.c_str(), nullptr, 0, 0))) return fail(st);
    for (long long s = 0; s <= n_steps; ++s) {
        if (s == ins && nd > 0) {  // platforms inserted
            prev = lattice(plan->drifters_x, plan->drifters_y, lx, ly);
            if ((st = dc_drifters_set(ctx, prev.data(), nd))) return fail(st);
            drifting = true;
        }
        if (s > ins && (s - ins) % every == 0) {  // an observation time
            recs.clear();
            const double t = s * dt;
            if (nd > 0) {
                if ((st = dc_drifters_get(ctx, cur.data(), wind.data()))) return fail(st);
                ids.resize(nd);
                for (int i = 0; i < nd; ++i) ids[i] = i;
                eps.resize(2 * static_cast<size_t>(nd));
                y.resize(2 * static_cast<size_t>(nd));
                if ((st = dc_obs_noise(ctx, 0, ids.data(), nd, obs_index, plan->r_hu, plan->r_hv,
                                       eps.data())))
                    return fail(st);
                if ((st = dc_observe_drifters(ctx, prev.data(), cur.data(), nd, every * dt,
                                              eps.data(), y.data())))
                    return fail(st);
                for (int i = 0; i < nd; ++i)
                    recs.push_back({t, 0, i, cur[2 * i], cur[2 * i + 1], y[2 * i], y[2 * i + 1]});
                prev = cur;
            }
            if (nm > 0) {
                ids.resize(nm);
                for (int i = 0; i < nm; ++i) ids[i] = i;
                eps.resize(2 * static_cast<size_t>(nm));
                y.resize(2 * static_cast<size_t>(nm));
                if ((st = dc_obs_noise(ctx, 1, ids.data(), nm, obs_index, plan->r_hu, plan->r_hv,
                                       eps.data())))
                    return fail(st);
                if ((st = dc_observe_mooring(ctx, 0, moor.data(), nm, y.data()))) return fail(st);
                for (int i = 0; i < nm; ++i)
                    recs.push_back({t, 1, i, moor[2 * i], moor[2 * i + 1], y[2 * i] + eps[2 * i],
                                    y[2 * i + 1] + eps[2 * i + 1]});
            }
            if ((st = dc_obs_file_write(obs_path.c_str(), recs.data(),
                                        static_cast<int32_t>(recs.size()), 1)))
                return fail(st);
            if (n_records) *n_records += static_cast<int64_t>(recs.size());
            ++obs_index;
        }
        if (snap > 0 && s > 0 && s % snap == 0 && (st = snapshot(s))) return fail(st);
        if (s == n_steps) break;
        // one model step of the truth: drifters with the state at the start of the
        // interval, the step, then model error (truth stream)
        if (drifting && (st = dc_drifters_advect(ctx, dt))) return fail(st);
        if ((st = dc_step(ctx, 1))) return fail(st);
        if ((st = dc_perturb(ctx, DC_NOISE_PHILOX, nullptr, nullptr))) return fail(st);
    }
    if (snap == 0 && n_steps > 0 && (st = snapshot(n_steps))) return fail(st);
    if ((st = dc_sync(ctx))) return fail(st);
    dc_destroy(ctx);
    return DC_OK;
}

} // extern "C"
