// cpp_driver_example.cpp -- the C++ driver side of the drop-in: runs a few DA cycles of
// the paper setup through include/driftcast_gpu.hpp and prints per-cycle diagnostics.
// Build (add -I<reference>/proj/include -std=c++20 to throw the
// reference's own driftcast::DryCellError):
//   g++ -std=c++17 -O2 -Iinclude tools/cpp_driver_example.cpp
//       -Lpaper_1910_01031_b200 -ldriftcast_gpu -Wl,-rpath,$PWD/paper_1910_01031_b200
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "driftcast_gpu.hpp"

int main(int argc, char** argv) {
    using namespace driftcast::gpu;
    const int members = argc > 1 ? std::atoi(argv[1]) : 16;
    const int cycles = argc > 2 ? std::atoi(argv[2]) : 2;
    dc_config cfg = default_config();
    FilterOperators ops = precompute_filter_operators(cfg);
    std::printf("S = [%.6f %.3g; %.3g %.6f]\n", ops.S[0], ops.S[1], ops.S[2], ops.S[3]);

    Ensemble ens(cfg, members);
    ens.init_double_jet();
    // 64 drifters on an 8x8 lattice, copied into every member
    std::vector<double> pos;
    const double lx = cfg.nx * cfg.dx, ly = cfg.ny * cfg.dy;
    for (int i = 0; i < members; ++i)
        for (int b = 0; b < 8; ++b)
            for (int a = 0; a < 8; ++a) {
                pos.push_back((a + 0.5) / 8 * lx);
                pos.push_back((b + 0.5) / 8 * ly);
            }
    ens.set_drifters(pos, 64);
    std::vector<dc_obs> obs;
    for (int b = 0; b < 8; ++b)
        for (int a = 0; a < 8; ++a)
            obs.push_back(dc_obs{(a + 0.5) / 8 * lx, (b + 0.5) / 8 * ly, 20.0 * std::sin(a + b), 5.0});
    for (int c = 0; c < cycles; ++c) {
        ens.da_cycle(5, obs, ops, static_cast<std::uint64_t>(c));
        double wb[2];
        auto d = ens.diagnostics(wb);
        double amin = 1.0, amax = 0.0;
        for (auto& x : d) {
            amin = std::fmin(amin, x.alpha);
            amax = std::fmax(amax, x.alpha);
        }
        std::printf("cycle %d: w_target %.4f beta %.6f alpha in [%.6f, %.6f]\n", c, wb[0], wb[1],
                    amin, amax);
    }
    std::vector<float> e, u, v;
    double t = 0.0;
    ens.download(0, e, u, v, &t);
    std::printf("t = %.1f s, eta[0] = %.6e\n", t, e[0]);
    // checkpoint, continue one cycle, restore, repeat it: the two runs agree bit for bit
    const char* dir = argc > 3 ? argv[3] : "/tmp/dc_cpp_checkpoint";
    ens.checkpoint_save(dir, static_cast<std::uint64_t>(cycles));
    ens.da_cycle(5, obs, ops, static_cast<std::uint64_t>(cycles));
    std::vector<float> e1, u1, v1;
    ens.download(members - 1, e1, u1, v1, &t);
    const std::uint64_t c0 = ens.checkpoint_load(dir);
    ens.da_cycle(5, obs, ops, c0);
    std::vector<float> e2, u2, v2;
    ens.download(members - 1, e2, u2, v2, &t);
    std::printf("restart from checkpoint reproduces the run: %s\n",
                (e1 == e2 && u1 == u2 && v1 == v2) ? "yes" : "NO");
    // SIR comparison: standard PF log-likelihoods of the members
    const std::vector<double> ll = ens.pf_loglik(obs);
    double lmax = -1e300;
    for (double x : ll) lmax = std::fmax(lmax, x);
    std::printf("max PF log-likelihood %.3f\n", lmax);
    // the reference's exception types come back through the shim
    try {
        dc_config bad = cfg;
        bad.c_omega = 4;
        Ensemble oops(bad, 2);
    } catch (const std::invalid_argument& ex) {
        std::printf("invalid_argument caught as expected\n");
    }
    return 0;
}
