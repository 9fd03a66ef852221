// cpp_driver_mgpu.cpp -- the multi-GPU C++ driver of the drop-in: one
// process per GPU, contiguous particle ranges, NCCL inside the library (dc_comm_attach).
//
//   cpp_driver_mgpu <world> <members_total> <cycles> <bootstrap_dir> [nx ny]
//
// Without RANK in the environment the program launches <world> copies of itself, rank r
// on GPU r % (visible devices), and waits for them (a torchrun / mpirun launch that sets
// RANK, WORLD_SIZE and LOCAL_RANK works the same way). Rank 0 creates the NCCL id and
// publishes it in <bootstrap_dir>/nccl_id (written to a temporary name, then renamed);
// the other ranks wait for the file. Every rank runs the same DA cycles (drifter copies,
// Philox model error, the two-stage IEWPF with the barrier exchange over NCCL), reading
// each cycle's diagnostics and forecast statistics through the pipelined readback.
// Rank 0 then replays the run in ONE context holding every member and checks that its own
// slice and the statistics are bitwise equal ("identical results for W workers",
// SPEC.md:624,634).
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "driftcast_gpu.hpp"

using namespace driftcast::gpu;

namespace {

std::vector<double> lattice(const dc_config& c, int nxp, int nyp, double shift) {
    std::vector<double> xy;
    const double lx = c.nx * c.dx, ly = c.ny * c.dy;
    for (int b = 0; b < nyp; ++b)
        for (int a = 0; a < nxp; ++a) {
            xy.push_back(std::fmod((a + 0.5) / nxp * lx + shift, lx));
            xy.push_back(std::fmod((b + 0.5) / nyp * ly + 0.5 * shift, ly));
        }
    return xy;
}

// observations of cycle c: the 8x8 lattice shifted a little per cycle, smooth values
std::vector<dc_obs> cycle_obs(const dc_config& cfg, int c) {
    const std::vector<double> xy = lattice(cfg, 8, 8, 700.0 * (c + 1));
    std::vector<dc_obs> o;
    for (size_t i = 0; i < xy.size() / 2; ++i)
        o.push_back(dc_obs{xy[2 * i], xy[2 * i + 1], 15.0 * std::sin(0.37 * i + c),
                           10.0 * std::cos(0.23 * i - c)});
    return o;
}

struct RunOut {
    std::vector<std::vector<float>> e, u, v;  // [member][cells]
    std::vector<double> E, R;                 // per cycle (rank 0)
    std::vector<double> c;                    // per member, last cycle
};

RunOut run(const dc_config& cfg, int M, std::int64_t base, int device, int cycles,
           const FilterOperators& ops, const std::uint8_t* nccl_id, int rank, int world,
           std::int64_t total) {
    Ensemble ens(cfg, M, base, device);
    if (nccl_id) ens.comm_attach(nccl_id, rank, world, total);
    ens.init_double_jet();
    const std::vector<double> lat = lattice(cfg, 8, 8, 0.0);
    std::vector<double> pos;
    for (int m = 0; m < M; ++m) pos.insert(pos.end(), lat.begin(), lat.end());
    ens.set_drifters(pos, 64);
    RunOut out;
    for (int c = 0; c < cycles; ++c) {
        ens.da_cycle(5, cycle_obs(cfg, c), ops, static_cast<std::uint64_t>(c));
        const std::vector<double> truth = lattice(cfg, 8, 8, 40.0 * (c + 1));
        ens.readback_enqueue(c % 2, &truth);
        if (c > 0) {
            auto r = ens.readback_wait((c - 1) % 2, 64);
            out.E.push_back(r.E);
            out.R.push_back(r.RMSE);
        }
    }
    auto r = ens.readback_wait((cycles - 1) % 2, 64);
    out.E.push_back(r.E);
    out.R.push_back(r.RMSE);
    for (auto& d : r.diag) out.c.push_back(d.c);
    for (int m = 0; m < M; ++m) {
        std::vector<float> e, u, v;
        double t = 0.0;
        ens.download(m, e, u, v, &t);
        out.e.push_back(std::move(e));
        out.u.push_back(std::move(u));
        out.v.push_back(std::move(v));
    }
    return out;
}

int launch_ranks(char** argv, int world) {
    int ndev = 1;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) ndev = 1;
    std::vector<pid_t> kids;
    for (int r = 0; r < world; ++r) {
        const pid_t p = fork();
        if (p == 0) {
            setenv("RANK", std::to_string(r).c_str(), 1);
            setenv("WORLD_SIZE", std::to_string(world).c_str(), 1);
            setenv("LOCAL_RANK", std::to_string(r % ndev).c_str(), 1);
            execv("/proc/self/exe", argv);
            std::perror("execv");
            _exit(127);
        }
        kids.push_back(p);
    }
    int rc = 0;
    for (pid_t p : kids) {
        int st = 0;
        waitpid(p, &st, 0);
        if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) rc = 1;
    }
    return rc;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s world members_total cycles bootstrap_dir [nx ny]\n", argv[0]);
        return 2;
    }
    const int world = std::atoi(argv[1]);
    const std::int64_t total = std::atoll(argv[2]);
    const int cycles = std::atoi(argv[3]);
    const std::string boot = argv[4];
    if (!std::getenv("RANK")) return launch_ranks(argv, world);
    const int rank = std::atoi(std::getenv("RANK"));
    const int device = std::getenv("LOCAL_RANK") ? std::atoi(std::getenv("LOCAL_RANK")) : 0;

    dc_config cfg = default_config();
    if (argc >= 7) {
        cfg.nx = std::atoi(argv[5]);
        cfg.ny = std::atoi(argv[6]);
        cfg.dx = cfg.dy = 2220.0 * 500 / cfg.nx;
        cfg.l0 = 0.75 * cfg.c_omega * cfg.dx;
    }
    const FilterOperators ops = precompute_filter_operators(cfg);
    const std::int64_t base = total * rank / world;
    const int M = static_cast<int>(total * (rank + 1) / world - base);

    // bootstrap: rank 0 publishes the NCCL id through the shared directory
    std::uint8_t id[DC_COMM_ID_BYTES];
    const std::string id_path = boot + "/nccl_id";
    if (rank == 0) {
        mkdir(boot.c_str(), 0755);
        if (dc_comm_unique_id(id) != DC_OK) {
            std::fprintf(stderr, "rank 0: dc_comm_unique_id failed\n");
            return 1;
        }
        const std::string tmp = id_path + ".tmp";
        std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(id), sizeof(id));
        std::rename(tmp.c_str(), id_path.c_str());
    } else {
        for (int i = 0;; ++i) {
            std::ifstream is(id_path, std::ios::binary);
            if (is.read(reinterpret_cast<char*>(id), sizeof(id))) break;
            if (i > 6000) {
                std::fprintf(stderr, "rank %d: no NCCL id after 60 s\n", rank);
                return 1;
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(10));
        }
    }
    RunOut got = run(cfg, M, base, device, cycles, ops, id, rank, world, total);
    if (rank != 0) return 0;
    std::remove(id_path.c_str());
    for (int c = 0; c < cycles; ++c)
        std::printf("cycle %d: E %.6f RMSE %.6f (%lld members on %d ranks)\n", c, got.E[c], got.R[c],
                    static_cast<long long>(total), world);
    // replay in one context holding every member, no communicator
    RunOut one = run(cfg, static_cast<int>(total), 0, device, cycles, ops, nullptr, 0, 1, total);
    bool same = true;
    for (int m = 0; m < M; ++m)
        same = same && got.e[m] == one.e[m] && got.u[m] == one.u[m] && got.v[m] == one.v[m] &&
               got.c[m] == one.c[m];
    for (int c = 0; c < cycles; ++c) same = same && got.E[c] == one.E[c] && got.R[c] == one.R[c];
    std::printf("rank 0 slice and statistics bitwise equal to one context: %s\n", same ? "yes" : "NO");
    return same ? 0 : 1;
}
