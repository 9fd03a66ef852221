// io.cpp -- DCST snapshots and ensemble checkpoints (host C++ over the C ABI).
//
// Snapshot format: state.hpp:43-116 (save_snapshot / load_snapshot), byte for byte:
//   "DCST" | u32 version (1) | u32 nx | u32 ny | f64 t | eta f32[nx*ny] | hu | hv
// little endian, Field2D row-major with j fastest. Errors carry the reference's messages.
//
// Checkpoint directory: SPEC.md ensemble_engine "External Interfaces" --
//   dir/ensemble/particle_<i>.dcst  (global particle id i)
//   dir/rng_state.txt               (the counter-based RNG state: master seed, model-error
//                                    draw counter, filter cycle)
//   dir/meta.txt                    (parameter echo)
#include <sys/stat.h>
#include <sys/types.h>

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/driftcast_gpu.h"

namespace dcg {
dc_status ctx_error(dc_ctx* ctx, dc_status st, const std::string& msg, int m);
}

namespace {

constexpr uint32_t kSnapshotVersion = 1;  // state.hpp:49

static_assert(sizeof(float) == 4 && sizeof(double) == 8, "IEEE types");

bool little_endian() {
    const uint16_t one = 1;
    unsigned char b;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

template <typename T>
void put(std::ostream& os, const T& v) {
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <typename T>
bool get(std::istream& is, T* v) {
    is.read(reinterpret_cast<char*>(v), sizeof(T));
    return static_cast<bool>(is);
}

struct Member {
    std::vector<float> eta, hu, hv;
    double t = 0.0;
};

dc_status write_snapshot(dc_ctx* ctx, const std::string& path, int nx, int ny, const Member& s) {
    std::ofstream os(path, std::ios::binary);
    if (!os) return dcg::ctx_error(ctx, DC_EIO, "snapshot: cannot open " + path, -1);
    os.write("DCST", 4);
    put(os, kSnapshotVersion);
    put(os, static_cast<uint32_t>(nx));
    put(os, static_cast<uint32_t>(ny));
    put(os, s.t);
    for (const std::vector<float>* f : {&s.eta, &s.hu, &s.hv})
        os.write(reinterpret_cast<const char*>(f->data()),
                 static_cast<std::streamsize>(f->size() * sizeof(float)));
    if (!os) return dcg::ctx_error(ctx, DC_EIO, "snapshot: write failed", -1);
    return DC_OK;
}

// load_snapshot (state.hpp:93-114) with the same checks, then the context's extent check
dc_status read_snapshot(dc_ctx* ctx, const std::string& path, int nx, int ny, Member* s) {
    std::ifstream is(path, std::ios::binary);
    if (!is) return dcg::ctx_error(ctx, DC_EIO, "snapshot: cannot open " + path, -1);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, "DCST", 4) != 0)
        return dcg::ctx_error(ctx, DC_EIO, "snapshot: bad magic", -1);
    uint32_t version = 0, fnx = 0, fny = 0;
    if (!get(is, &version)) return dcg::ctx_error(ctx, DC_EIO, "snapshot: truncated stream", -1);
    if (version != kSnapshotVersion)
        return dcg::ctx_error(ctx, DC_EIO,
                              "snapshot: unsupported version " + std::to_string(version), -1);
    if (!get(is, &fnx) || !get(is, &fny))
        return dcg::ctx_error(ctx, DC_EIO, "snapshot: truncated stream", -1);
    if (fnx == 0 || fny == 0 || fnx > (1u << 20) || fny > (1u << 20))
        return dcg::ctx_error(ctx, DC_EIO, "snapshot: implausible extents", -1);
    if (!get(is, &s->t)) return dcg::ctx_error(ctx, DC_EIO, "snapshot: truncated stream", -1);
    if (static_cast<int>(fnx) != nx || static_cast<int>(fny) != ny)
        return dcg::ctx_error(ctx, DC_EINVAL,
                              "snapshot: extents " + std::to_string(fnx) + "x" +
                                  std::to_string(fny) + " do not match the grid " +
                                  std::to_string(nx) + "x" + std::to_string(ny),
                              -1);
    const size_t n = static_cast<size_t>(nx) * ny;
    for (std::vector<float>* f : {&s->eta, &s->hu, &s->hv}) {
        f->assign(n, 0.0f);
        is.read(reinterpret_cast<char*>(f->data()), static_cast<std::streamsize>(n * sizeof(float)));
        if (!is) return dcg::ctx_error(ctx, DC_EIO, "snapshot: truncated field data", -1);
    }
    return DC_OK;
}

bool make_dir(const std::string& d) {
    if (mkdir(d.c_str(), 0755) == 0 || errno == EEXIST) {
        struct stat st;
        return stat(d.c_str(), &st) == 0 && S_ISDIR(st.st_mode);
    }
    return false;
}

std::string particle_path(const std::string& dir, int64_t id) {
    return dir + "/ensemble/particle_" + std::to_string(id) + ".dcst";
}

std::string drifters_path(const std::string& dir, int64_t id) {
    return dir + "/ensemble/particle_" + std::to_string(id) + ".drifters";
}

std::string rng_path(const std::string& dir, int64_t first) {
    return dir + "/rng_state_" + std::to_string(first) + ".txt";
}

std::string fmt17(double v) {
    char b[40];
    std::snprintf(b, sizeof(b), "%.17g", v);
    return b;
}

} // namespace

extern "C" {

dc_status dc_save_snapshot(dc_ctx* ctx, int32_t m, const char* path) {
    if (!ctx || !path) return DC_ESTATE;
    if (!little_endian()) return dcg::ctx_error(ctx, DC_EIO, "snapshot: big-endian host", -1);
    dc_config cfg;
    int32_t M = 0;
    dc_get_config(ctx, &cfg, &M, nullptr);
    if (m < 0 || m >= M) return dcg::ctx_error(ctx, DC_ESTATE, "member index out of range", m);
    Member s;
    const size_t n = static_cast<size_t>(cfg.nx) * cfg.ny;
    s.eta.resize(n);
    s.hu.resize(n);
    s.hv.resize(n);
    dc_status st = dc_download_member(ctx, m, s.eta.data(), s.hu.data(), s.hv.data(), &s.t);
    if (st) return st;
    return write_snapshot(ctx, path, cfg.nx, cfg.ny, s);
}

dc_status dc_load_snapshot(dc_ctx* ctx, int32_t m, const char* path) {
    if (!ctx || !path) return DC_ESTATE;
    dc_config cfg;
    int32_t M = 0;
    dc_get_config(ctx, &cfg, &M, nullptr);
    if (m < 0 || m >= M) return dcg::ctx_error(ctx, DC_ESTATE, "member index out of range", m);
    Member s;
    dc_status st = read_snapshot(ctx, path, cfg.nx, cfg.ny, &s);
    if (st) return st;
    return dc_upload_member(ctx, m, s.eta.data(), s.hu.data(), s.hv.data(), s.t);
}

dc_status dc_checkpoint_save(dc_ctx* ctx, const char* dir, uint64_t filter_cycle) {
    if (!ctx || !dir) return DC_ESTATE;
    if (!little_endian()) return dcg::ctx_error(ctx, DC_EIO, "snapshot: big-endian host", -1);
    const std::string d(dir);
    if (!make_dir(d) || !make_dir(d + "/ensemble"))
        return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot create " + d + "/ensemble", -1);
    dc_config cfg;
    int32_t M = 0;
    int64_t base = 0;
    dc_get_config(ctx, &cfg, &M, &base);
    const size_t n = static_cast<size_t>(cfg.nx) * cfg.ny;
    // one batched download of the whole slice, then the per-particle files
    std::vector<float> e(n * M), u(n * M), v(n * M);
    std::vector<double> t(M);
    dc_status st = dc_download_all(ctx, e.data(), u.data(), v.data(), t.data());
    if (st) return st;
    Member s;
    for (int m = 0; m < M; ++m) {
        s.eta.assign(e.begin() + m * n, e.begin() + (m + 1) * n);
        s.hu.assign(u.begin() + m * n, u.begin() + (m + 1) * n);
        s.hv.assign(v.begin() + m * n, v.begin() + (m + 1) * n);
        s.t = t[m];
        st = write_snapshot(ctx, particle_path(d, base + m), cfg.nx, cfg.ny, s);
        if (st) return st;
    }
    // drifter copies with their winding counts (dc_da_cycle advects them: a resume
    // without them would not be bitwise)
    int32_t n_d = 0;
    if (dc_drifters_count(ctx, &n_d) == DC_OK && n_d > 0) {
        std::vector<double> pos(static_cast<size_t>(M) * n_d * 2);
        std::vector<int32_t> wind(pos.size());
        st = dc_drifters_get(ctx, pos.data(), wind.data());
        if (st) return st;
        for (int m = 0; m < M; ++m) {
            std::ofstream os(drifters_path(d, base + m));
            for (int q = 0; q < n_d; ++q) {
                const size_t i = (static_cast<size_t>(m) * n_d + q) * 2;
                os << q << "," << fmt17(pos[i]) << "," << fmt17(pos[i + 1]) << "," << wind[i]
                   << "," << wind[i + 1] << "\n";
            }
            if (!os) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot write drifters", -1);
        }
    }
    uint64_t draw = 0, tag = 1;
    int32_t mode = 0;
    dc_get_draw_counter(ctx, &draw);
    dc_get_model_error_tag(ctx, &tag);
    dc_iewpf_get_mode(ctx, &mode);
    {
        std::ofstream os(rng_path(d, base));
        os << "seed " << cfg.seed << "\n"
           << "model_error_draw " << draw << "\n"
           << "model_error_tag " << tag << "\n"
           << "filter_cycle " << filter_cycle << "\n"
           << "iewpf_mode " << mode << "\n"
           << "drifters " << n_d << "\n";
        if (!os) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot write rng_state", -1);
    }
    {
        std::ofstream os(d + "/meta.txt");
        os << "format driftcast-b200 checkpoint 1\n"
           << "nx " << cfg.nx << "\nny " << cfg.ny << "\ndx " << fmt17(cfg.dx) << "\ndy "
           << fmt17(cfg.dy) << "\ng " << fmt17(cfg.g) << "\nf " << fmt17(cfg.f) << "\nh_eq "
           << fmt17(cfg.h_eq) << "\ncourant " << fmt17(cfg.courant) << "\nlimiter_theta "
           << fmt17(cfg.limiter_theta) << "\nmodel_dt " << fmt17(cfg.model_dt) << "\nq0 "
           << fmt17(cfg.q0) << "\nl0 " << fmt17(cfg.l0) << "\nc_omega " << cfg.c_omega
           << "\nc_soar " << cfg.c_soar << "\nseed " << cfg.seed << "\nmember_base " << base
           << "\nn_members " << M << "\n";
        if (!os) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot write meta.txt", -1);
    }
    return DC_OK;
}

// ---- observation file: time,kind,id,x,y,y_hu,y_hv, %.17g round trip ----
dc_status dc_obs_file_write(const char* path, const dc_obs_record* recs, int32_t n,
                            int32_t append) {
    if (!path || (n > 0 && !recs)) return DC_EINVAL;
    std::FILE* f = std::fopen(path, append ? "a" : "w");
    if (!f) return DC_EIO;
    for (int i = 0; i < n; ++i) {
        const dc_obs_record& r = recs[i];
        if (r.kind != 0 && r.kind != 1) {
            std::fclose(f);
            return DC_EINVAL;
        }
        std::fprintf(f, "%.17g,%s,%d,%.17g,%.17g,%.17g,%.17g\n", r.time,
                     r.kind == 0 ? "drifter" : "mooring", r.id, r.x, r.y, r.y_hu, r.y_hv);
    }
    const bool ok = std::ferror(f) == 0;
    return (std::fclose(f) == 0 && ok) ? DC_OK : DC_EIO;
}

dc_status dc_obs_file_read(const char* path, dc_obs_record* recs, int32_t capacity,
                           int32_t* n_out) {
    if (!path || !n_out) return DC_EINVAL;
    std::ifstream is(path);
    if (!is) return DC_EIO;
    std::string line;
    int32_t n = 0;
    while (std::getline(is, line)) {
        if (line.empty()) continue;
        std::vector<std::string> tok;
        std::stringstream ss(line);
        std::string t;
        while (std::getline(ss, t, ',')) tok.push_back(t);
        if (tok.size() != 7) return DC_EIO;
        dc_obs_record r{};
        char* end = nullptr;
        r.time = std::strtod(tok[0].c_str(), &end);
        if (*end) return DC_EIO;
        if (tok[1] == "drifter") r.kind = 0;
        else if (tok[1] == "mooring") r.kind = 1;
        else return DC_EIO;
        r.id = static_cast<int32_t>(std::strtol(tok[2].c_str(), &end, 10));
        if (*end) return DC_EIO;
        double* dst[4] = {&r.x, &r.y, &r.y_hu, &r.y_hv};
        for (int k = 0; k < 4; ++k) {
            *dst[k] = std::strtod(tok[3 + k].c_str(), &end);
            if (*end) return DC_EIO;
        }
        if (recs && n < capacity) recs[n] = r;
        ++n;
    }
    *n_out = n;
    return (recs && n > capacity) ? DC_EINVAL : DC_OK;
}

// ---- trajectory output: time,particle,drifter,x,y,wind_x,wind_y ----
dc_status dc_trajectory_write(dc_ctx* ctx, const char* path, double time, int32_t append) {
    if (!ctx || !path) return DC_ESTATE;
    dc_config cfg;
    int32_t M = 0;
    int64_t base = 0;
    dc_get_config(ctx, &cfg, &M, &base);
    int32_t n_d = 0;
    dc_status st = dc_drifters_count(ctx, &n_d);
    if (st) return st;
    std::vector<double> pos(static_cast<size_t>(M) * n_d * 2);
    std::vector<int32_t> wind(pos.size());
    st = dc_drifters_get(ctx, pos.data(), wind.data());
    if (st) return st;
    std::FILE* f = std::fopen(path, append ? "a" : "w");
    if (!f) return dcg::ctx_error(ctx, DC_EIO, std::string("trajectory: cannot open ") + path, -1);
    for (int m = 0; m < M; ++m)
        for (int d = 0; d < n_d; ++d) {
            const size_t q = (static_cast<size_t>(m) * n_d + d) * 2;
            std::fprintf(f, "%.17g,%lld,%d,%.17g,%.17g,%d,%d\n", time,
                         static_cast<long long>(base + m), d, pos[q], pos[q + 1], wind[q],
                         wind[q + 1]);
        }
    const bool ok = std::ferror(f) == 0;
    if (std::fclose(f) != 0 || !ok)
        return dcg::ctx_error(ctx, DC_EIO, "trajectory: write failed", -1);
    return DC_OK;
}

// ---- per-cycle IEWPF diagnostics (SPEC.md iewpf_filter External Interfaces) ----
// lines "cycle,particle,c,gamma,zeta,alpha,beta,w_target" for the context's members
dc_status dc_iewpf_diagnostics_write(dc_ctx* ctx, const char* path, uint64_t cycle,
                                     int32_t append) {
    if (!ctx || !path) return DC_ESTATE;
    int32_t M = 0;
    int64_t base = 0;
    dc_get_config(ctx, nullptr, &M, &base);
    std::vector<dc_particle_diag> d(M);
    double wb[2] = {0.0, 0.0};
    dc_status st = dc_iewpf_diagnostics(ctx, d.data(), wb);
    if (st) return st;
    std::FILE* f = std::fopen(path, append ? "a" : "w");
    if (!f) return dcg::ctx_error(ctx, DC_EIO, std::string("diagnostics: cannot open ") + path, -1);
    for (int m = 0; m < M; ++m)
        std::fprintf(f, "%llu,%lld,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n",
                     static_cast<unsigned long long>(cycle), static_cast<long long>(base + m),
                     d[m].c, d[m].gamma, d[m].zeta, d[m].alpha, wb[1], wb[0]);
    const bool ok = std::ferror(f) == 0;
    if (std::fclose(f) != 0 || !ok)
        return dcg::ctx_error(ctx, DC_EIO, "diagnostics: write failed", -1);
    return DC_OK;
}

dc_status dc_checkpoint_load(dc_ctx* ctx, const char* dir, uint64_t* filter_cycle) {
    if (!ctx || !dir) return DC_ESTATE;
    const std::string d(dir);
    dc_config cfg;
    int32_t M = 0;
    int64_t base = 0;
    dc_get_config(ctx, &cfg, &M, &base);
    uint64_t seed = 0, draw = 0, cycle = 0, tag = 1, mode = 0, n_d = 0;
    {
        std::ifstream is(rng_path(d, base));
        if (!is) is.open(d + "/rng_state.txt");
        if (!is) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot open rng_state", -1);
        std::string key;
        uint64_t val = 0;
        int seen = 0;
        while (is >> key >> val) {
            if (key == "seed") seed = val, seen |= 1;
            else if (key == "model_error_draw") draw = val, seen |= 2;
            else if (key == "filter_cycle") cycle = val, seen |= 4;
            else if (key == "model_error_tag") tag = val;
            else if (key == "iewpf_mode") mode = val;
            else if (key == "drifters") n_d = val;
        }
        if (seen != 7) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: malformed rng_state", -1);
    }
    if (seed != cfg.seed)
        return dcg::ctx_error(ctx, DC_EINVAL,
                              "checkpoint: master seed " + std::to_string(seed) +
                                  " differs from the context's " + std::to_string(cfg.seed),
                              -1);
    Member s;
    for (int m = 0; m < M; ++m) {
        dc_status st = read_snapshot(ctx, particle_path(d, base + m), cfg.nx, cfg.ny, &s);
        if (st) return st;
        st = dc_upload_member(ctx, m, s.eta.data(), s.hu.data(), s.hv.data(), s.t);
        if (st) return st;
    }
    if (n_d > 0) {
        std::vector<double> pos(static_cast<size_t>(M) * n_d * 2);
        std::vector<int32_t> wind(pos.size());
        for (int m = 0; m < M; ++m) {
            std::ifstream is(drifters_path(d, base + m));
            if (!is) return dcg::ctx_error(ctx, DC_EIO, "checkpoint: cannot open drifters", m);
            std::string line;
            for (uint64_t q = 0; q < n_d; ++q) {
                if (!std::getline(is, line))
                    return dcg::ctx_error(ctx, DC_EIO, "checkpoint: truncated drifters file", m);
                unsigned long long id = 0;
                long long wx = 0, wy = 0;
                double x = 0.0, y = 0.0;
                if (std::sscanf(line.c_str(), "%llu,%lf,%lf,%lld,%lld", &id, &x, &y, &wx, &wy) != 5 ||
                    id != q)
                    return dcg::ctx_error(ctx, DC_EIO, "checkpoint: malformed drifters file", m);
                const size_t i = (static_cast<size_t>(m) * n_d + q) * 2;
                pos[i] = x;
                pos[i + 1] = y;
                wind[i] = static_cast<int32_t>(wx);
                wind[i + 1] = static_cast<int32_t>(wy);
            }
        }
        dc_status st = dc_drifters_restore(ctx, pos.data(), wind.data(), static_cast<int32_t>(n_d));
        if (st) return st;
    }
    dc_set_draw_counter(ctx, draw);
    dc_status st = dc_set_model_error_tag(ctx, tag);
    if (st) return st;
    if ((st = dc_iewpf_set_mode(ctx, static_cast<int32_t>(mode)))) return st;
    if (filter_cycle) *filter_cycle = cycle;
    return DC_OK;
}

} // extern "C"
