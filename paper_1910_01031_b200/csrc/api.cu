// api.cu -- the C ABI (include/driftcast_gpu.h): ensemble context, device memory,
// the device-side substep loop as a CUDA graph with a while-node, error surfacing.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "dc_internal.h"
#include "detmath.cuh"
#include "iewpf_host.h"

using namespace dcg;

// NCCL communicator + partition of a multi-GPU context (dc_comm_attach, comm_api.inc)
struct CommState {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    int64_t n_total = 0;
    std::vector<int64_t> base;  // [world + 1]: first global particle id of each rank
    double* gpos = nullptr;     // rank 0: every member's drifters, id order [n_total][n_d][2]
    int* gwind = nullptr;
    size_t gcap = 0;            // members x drifters the gather buffers hold
};

struct dc_ctx {
    dc_config cfg{};
    int M = 0;
    int64_t base = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool exact = true;
    SweParams sp{};
    ErrParams ep{};
    int nr = 0;
    size_t field_elems = 0;   // floats per field (M x mstride)
    float* blk[2] = {nullptr};  // the two state sets (psi^n, psi*), 3 fields each
    float* f[6] = {nullptr};  // eta, hu, hv, stage eta, stage hu, stage hv (views into blk)
    CUtensorMap maps[2];      // TMA maps of the two state sets (stage kernels)
    CUtensorMap qmap;         // state set 0, box of one 32x30 tile + halo (tile kernels)
    StepCtl ctl{};
    void* ctl_mem = nullptr;
    unsigned long long* substep_iters = nullptr; // device counters (graph path): [iters, member-substeps]
    unsigned long long* host_iters = nullptr;    // same counters for the host-loop path
    double* xi = nullptr;
    double* corr = nullptr;
    int* offs = nullptr;
    uint64_t me_draw = 0;
    uint64_t me_tag = 1;  // StreamTag of the model-error draws (1 model_error, 3 truth)
    // flux_rhs scratch (one member)
    float* rhs = nullptr;
    unsigned long long* gmax = nullptr;
    // graph of one model step
    cudaGraphExec_t step_exec = nullptr;       // step graph that scans the CFL stats first
    cudaGraphExec_t step_exec_fused = nullptr; // step graph relying on fused stats
    // CFL accumulator state: 0 = reset, 1 = hold the stats of the current state
    // (fused into the last state-changing kernel), 2 = stale
    int stats = 2;
    // the periodic ghost frame of the model state is current (every writer but the stage
    // kernels and q_half_apply leaves it stale; dc_step refreshes it only when needed)
    bool ghosts_ok = false;
    bool use_graph = true;
    int64_t launches = 0;
    int last_max_sub = 8;
    // CTA row units of the SWE stage grid (big strips first, short ones last)
    int2* units = nullptr;
    // IEWPF / observation / drifter state
    IewpfBuffers iw{};
    FeScratch fe{};  // forecast_error scratch
    ReadbackSlot rb[kReadbackSlots];  // pipelined per-cycle outputs
    CommState* comm = nullptr;        // dc_comm_attach (multi-GPU), else single context
    // error reporting
    std::string err;
    int em = -1, ej = -1, ek = -1, esub = -1;
};


// Every entry point that takes a context runs on that context's device (a process may
// drive several GPUs, one context each) and restores the caller's current device.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const dc_ctx* c) {
        int cur = 0;
        if (c && cudaGetDevice(&cur) == cudaSuccess && cur != c->device) {
            prev = cur;
            cudaSetDevice(c->device);
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

namespace {

// comm_api.inc (included at the end of this file)
void comm_free(dc_ctx* ctx);
dc_status iewpf_assimilate_comm(dc_ctx* ctx, const dc_obs* obs, int32_t n_obs, const double* S,
                                const double* usig, uint64_t cycle);
dc_status comm_gather_drifters(dc_ctx* ctx);

const char* kVersion = "driftcast-b200 0.1 (sm_100a)";

dc_status set_err(dc_ctx* c, dc_status st, const std::string& msg, int m = -1, int j = -1,
                  int k = -1, int sub = -1) {
    if (c) {
        c->err = msg;
        c->em = m;
        c->ej = j;
        c->ek = k;
        c->esub = sub;
    }
    return st;
}

#define CU(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return set_err(ctx, DC_ECUDA, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                              " at " #call);                               \
    } while (0)

dc_status validate(const dc_config* c, std::string* why) {
    if (c->nx < 8 || c->ny < 8) return *why = "ModelGrid: need nx,ny >= 8", DC_EINVAL;
    if (!(c->dx > 0.0) || !(c->dy > 0.0)) return *why = "ModelGrid: need dx,dy > 0", DC_EINVAL;
    if (!(c->g > 0.0)) return *why = "PhysParams: g must be > 0", DC_EINVAL;
    if (!(c->h_eq > 0.0)) return *why = "PhysParams: h_eq must be > 0", DC_EINVAL;
    if (c->f == 0.0) return *why = "PhysParams: f must be nonzero", DC_EINVAL;
    if (!(c->courant > 0.0 && c->courant < 1.0))
        return *why = "SchemeParams: courant in (0,1)", DC_EINVAL;
    if (!(c->limiter_theta >= 1.0 && c->limiter_theta <= 2.0))
        return *why = "SchemeParams: limiter_theta in [1,2]", DC_EINVAL;
    if (!(c->model_dt > 0.0)) return *why = "SchemeParams: model_dt > 0", DC_EINVAL;
    if (c->q0 < 0.0) return *why = "ErrorParams: q0 must be >= 0", DC_EINVAL;
    if (c->q0 > 0.0 && !(c->l0 > 0.0)) return *why = "ErrorParams: l0 must be > 0", DC_EINVAL;
    if (c->c_omega <= 0 || c->c_omega % 2 == 0)
        return *why = "CoarseGrid: coarsening factor must be odd and positive", DC_EINVAL;
    if (c->nx % c->c_omega != 0 || c->ny % c->c_omega != 0)
        return *why = "CoarseGrid: c_omega must divide nx and ny", DC_EINVAL;
    if (c->c_soar != 2) return *why = "ErrorParams: c_soar is fixed at 2", DC_EINVAL;
    return DC_OK;
}

double soar_kernel(double dist, double q0, double l0) { // stochastic.hpp:43-45
    return q0 * (1.0 + dist / l0) * std::exp(-dist / l0);
}

void derive_params(dc_ctx* c) {
    const dc_config& g = c->cfg;
    SweParams& P = c->sp;
    P.nx = g.nx;
    P.ny = g.ny;
    P.pitch = (g.nx + 4 + 31) / 32 * 32;  // + the 2-cell ghost frame on both sides
    P.mstride = static_cast<size_t>(g.ny + 4) * P.pitch;
    P.M = c->M;
    P.strips = (g.ny + 31) / 32;
    P.by = (g.ny + P.strips - 1) / P.strips;
    P.strips = (g.ny + P.by - 1) / P.by;
    P.H = static_cast<float>(g.h_eq);
    P.g = static_cast<float>(g.g);
    P.theta = static_cast<float>(g.limiter_theta);
    P.cf_x = static_cast<float>(g.f * g.dx / (2.0 * g.h_eq));
    P.cf_y = static_cast<float>(g.f * g.dy / (2.0 * g.h_eq));
    P.inv_g = 1.0f / P.g;
    P.idx = static_cast<float>(1.0 / g.dx);
    P.idy = static_cast<float>(1.0 / g.dy);
    P.fH = static_cast<float>(g.f / g.h_eq);
    P.half_theta = 0.5f * P.theta;
    P.fH_4 = 0.25f * P.fH;
    P.dx = g.dx;
    P.dy = g.dy;
    P.courant = g.courant;
    P.model_dt = g.model_dt;
    P.h_eq = g.h_eq;
    P.gd = g.g;
    P.neg_zero = -0.0f;
    ErrParams& E = c->ep;
    E.c = g.c_omega;
    E.nxc = g.nx / g.c_omega;
    E.nyc = g.ny / g.c_omega;
    E.dxc = g.c_omega * g.dx;
    E.dyc = g.c_omega * g.dy;
    E.inv_c = 1.0 / g.c_omega;
    E.cx = g.g * g.h_eq / (g.f * 2.0 * g.dx);
    E.cy = g.g * g.h_eq / (g.f * 2.0 * g.dy);
    E.cxc = g.g * g.h_eq / (g.f * 2.0 * E.dxc);
    E.cyc = g.g * g.h_eq / (g.f * 2.0 * E.dyc);
    for (int db = -2; db <= 2; ++db)
        for (int da = -2; da <= 2; ++da)
            E.w[(db + 2) * 5 + (da + 2)] =
                g.q0 == 0.0 ? 0.0 : soar_kernel(std::hypot(da * E.dxc, db * E.dyc), g.q0, g.l0);
    E.h_eq = g.h_eq;
    c->nr = E.nxc * E.nyc;
}

// Device errors -> the reference's exception message shapes.
dc_status surface_errors(dc_ctx* ctx) {
    std::vector<int> err(ctx->M), pos(ctx->M), sub(ctx->M);
    CU(cudaStreamSynchronize(ctx->stream));
    CU(cudaMemcpy(err.data(), ctx->ctl.err, ctx->M * sizeof(int), cudaMemcpyDeviceToHost));
    int m = -1;
    for (int i = 0; i < ctx->M; ++i)
        if (err[i]) {
            m = i;
            break;
        }
    if (m < 0) return DC_OK;
    CU(cudaMemcpy(pos.data(), ctx->ctl.err_pos, ctx->M * sizeof(int), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(sub.data(), ctx->ctl.err_sub, ctx->M * sizeof(int), cudaMemcpyDeviceToHost));
    const int nx = ctx->cfg.nx;
    const int p = pos[m];
    const int j = (p >= 0 && p != 0x7fffffff) ? p % nx : -1;
    const int k = (p >= 0 && p != 0x7fffffff) ? p / nx : -1;
    const std::string who = " (particle " + std::to_string(ctx->base + m) + ")";
    switch (err[m]) {
    case E_DRY_CELL:
        if (j >= 0)
            return set_err(ctx, DC_EDRY,
                           "flux_rhs: dry cell at (" + std::to_string(j) + "," +
                               std::to_string(k) + ")" + who,
                           m, j, k);
        return set_err(ctx, DC_EDRY, "flux_rhs: dry cell (non-finite eta)" + who, m);
    case E_DRY_FACE:
        return set_err(ctx, DC_EDRY, "flux_rhs: dry reconstructed face value" + who, m);
    case E_NONFINITE:
        return set_err(ctx, DC_ENONFINITE,
                       "model_step: non-finite value after substep " + std::to_string(sub[m]) +
                           who,
                       m, -1, -1, sub[m]);
    case E_RUNAWAY:
        return set_err(ctx, DC_ERUNAWAY, "model_step: substep count exploded" + who, m);
    case E_DRY_ADD:
        return set_err(ctx, DC_EDRY, "add_q_half: perturbation dried a cell" + who, m, j, k);
    case E_DRY_DRIFTER:
        return set_err(ctx, DC_EDRY, "advect_drifters: dry cell" + who, m);
    case E_ALPHA:
        return set_err(ctx, DC_ENONFINITE, "solve_alpha: Lambert-W failure" + who, m);
    case E_BETA:
        return set_err(ctx, DC_EINVAL, "sync_target_beta: zeta <= 0 or beta < 0" + who, m);
    default:
        return set_err(ctx, DC_ESTATE, "device error " + std::to_string(err[m]) + who, m);
    }
}

dc_status check_member(dc_ctx* ctx, int m) {
    if (m < 0 || m >= ctx->M)
        return set_err(ctx, DC_ESTATE, "member index " + std::to_string(m) + " out of range");
    return DC_OK;
}

// A member whose state is overwritten (upload, init, snapshot / checkpoint load, import)
// starts healthy: its device error flags are cleared. The reference throws per call and
// never poisons a particle, so a failed member must be recoverable by reloading it.
dc_status clear_member_errors(dc_ctx* ctx, int m0, int n) {
    cudaStream_t s = ctx->stream;
    CU(cudaMemsetAsync(ctx->ctl.err + m0, 0, n * sizeof(int), s));
    CU(cudaMemsetAsync(ctx->ctl.err_sub + m0, 0, n * sizeof(int), s));
    const std::vector<int> big(n, 0x7fffffff);  // pageable: staged before the call returns
    CU(cudaMemcpyAsync(ctx->ctl.err_pos + m0, big.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
    return DC_OK;
}

// The two stages of one substep: psi^n (set 0) -> psi* (set 1) -> psi^n+1 (set 0).
void launch_stage1(dc_ctx* ctx, cudaStream_t s) {
    const CUtensorMap maps[2] = {ctx->maps[0], ctx->maps[0]};
    launch_stage(s, ctx->sp, ctx->exact, 1, maps, ctx->f[0], ctx->f[1], ctx->f[2], ctx->f[3],
                 ctx->f[4], ctx->f[5], ctx->ctl);
}
// iters: the substep counters the fused end accumulates into (graph path / host loop)
void launch_stage2(dc_ctx* ctx, cudaStream_t s, unsigned long long cond, int end_mode,
                   unsigned long long* iters) {
    const CUtensorMap maps[2] = {ctx->maps[1], ctx->maps[0]};
    StepCtl ctl = ctx->ctl;
    ctl.iters = iters;
    launch_stage(s, ctx->sp, ctx->exact, 2, maps, ctx->f[3], ctx->f[4], ctx->f[5], ctx->f[0],
                 ctx->f[1], ctx->f[2], ctl, cond, end_mode);
}

// the ghost frame of the model state (every writer but the stage kernels leaves it stale)
void fix_ghosts(dc_ctx* ctx, cudaStream_t s) {
    launch_fix_ghosts(s, ctx->sp, ctx->f[0], ctx->field_elems);
}

// One model step as a graph: [reset + cfl_scan] -> step_begin -> while(any active){stage1,
// stage2, substep_end}. The while condition is set on the device by substep_end. The
// scan is skipped when the kernel that last changed the state already reduced the CFL
// statistics of its output (stage 2, q_half_apply).
dc_status build_step_graph(dc_ctx* ctx, bool with_scan, cudaGraphExec_t* exec) {
    cudaStream_t s = ctx->stream;
    CU(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    if (with_scan) {
        launch_reset_stats(s, ctx->sp, ctx->ctl);
        launch_cfl_scan(s, ctx->sp, ctx->f[0], ctx->f[1], ctx->f[2], ctx->ctl);
    }
    cudaStreamCaptureStatus st;
    cudaGraph_t cap = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CU(cudaStreamGetCaptureInfo(s, &st, nullptr, &cap, &deps, &ndeps));
    cudaGraphConditionalHandle handle;
    CU(cudaGraphConditionalHandleCreate(&handle, cap, 1, cudaGraphCondAssignDefault));
    const unsigned long long h = static_cast<unsigned long long>(handle);
    launch_step_begin(s, ctx->sp, ctx->ctl, h, 1);
    CU(cudaStreamGetCaptureInfo(s, &st, nullptr, &cap, &deps, &ndeps));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    CU(cudaGraphAddNode(&cnode, cap, deps, ndeps, &cp));
    CU(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t bs;
    CU(cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking));
    CU(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    launch_stage1(ctx, bs);
    launch_stage2(ctx, bs, h, 2, ctx->substep_iters);
    cudaGraph_t body_out = nullptr;
    CU(cudaStreamEndCapture(bs, &body_out));
    CU(cudaStreamDestroy(bs));
    cudaGraph_t g = nullptr;
    CU(cudaStreamEndCapture(s, &g));
    CU(cudaGraphInstantiate(exec, g, 0));
    CU(cudaGraphDestroy(g));
    return DC_OK;
}

// Host-driven fallback (DC_NO_GRAPH=1): guess the substep count from the previous step,
// then confirm on the host and continue one substep at a time.
dc_status step_host_loop(dc_ctx* ctx, bool with_scan) {
    cudaStream_t s = ctx->stream;
    if (with_scan) {
        launch_reset_stats(s, ctx->sp, ctx->ctl);
        launch_cfl_scan(s, ctx->sp, ctx->f[0], ctx->f[1], ctx->f[2], ctx->ctl);
        ctx->launches += 2;
    }
    launch_step_begin(s, ctx->sp, ctx->ctl);
    ctx->launches += 1;
    int done = 0;
    int guess = ctx->last_max_sub;
    while (true) {
        for (int i = 0; i < guess; ++i) {
            launch_stage1(ctx, s);
            launch_stage2(ctx, s, 0ull, 1, ctx->host_iters);
            ctx->launches += 2;
        }
        done += guess;
        int any = 0;
        CU(cudaMemcpyAsync(&any, ctx->ctl.any_active, sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (!any) break;
        guess = 1;
    }
    ctx->last_max_sub = std::max(1, done);
    return DC_OK;
}

// q_half_apply on ctx->corr with the CFL statistics of the result fused in (the
// accumulators are reset first unless they already are).
void apply_q_half_with_stats(dc_ctx* ctx, const int* offsets, double scale,
                             const char* prof_name = "q_half_apply") {
    if (ctx->stats != 0) {
        launch_reset_stats(ctx->stream, ctx->sp, ctx->ctl);
        ctx->launches += 1;
    }
    launch_q_half_apply(ctx->stream, &ctx->qmap, ctx->sp, ctx->ep, ctx->corr, offsets, scale, ctx->f[0],
                        ctx->f[1], ctx->f[2], ctx->ctl.err, ctx->ctl.err_pos, ctx->M,
                        ctx->ctl.mx, prof_name);
    ctx->stats = 1;
    ctx->ghosts_ok = true;  // q_half_apply rewrites every cell and its ghost copies
}

} // namespace

namespace dcg {
// error hook for the host-side modules layered on the C ABI (io.cpp)
dc_status ctx_error(dc_ctx* ctx, dc_status st, const std::string& msg, int m) {
    return set_err(ctx, st, msg, m);
}

} // namespace dcg

extern "C" {
static dc_status dc_create_device(dc_ctx* ctx, int32_t device, void* stream);


const char* dc_version(void) { return kVersion; }

dc_status dc_create(const dc_config* cfg, int32_t n_members, int64_t member_base, int32_t device,
                    void* stream, dc_ctx** out) {
    if (!cfg || !out || n_members <= 0) return DC_EINVAL;
    std::string why;
    dc_status v = validate(cfg, &why);
    if (v) {
        std::fprintf(stderr, "dc_create: %s\n", why.c_str());
        return v;
    }
    dc_ctx* ctx = new dc_ctx();
    ctx->cfg = *cfg;
    ctx->M = n_members;
    ctx->base = member_base;
    ctx->device = device;
    ctx->exact = cfg->exact_fp != 0;
    // DC_NO_GRAPH=1: the host-driven substep loop (profiling: ncu does not descend into
    // the conditional node of the step graph)
    const char* ng = std::getenv("DC_NO_GRAPH");
    ctx->use_graph = !(ng && ng[0] == '1');
    derive_params(ctx);
    *out = ctx;
    int prev_dev = -1;
    cudaGetDevice(&prev_dev);
    dc_status st = dc_create_device(ctx, device, stream);
    if (prev_dev >= 0 && prev_dev != device) cudaSetDevice(prev_dev);  // caller's device
    if (st) {
        std::fprintf(stderr, "dc_create: %s\n", ctx->err.c_str());
        dc_destroy(ctx);
        *out = nullptr;
    }
    return st;
}

// Strip height of the SWE stage grid: balance the y prologue of a strip (the two rows
// above it are loaded and reconstructed again: ~1.4 rows of work per strip, measured)
// against wave quantisation of (x tiles x members x strips) CTAs over SMs x resident
// CTAs -- softened when there are many waves, since each member's two short tail strips
// fill the last one.
// Measured at 1000x600: 1000 members 154.9 / 153.8 / 152.2 ms per model step at 47 / 64 /
// 120-row strips; 125 members 19.90 / 19.67 / 19.57 at 40 / 86 / 120; at 500x300 x 100
// members 28 rows stays best (86: +14 %, 120: +28 %: too few CTAs to fill the waves).
static void choose_strips(SweParams& P, int sms, int per_sm) {
    const int xt = (P.nx + kSweOut - 1) / kSweOut;
    const double slots = static_cast<double>(sms) * per_sm;
    double best = 1e30;
    for (int s = std::max(1, (P.ny + 255) / 256); s <= std::max(1, (P.ny + 7) / 8); ++s) {
        const int by = (P.ny + s - 1) / s;
        const int strips = (P.ny + by - 1) / by;
        const double n = static_cast<double>(xt) * P.M * strips;
        const double waves = n / slots;
        // few waves: a partial last wave idles SMs outright; many waves: the tail strips
        // absorb most of it
        const double quant = waves < 8.0 ? std::ceil(waves) / waves
                                         : 1.0 + 0.3 * (std::ceil(waves) - waves) / waves;
        const double cost = quant * (1.0 + 1.4 / by);
        if (cost < best - 1e-9) {
            best = cost;
            P.by = by;
            P.strips = strips;
        }
    }
}

// Row units {m, y0 | y1 << 16} of the stage grid: every member's rows as big strips (the
// choose_strips height) followed by n_tail short strips of tail_rows rows; all members' big
// units come first in launch order, the short ones last, so the final wave of each stage
// launch drains in a fraction of a big CTA's time.
static std::vector<int2> build_units(const SweParams& P, int tail_rows, int n_tail) {
    std::vector<int2> big, small;
    const int ys = std::max(0, P.ny - tail_rows * n_tail);
    const int nb = std::max(1, (ys + P.by - 1) / std::max(1, P.by));
    for (int m = 0; m < P.M; ++m) {
        for (int b = 0; b < nb; ++b) {
            const int y0 = static_cast<int>(static_cast<long long>(ys) * b / nb);
            const int y1 = static_cast<int>(static_cast<long long>(ys) * (b + 1) / nb);
            if (y1 > y0) big.push_back(make_int2(m, y0 | (y1 << 16)));
        }
        for (int t = 0; t < n_tail; ++t) {
            const int y0 = ys + t * tail_rows, y1 = std::min(P.ny, y0 + tail_rows);
            if (y1 > y0) small.push_back(make_int2(m, y0 | (y1 << 16)));
        }
    }
    big.insert(big.end(), small.begin(), small.end());
    return big;
}

static dc_status dc_create_device(dc_ctx* ctx, int32_t device, void* stream) {
    CU(cudaSetDevice(device));
    double stage_waves = 0.0;  // waves of big strips in one stage launch
    {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int per_sm = swe_stage_occupancy();
        choose_strips(ctx->sp, sms, per_sm);
        stage_waves = static_cast<double>((ctx->sp.nx + kSweOut - 1) / kSweOut) * ctx->M * ctx->sp.strips /
                      (static_cast<double>(sms) * per_sm);
    }
    // per-member kernels put the member index in gridDim.y / z (<= 65535)
    if (ctx->M > 65535)
        return set_err(ctx, DC_EINVAL,
                       "too many members for one context (> 65535): split them over several "
                       "contexts / GPUs");
    {
        // short strips of ~2/5 of a big strip per member, launched after every big one:
        // two when a launch has few waves (500x300 x 100: -2.6 % per model step against
        // uniform strips; one: +0.4 %), one when it has many (1000x600 x 1000: -0.4 %,
        // x 125: -0.85 % against two; none: +0.5 %) -- each tail adds a strip prologue
        const int tail_rows = std::max(4, (2 * ctx->sp.by) / 5);
        const int n_tail = ctx->sp.ny >= 4 * ctx->sp.by ? (stage_waves >= 6.0 ? 1 : 2) : 0;
        if (tail_rows > 0 && n_tail > 0 && tail_rows * n_tail < ctx->sp.ny && ctx->sp.ny < 32768) {
            const std::vector<int2> u = build_units(ctx->sp, tail_rows, n_tail);
            CU(DMALLOC(&ctx->units, u.size() * sizeof(int2)));
            CU(cudaMemcpy(ctx->units, u.data(), u.size() * sizeof(int2), cudaMemcpyHostToDevice));
            ctx->sp.units = ctx->units;
            ctx->sp.n_units = static_cast<int>(u.size());
        }
    }
    if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
        CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    ctx->field_elems = static_cast<size_t>(ctx->M) * ctx->sp.mstride;
    // each state set is one allocation of 3 fields field_elems apart, so one 3-D TMA box
    // brings rows of all three fields; field pointers address cell (0, 0) inside the
    // 2-cell ghost frame (SweParams::mstride)
    const size_t origin = 2 * static_cast<size_t>(ctx->sp.pitch) + 2;
    for (int s = 0; s < 2; ++s) {
        const size_t bytes = 3 * ctx->field_elems * sizeof(float);
        CU(DMALLOC(&ctx->blk[s], bytes));
        CU(cudaMemsetAsync(ctx->blk[s], 0, bytes, ctx->stream));
        for (int i = 0; i < 3; ++i) ctx->f[3 * s + i] = ctx->blk[s] + i * ctx->field_elems + origin;
        if (!make_state_map(&ctx->maps[s], ctx->blk[s], ctx->sp, ctx->field_elems))
            return set_err(ctx, DC_ECUDA, "cuTensorMapEncodeTiled failed for the state maps");
    }
    if (!make_state_map(&ctx->qmap, ctx->blk[0], ctx->sp, ctx->field_elems, 36, 30))
        return set_err(ctx, DC_ECUDA, "cuTensorMapEncodeTiled failed for the tile map");
    const int M = ctx->M;
    // 17 arrays, each rounded up to 16 bytes by take()
    size_t bytes = 17 * ((static_cast<size_t>(M) * 4 * sizeof(double) + 15) / 16 * 16) + 64;
    CU(DMALLOC(&ctx->ctl_mem, bytes));
    CU(cudaMemsetAsync(ctx->ctl_mem, 0, bytes, ctx->stream));
    char* p = static_cast<char*>(ctx->ctl_mem);
    auto take = [&](size_t n) {
        char* r = p;
        p += (n + 15) / 16 * 16;
        return r;
    };
    ctx->ctl.t = reinterpret_cast<double*>(take(M * sizeof(double)));
    ctx->ctl.t_end = reinterpret_cast<double*>(take(M * sizeof(double)));
    ctx->ctl.remaining = reinterpret_cast<double*>(take(M * sizeof(double)));
    ctx->ctl.dt = reinterpret_cast<double*>(take(M * sizeof(double)));
    ctx->ctl.sub = reinterpret_cast<int*>(take(M * sizeof(int)));
    ctx->ctl.active = reinterpret_cast<int*>(take(M * sizeof(int)));
    ctx->ctl.err = reinterpret_cast<int*>(take(M * sizeof(int)));
    ctx->ctl.err_pos = reinterpret_cast<int*>(take(M * sizeof(int)));
    ctx->ctl.err_sub = reinterpret_cast<int*>(take(M * sizeof(int)));
    ctx->ctl.mx = reinterpret_cast<unsigned*>(take(4 * M * sizeof(unsigned)));
    ctx->ctl.any_active = reinterpret_cast<int*>(take(sizeof(int)));
    ctx->ctl.n_active = reinterpret_cast<int*>(take(sizeof(int)));
    ctx->ctl.mdone = reinterpret_cast<unsigned*>(take(M * sizeof(unsigned)));
    ctx->ctl.step_max = reinterpret_cast<unsigned*>(take(sizeof(unsigned)));
    CU(DMALLOC(&ctx->substep_iters, 2 * sizeof(unsigned long long)));
    CU(DMALLOC(&ctx->host_iters, 2 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(ctx->host_iters, 0, 2 * sizeof(unsigned long long), ctx->stream));
    CU(cudaMemsetAsync(ctx->substep_iters, 0, 2 * sizeof(unsigned long long), ctx->stream));
    ctx->ctl.iters = ctx->substep_iters;
    // accumulators: max fields 0, min field all-ones (ordered +inf side), err_pos INT_MAX
    std::vector<unsigned> mx(4 * M);
    for (int m = 0; m < M; ++m) {
        mx[4 * m] = 0u;
        mx[4 * m + 1] = 0u;
        mx[4 * m + 2] = 0xffffffffu;
        mx[4 * m + 3] = 0u;
    }
    CU(cudaMemcpyAsync(ctx->ctl.mx, mx.data(), mx.size() * sizeof(unsigned),
                       cudaMemcpyHostToDevice, ctx->stream));
    std::vector<int> big(M, 0x7fffffff);
    CU(cudaMemcpyAsync(ctx->ctl.err_pos, big.data(), M * sizeof(int), cudaMemcpyHostToDevice,
                       ctx->stream));
    CU(DMALLOC(&ctx->xi, static_cast<size_t>(M) * ctx->nr * sizeof(double)));
    CU(DMALLOC(&ctx->corr, static_cast<size_t>(M) * ctx->nr * sizeof(double)));
    CU(DMALLOC(&ctx->offs, 2 * M * sizeof(int)));
    CU(cudaMemsetAsync(ctx->offs, 0, 2 * M * sizeof(int), ctx->stream));
    CU(DMALLOC(&ctx->gmax, 2 * M * sizeof(unsigned long long)));
    CU(cudaStreamSynchronize(ctx->stream));
    return DC_OK;
}

dc_status dc_destroy(dc_ctx* ctx) {
    DeviceGuard dg_(ctx);
    if (!ctx) return DC_OK;
    cudaStreamSynchronize(ctx->stream);
    if (ctx->step_exec) cudaGraphExecDestroy(ctx->step_exec);
    if (ctx->step_exec_fused) cudaGraphExecDestroy(ctx->step_exec_fused);
    for (auto* q : ctx->blk) dcg::dfree(q);
    dcg::dfree(ctx->ctl_mem);
    if (ctx->units) dcg::dfree(ctx->units);
    dcg::dfree(ctx->substep_iters);
    dcg::dfree(ctx->host_iters);
    dcg::dfree(ctx->xi);
    dcg::dfree(ctx->corr);
    dcg::dfree(ctx->offs);
    dcg::dfree(ctx->gmax);
    dcg::dfree(ctx->rhs);
    iewpf_free(ctx->iw);
    fe_free(ctx->fe);
    readback_free(ctx->rb);
    comm_free(ctx);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return DC_OK;
}

dc_status dc_sync(dc_ctx* ctx) { return surface_errors(ctx); }

const char* dc_last_error(dc_ctx* ctx, int32_t* member, int32_t* j, int32_t* k,
                          int32_t* substep) {
    DeviceGuard dg_(ctx);
    if (!ctx) return "null context";
    if (member) *member = ctx->em;
    if (j) *j = ctx->ej;
    if (k) *k = ctx->ek;
    if (substep) *substep = ctx->esub;
    return ctx->err.c_str();
}

dc_status dc_upload_member(dc_ctx* ctx, int32_t m, const float* eta, const float* hu,
                           const float* hv, double t) {
    DeviceGuard dg_(ctx);
    ctx->ghosts_ok = false;
    dc_status st = check_member(ctx, m);
    if (st) return st;
    const size_t off = static_cast<size_t>(m) * ctx->sp.mstride;
    const float* src[3] = {eta, hu, hv};
    for (int i = 0; i < 3; ++i)
        CU(cudaMemcpy2DAsync(ctx->f[i] + off, ctx->sp.pitch * sizeof(float), src[i],
                             ctx->sp.nx * sizeof(float), ctx->sp.nx * sizeof(float), ctx->sp.ny,
                             cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(ctx->ctl.t + m, &t, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if ((st = clear_member_errors(ctx, m, 1))) return st;
    CU(cudaStreamSynchronize(ctx->stream)); // t is a stack value
    ctx->stats = 2;
    return DC_OK;
}

dc_status dc_upload_all(dc_ctx* ctx, const float* eta, const float* hu, const float* hv,
                        const double* t) {
    DeviceGuard dg_(ctx);
    ctx->ghosts_ok = false;
    const float* src[3] = {eta, hu, hv};
    const size_t cells = static_cast<size_t>(ctx->sp.nx) * ctx->sp.ny;
    for (int m = 0; m < ctx->M; ++m)
        for (int i = 0; i < 3; ++i)
            CU(cudaMemcpy2DAsync(ctx->f[i] + m * ctx->sp.mstride, ctx->sp.pitch * sizeof(float),
                                 src[i] + m * cells, ctx->sp.nx * sizeof(float),
                                 ctx->sp.nx * sizeof(float), ctx->sp.ny, cudaMemcpyHostToDevice,
                                 ctx->stream));
    if (t)
        CU(cudaMemcpyAsync(ctx->ctl.t, t, ctx->M * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
    ctx->stats = 2;
    return clear_member_errors(ctx, 0, ctx->M);
}

dc_status dc_download_member(dc_ctx* ctx, int32_t m, float* eta, float* hu, float* hv,
                             double* t) {
    DeviceGuard dg_(ctx);
    dc_status st = check_member(ctx, m);
    if (st) return st;
    st = surface_errors(ctx);
    const size_t off = static_cast<size_t>(m) * ctx->sp.mstride;
    float* dst[3] = {eta, hu, hv};
    for (int i = 0; i < 3; ++i)
        if (dst[i])
            CU(cudaMemcpy2DAsync(dst[i], ctx->sp.nx * sizeof(float), ctx->f[i] + off,
                                 ctx->sp.pitch * sizeof(float), ctx->sp.nx * sizeof(float),
                                 ctx->sp.ny, cudaMemcpyDeviceToHost, ctx->stream));
    if (t)
        CU(cudaMemcpyAsync(t, ctx->ctl.t + m, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return st;
}

dc_status dc_download_all(dc_ctx* ctx, float* eta, float* hu, float* hv, double* t) {
    DeviceGuard dg_(ctx);
    dc_status st = surface_errors(ctx);
    float* dst[3] = {eta, hu, hv};
    const size_t cells = static_cast<size_t>(ctx->sp.nx) * ctx->sp.ny;
    for (int m = 0; m < ctx->M; ++m)
        for (int i = 0; i < 3; ++i)
            if (dst[i])
                CU(cudaMemcpy2DAsync(dst[i] + m * cells, ctx->sp.nx * sizeof(float),
                                     ctx->f[i] + m * ctx->sp.mstride, ctx->sp.pitch * sizeof(float),
                                     ctx->sp.nx * sizeof(float), ctx->sp.ny,
                                     cudaMemcpyDeviceToHost, ctx->stream));
    if (t)
        CU(cudaMemcpyAsync(t, ctx->ctl.t, ctx->M * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return st;
}

// init_double_jet (swe.hpp:459-500): fp64 profile on the host (same libm as the
// reference build), broadcast to every member, t = 0.
dc_status dc_init_double_jet(dc_ctx* ctx) {
    DeviceGuard dg_(ctx);
    ctx->ghosts_ok = false;
    const dc_config& g = ctx->cfg;
    const int nx = g.nx, ny = g.ny;
    const double ly = ny * g.dy;
    const double width = (1.0 / 6.0) * ly, y1 = 0.25 * ly, y2 = 0.75 * ly;
    const double peak = 0.5 * g.h_eq;
    auto bump = [&](double y, double yc) {
        double s = (y - (yc - 0.5 * width)) / width;
        if (s <= 0.0 || s >= 1.0) return 0.0;
        return std::exp(4.0) * std::exp(1.0 / ((s - 1.0) * s));
    };
    std::vector<double> hu_p(ny), eta_p(ny, 0.0);
    for (int k = 0; k < ny; ++k) hu_p[k] = peak * (bump((k + 0.5) * g.dy, y1) - bump((k + 0.5) * g.dy, y2));
    const double cf = g.f / (g.g * g.h_eq);
    for (int k = 1; k < ny; ++k) eta_p[k] = eta_p[k - 1] - 0.5 * g.dy * cf * (hu_p[k - 1] + hu_p[k]);
    double mean = 0.0;
    for (double e : eta_p) mean += e;
    mean /= ny;
    for (double& e : eta_p) e -= mean;
    const int pitch = ctx->sp.pitch;
    std::vector<float> e(static_cast<size_t>(ny) * pitch, 0.0f), u(e.size(), 0.0f), z(e.size(), 0.0f);
    for (int k = 0; k < ny; ++k)
        for (int j = 0; j < nx; ++j) {
            e[static_cast<size_t>(k) * pitch + j] = static_cast<float>(eta_p[k]);
            u[static_cast<size_t>(k) * pitch + j] = static_cast<float>(hu_p[k]);
        }
    const size_t per = static_cast<size_t>(ny) * pitch;
    const size_t ms = ctx->sp.mstride;
    for (int m = 0; m < ctx->M; ++m) {
        CU(cudaMemcpyAsync(ctx->f[0] + m * ms, e.data(), per * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(ctx->f[1] + m * ms, u.data(), per * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(ctx->f[2] + m * ms, z.data(), per * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    }
    CU(cudaMemsetAsync(ctx->ctl.t, 0, ctx->M * sizeof(double), ctx->stream));
    dc_status st = clear_member_errors(ctx, 0, ctx->M);
    if (st) return st;
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->stats = 2;
    return DC_OK;
}

dc_status dc_step(dc_ctx* ctx, int32_t n_steps) {
    DeviceGuard dg_(ctx);
    if (n_steps < 0) return set_err(ctx, DC_EINVAL, "dc_step: n_steps < 0");
    if (ctx->use_graph && !ctx->step_exec) {
        dc_status st = build_step_graph(ctx, true, &ctx->step_exec);
        if (!st) st = build_step_graph(ctx, false, &ctx->step_exec_fused);
        if (st) {
            cudaGetLastError();
            std::fprintf(stderr, "dc_step: graph path unavailable (%s); using host loop\n",
                         ctx->err.c_str());
            ctx->use_graph = false;
            cudaStreamCaptureStatus cs;
            if (cudaStreamIsCapturing(ctx->stream, &cs) == cudaSuccess &&
                cs != cudaStreamCaptureStatusNone) {
                cudaGraph_t junk;
                cudaStreamEndCapture(ctx->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
            }
        }
    }
    for (int i = 0; i < n_steps; ++i) {
        const bool scan = ctx->stats != 1;
        if (!ctx->ghosts_ok) {
            fix_ghosts(ctx, ctx->stream);
            ctx->launches += 1;
        }
        // inside a profile window the stage kernels are launched (and timed) one by one
        if (ctx->use_graph && !kprof_active()) {
            CU(cudaGraphLaunch(scan ? ctx->step_exec : ctx->step_exec_fused, ctx->stream));
            ctx->launches += scan ? 3 : 1;  // [reset, cfl_scan,] step_begin
        } else {
            dc_status st = step_host_loop(ctx, scan);
            if (st) return st;
        }
        ctx->stats = 0;  // every member's final substep_end resets the accumulators
        ctx->ghosts_ok = true;  // stage 2 writes its own ghost copies
    }
    CU(cudaGetLastError());
    return DC_OK;
}

dc_status dc_substeps(dc_ctx* ctx, int32_t* out) {
    DeviceGuard dg_(ctx);
    CU(cudaMemcpyAsync(out, ctx->ctl.sub, ctx->M * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return DC_OK;
}

dc_status dc_flux_rhs(dc_ctx* ctx, int32_t m, float* d_eta, float* d_hu, float* d_hv) {
    DeviceGuard dg_(ctx);
    dc_status st = check_member(ctx, m);
    if (st) return st;
    const size_t per = ctx->sp.mstride;
    if (!ctx->rhs) CU(DMALLOC(&ctx->rhs, 3 * per * sizeof(float)));  // per = mstride
    // dry-cell check of load() (swe.hpp:319): flux_rhs throws before computing
    std::vector<float> e(static_cast<size_t>(ctx->sp.nx) * ctx->sp.ny);
    CU(cudaMemcpy2DAsync(e.data(), ctx->sp.nx * sizeof(float), ctx->f[0] + m * ctx->sp.mstride,
                         ctx->sp.pitch * sizeof(float), ctx->sp.nx * sizeof(float), ctx->sp.ny,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    const float H = ctx->sp.H;
    bool dry = false;
    for (float v : e) dry |= !(H + v > 0.0f) && !std::isnan(v);
    if (dry) {
        for (int k = 0; k < ctx->sp.ny; ++k)
            for (int j = 0; j < ctx->sp.nx; ++j)
                if (!(ctx->cfg.h_eq + e[static_cast<size_t>(k) * ctx->sp.nx + j] > 0.0))
                    return set_err(ctx, DC_EDRY,
                                   "flux_rhs: dry cell at (" + std::to_string(j) + "," +
                                       std::to_string(k) + ")",
                                   m, j, k);
        return set_err(ctx, DC_EDRY, "flux_rhs: dry cell (non-finite eta)", m);
    }
    fix_ghosts(ctx, ctx->stream);
    launch_flux_rhs(ctx->stream, ctx->sp, ctx->exact, m, &ctx->maps[0], ctx->f[0], ctx->f[1],
                    ctx->f[2], ctx->rhs + 2 * ctx->sp.pitch + 2, ctx->rhs + per + 2 * ctx->sp.pitch + 2,
                    ctx->rhs + 2 * per + 2 * ctx->sp.pitch + 2, ctx->ctl);
    ctx->launches += 1;
    ctx->launches += 1;
    float* dst[3] = {d_eta, d_hu, d_hv};
    for (int i = 0; i < 3; ++i)
        CU(cudaMemcpy2DAsync(dst[i], ctx->sp.nx * sizeof(float), ctx->rhs + i * per + 2 * ctx->sp.pitch + 2,
                             ctx->sp.pitch * sizeof(float), ctx->sp.nx * sizeof(float),
                             ctx->sp.ny, cudaMemcpyDeviceToHost, ctx->stream));
    return surface_errors(ctx);
}

dc_status dc_cfl_dt(dc_ctx* ctx, double* dt_out) {
    DeviceGuard dg_(ctx);
    const int M = ctx->M;
    CU(cudaMemsetAsync(ctx->gmax, 0, 2 * M * sizeof(unsigned long long), ctx->stream));
    std::vector<int> big(M, 0x7fffffff);
    CU(cudaMemcpyAsync(ctx->ctl.err_pos, big.data(), M * sizeof(int), cudaMemcpyHostToDevice,
                       ctx->stream));
    launch_cfl_public(ctx->stream, ctx->sp, ctx->f[0], ctx->f[1], ctx->f[2], ctx->gmax,
                      ctx->ctl.err_pos);
    ctx->launches += 1;
    std::vector<unsigned long long> g(2 * M);
    std::vector<int> pos(M);
    CU(cudaMemcpyAsync(g.data(), ctx->gmax, g.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(pos.data(), ctx->ctl.err_pos, M * sizeof(int), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int m = 0; m < M; ++m) {
        if (pos[m] != 0x7fffffff) {
            const int j = pos[m] % ctx->sp.nx, k = pos[m] / ctx->sp.nx;
            CU(cudaMemcpyAsync(ctx->ctl.err_pos, big.data(), M * sizeof(int),
                               cudaMemcpyHostToDevice, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            return set_err(ctx, DC_EDRY,
                           "cfl_dt: dry cell at (" + std::to_string(j) + "," + std::to_string(k) + ")",
                           m, j, k);
        }
        double gx, gy;
        std::memcpy(&gx, &g[2 * m], 8);
        std::memcpy(&gy, &g[2 * m + 1], 8);
        dt_out[m] = ctx->cfg.courant * 0.25 * std::min(ctx->cfg.dx / gx, ctx->cfg.dy / gy);
    }
    return DC_OK;
}

dc_status dc_perturb(dc_ctx* ctx, int32_t mode, const int32_t* offsets, const double* xi) {
    DeviceGuard dg_(ctx);
    if (ctx->cfg.q0 == 0.0) return DC_OK; // stochastic.hpp:167: consumes no randomness
    const int M = ctx->M;
    if (mode == DC_NOISE_PHILOX) {
        if (ctx->ep.nxc <= 1280) {  // fused noise + SOAR: xi never goes to HBM
            launch_philox_soar(ctx->stream, ctx->ep, M, ctx->cfg.seed, ctx->me_tag, ctx->base, 0,
                               ctx->me_draw, ctx->corr, ctx->offs, ctx->ctl.err);
            ctx->me_draw += 1;
            apply_q_half_with_stats(ctx, ctx->offs, 1.0);
            ctx->launches += 2;
            CU(cudaGetLastError());
            return DC_OK;
        }
        launch_philox_noise(ctx->stream, ctx->ep, M, ctx->cfg.seed, ctx->me_tag, ctx->base, 0,
                            ctx->me_draw, ctx->xi, ctx->offs, ctx->ctl.err);
        ctx->me_draw += 1;
    } else if (mode == DC_NOISE_INJECTED) {
        if (!offsets || !xi) return set_err(ctx, DC_EINVAL, "dc_perturb: injected noise missing");
        for (int m = 0; m < 2 * M; ++m)
            if (offsets[m] < 0 || offsets[m] >= ctx->cfg.c_omega)
                return set_err(ctx, DC_EINVAL, "CoarseGrid: offsets must lie in [0, c_omega)");
        CU(cudaMemcpyAsync(ctx->offs, offsets, 2 * M * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(ctx->xi, xi, static_cast<size_t>(M) * ctx->nr * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream)); // host buffers may be reused on return
    } else {
        return set_err(ctx, DC_EINVAL, "dc_perturb: unknown noise mode");
    }
    launch_coarse_soar(ctx->stream, ctx->ep, M, ctx->xi, ctx->corr, ctx->ctl.err);
    apply_q_half_with_stats(ctx, ctx->offs, 1.0);
    ctx->launches += (mode == DC_NOISE_PHILOX) ? 3 : 2;
    CU(cudaGetLastError());
    return DC_OK;
}

dc_status dc_add_q_half(dc_ctx* ctx, const int32_t* offsets, const double* coarse, double scale) {
    DeviceGuard dg_(ctx);
    const int M = ctx->M;
    for (int m = 0; m < 2 * M; ++m)
        if (offsets[m] < 0 || offsets[m] >= ctx->cfg.c_omega)
            return set_err(ctx, DC_EINVAL, "CoarseGrid: offsets must lie in [0, c_omega)");
    CU(cudaMemcpyAsync(ctx->offs, offsets, 2 * M * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyAsync(ctx->xi, coarse, static_cast<size_t>(M) * ctx->nr * sizeof(double),
                       cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    launch_coarse_soar(ctx->stream, ctx->ep, M, ctx->xi, ctx->corr, ctx->ctl.err);
    apply_q_half_with_stats(ctx, ctx->offs, scale);
    ctx->launches += 2;
    CU(cudaGetLastError());
    return DC_OK;
}

dc_status dc_get_config(dc_ctx* ctx, dc_config* cfg, int32_t* n_members, int64_t* member_base) {
    DeviceGuard dg_(ctx);
    if (!ctx) return DC_ESTATE;
    if (cfg) *cfg = ctx->cfg;
    if (n_members) *n_members = ctx->M;
    if (member_base) *member_base = ctx->base;
    return DC_OK;
}

dc_status dc_get_draw_counter(dc_ctx* ctx, uint64_t* d) {
    DeviceGuard dg_(ctx);
    *d = ctx->me_draw;
    return DC_OK;
}

dc_status dc_set_model_error_tag(dc_ctx* ctx, uint64_t tag) {
    DeviceGuard dg_(ctx);
    if (tag != 1 && tag != 3)
        return set_err(ctx, DC_EINVAL, "model-error stream tag must be model_error (1) or "
                                       "truth_model_error (3)");
    ctx->me_tag = tag;
    return DC_OK;
}

dc_status dc_get_model_error_tag(dc_ctx* ctx, uint64_t* tag) {
    if (!ctx || !tag) return DC_ESTATE;
    *tag = ctx->me_tag;
    return DC_OK;
}

dc_status dc_iewpf_get_mode(dc_ctx* ctx, int32_t* mode) {
    if (!ctx || !mode) return DC_ESTATE;
    *mode = ctx->iw.one_stage ? DC_IEWPF_ONE_STAGE : DC_IEWPF_TWO_STAGE;
    return DC_OK;
}

dc_status dc_set_draw_counter(dc_ctx* ctx, uint64_t d) {
    DeviceGuard dg_(ctx);
    ctx->me_draw = d;
    return DC_OK;
}

int64_t dc_kernel_launches(dc_ctx* ctx) {
    DeviceGuard dg_(ctx);
    // graph path: 2 kernels per step + 2 per substep iteration, iterations counted on the
    // device
    unsigned long long iters = 0;
    if (ctx->use_graph && ctx->substep_iters) {
        cudaMemcpyAsync(&iters, ctx->substep_iters, sizeof(iters), cudaMemcpyDeviceToHost,
                        ctx->stream);
        cudaStreamSynchronize(ctx->stream);
    }
    return ctx->launches + 2 * static_cast<int64_t>(iters);
}

void* dc_stream(dc_ctx* ctx) { return ctx->stream; }

dc_status dc_counters(dc_ctx* ctx, uint64_t* out) {
    DeviceGuard dg_(ctx);
    unsigned long long g[2] = {0, 0}, h[2] = {0, 0};
    CU(cudaMemcpyAsync(g, ctx->substep_iters, sizeof(g), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(h, ctx->host_iters, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    out[0] = static_cast<uint64_t>(dc_kernel_launches(ctx));
    out[1] = g[1] + h[1];  // member-substeps since creation
    out[2] = g[0] + h[0];  // substep-loop iterations since creation
    return DC_OK;
}

dc_status dc_time_stages(dc_ctx* ctx, int32_t n_substeps, double* ms_out) {
    DeviceGuard dg_(ctx);
    // One model step's worth of substeps launched individually with CUDA events around
    // each stage kernel on the context stream (advances the state like dc_step). All
    // launches and events are queued back to back and read after one synchronisation,
    // so each interval is the kernel's duration plus the queued-launch gap.
    if (n_substeps <= 0 || n_substeps > 64) return set_err(ctx, DC_EINVAL, "n_substeps in 1..64");
    cudaStream_t s = ctx->stream;
    std::vector<cudaEvent_t> ev(3 * static_cast<size_t>(n_substeps));
    for (auto& e : ev) CU(cudaEventCreate(&e));
    fix_ghosts(ctx, s);
    launch_reset_stats(s, ctx->sp, ctx->ctl);
    launch_cfl_scan(s, ctx->sp, ctx->f[0], ctx->f[1], ctx->f[2], ctx->ctl);
    ctx->stats = 2;
    launch_step_begin(s, ctx->sp, ctx->ctl);
    for (int i = 0; i < n_substeps; ++i) {
        CU(cudaEventRecord(ev[3 * i], s));
        launch_stage1(ctx, s);
        CU(cudaEventRecord(ev[3 * i + 1], s));
        launch_stage2(ctx, s, 0ull, 1, ctx->host_iters);
        CU(cudaEventRecord(ev[3 * i + 2], s));
    }
    CU(cudaStreamSynchronize(s));
    double t1 = 0.0, t2 = 0.0;
    for (int i = 0; i < n_substeps; ++i) {
        float a = 0.f, b = 0.f;
        CU(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]));
        CU(cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]));
        t1 += a;
        t2 += b;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    ctx->launches += 4 + 2 * n_substeps;
    ms_out[0] = t1 / n_substeps;
    ms_out[1] = t2 / n_substeps;
    return surface_errors(ctx);
}

dc_status dc_profile_begin(dc_ctx* ctx) {
    if (!ctx) return DC_ESTATE;
    kprof_begin();
    return DC_OK;
}

dc_status dc_profile_end(dc_ctx* ctx, dc_kernel_time* out, int32_t cap, int32_t* n_out) {
    DeviceGuard dg_(ctx);
    if (!ctx) return DC_ESTATE;
    const int n = kprof_end(out, cap);
    if (n_out) *n_out = n;
    return surface_errors(ctx);
}

dc_status dc_check_guards(char* msg, int32_t cap, int32_t* n_bad) {
    std::string m;
    const int bad = check_guards(&m);
    if (n_bad) *n_bad = bad;
    if (msg && cap > 0) {
        std::strncpy(msg, m.c_str(), cap - 1);
        msg[cap - 1] = 0;
    }
    return bad ? DC_ECUDA : DC_OK;
}

dc_status dc_selftest_math(int32_t device, uint64_t* counts) {
    if (cudaSetDevice(device) != cudaSuccess) return DC_ECUDA;
    unsigned long long* d = nullptr;
    if (DMALLOC(&d, 4 * sizeof(unsigned long long)) != cudaSuccess) return DC_ECUDA;
    cudaMemset(d, 0, 4 * sizeof(unsigned long long));
    launch_selftest_math(nullptr, d);
    cudaError_t e = cudaMemcpy(counts, d, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    dcg::dfree(d);
    return e == cudaSuccess ? DC_OK : DC_ECUDA;
}

} // extern "C"

// IEWPF / observation entry points live in iewpf_api.cu; they need the context layout.
#include "iewpf_api.inc"
#include "experiment_api.inc"
#include "comm_api.inc"
