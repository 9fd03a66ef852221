/*
 * driftcast_gpu.h -- C ABI of the B200-native IEWPF hot path (libdriftcast_gpu.so).
 *
 * Drop-in boundary for the reference's C++ operator surface (namespace driftcast,
 * proj/include/driftcast/{grid,field,rng,state,swe,stochastic}.hpp). Every entry point is batched over the
 * ensemble held by one context (one context per process / GPU); all calls are
 * stream-ordered and asynchronous unless stated. Plain pointers and sizes only.
 *
 * Host arrays use the reference layout: Field2D row-major, j fastest, element (j,k) at
 * k*nx+j (field.hpp:10-11,48-50); member-major for ensemble arrays. Device layout is
 * private (members batched along y, rows padded to 128 B).
 *
 * Errors: calls return a dc_status; the reference's exceptions map to codes
 * (std::invalid_argument -> DC_EINVAL, DryCellError -> DC_EDRY, "non-finite value after
 * substep" -> DC_ENONFINITE, "substep count exploded" -> DC_ERUNAWAY). Device-side
 * failures surface at the next synchronising call (dc_sync, downloads, diagnostics)
 * with the reference's message shapes via dc_last_error. include/driftcast_gpu.hpp maps
 * codes back to the reference exception types.
 */
#ifndef DRIFTCAST_GPU_H
#define DRIFTCAST_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dc_status {
    DC_OK = 0,
    DC_EINVAL = 1,     /* std::invalid_argument */
    DC_EDRY = 2,       /* DryCellError (swe.hpp:32-34) */
    DC_ENONFINITE = 3, /* std::runtime_error "model_step: non-finite value after substep k" */
    DC_ERUNAWAY = 4,   /* std::runtime_error "model_step: substep count exploded" */
    DC_EALIGN = 5,     /* apply_q_half_T: observation not co-located */
    DC_ECUDA = 6,      /* CUDA runtime failure */
    DC_ESTATE = 7,     /* API misuse (bad member index, wrong call order) */
    DC_EIO = 8,        /* std::runtime_error from snapshot / file I/O (state.hpp:71-116) */
    DC_ECOLLAPSE = 9,  /* standard PF weights: every weight underflows */
    DC_ENCCL = 10      /* NCCL failure (multi-GPU communicator, dc_comm_*) */
} dc_status;

/* Parameter block: ModelGrid + PhysParams + SchemeParams + ErrorParams + seed. */
typedef struct dc_config {
    int32_t nx, ny;                 /* ModelGrid (grid.hpp:11-29) */
    double dx, dy;
    double g, f, h_eq;              /* PhysParams (grid.hpp:31-42) */
    double courant, limiter_theta;  /* SchemeParams (swe.hpp:16-30) */
    double model_dt;
    double q0, l0;                  /* ErrorParams (stochastic.hpp:17-32) */
    int32_t c_omega;                /* CoarseGrid factor (grid.hpp:74-96), odd, divides nx,ny */
    int32_t c_soar;                 /* must be 2 (stochastic.hpp:20,54) */
    uint64_t seed;                  /* experiment master seed (rng.hpp:35-40) */
    int32_t exact_fp;               /* 1: IEEE, no FMA contraction (bitwise reference parity);
                                       0: FMA contraction in the stencil (tolerance parity) */
    int32_t reserved;
} dc_config;

/* Noise sources for model error / filter draws. */
typedef enum dc_noise_mode {
    DC_NOISE_PHILOX = 0,   /* counter-based Philox4x32-10 keyed by stream_seed(seed,tag,member) */
    DC_NOISE_INJECTED = 1  /* host-given offsets + xi (e.g. from the reference NoiseStream) */
} dc_noise_mode;

/* Observation record at t^n (SPEC.md ObservationRecord): location + observed transports. */
typedef struct dc_obs {
    double x, y;       /* m, periodic */
    double y_hu, y_hv; /* m^2/s */
} dc_obs;

/* Per-particle IEWPF diagnostics (SPEC.md ParticleDiagnostics). */
typedef struct dc_particle_diag {
    double c, phi, gamma, zeta, alpha;
} dc_particle_diag;

/* IEWPF variant: the two-stage scheme of the paper (default) or the
 * original one-stage IEWPF (target weight max c_i, update alpha^1/2 P^1/2 xi). */
typedef enum dc_iewpf_mode {
    DC_IEWPF_TWO_STAGE = 0,
    DC_IEWPF_ONE_STAGE = 1
} dc_iewpf_mode;

typedef struct dc_ctx dc_ctx;

/* ---- lifetime ------------------------------------------------------------------ */
/* Create a context holding n_members particles whose global ids are
 * member_base .. member_base+n_members-1 (RNG stream identity uses the global id,
 * rng.hpp:35-40). stream: a cudaStream_t to run on, or NULL for an owned stream.
 * Replaces: Stepper ctor (swe.hpp:194-207) + the ensemble container. */
dc_status dc_create(const dc_config* cfg, int32_t n_members, int64_t member_base,
                    int32_t device, void* stream, dc_ctx** out);
dc_status dc_destroy(dc_ctx* ctx);
dc_status dc_sync(dc_ctx* ctx); /* waits; surfaces device errors */
const char* dc_last_error(dc_ctx* ctx, int32_t* member, int32_t* j, int32_t* k,
                          int32_t* substep);
const char* dc_version(void);

/* ---- state I/O (OceanState, state.hpp:18-31) ---------------------------------- */
dc_status dc_upload_member(dc_ctx* ctx, int32_t m, const float* eta, const float* hu,
                           const float* hv, double t);
dc_status dc_download_member(dc_ctx* ctx, int32_t m, float* eta, float* hu, float* hv,
                             double* t);
/* all members, member-major [n_members][ny][nx]; t may be NULL */
dc_status dc_upload_all(dc_ctx* ctx, const float* eta, const float* hu, const float* hv,
                        const double* t);
dc_status dc_download_all(dc_ctx* ctx, float* eta, float* hu, float* hv, double* t);

/* ---- model operator M (swe.hpp) ----------------------------------------------- */
/* init_double_jet (swe.hpp:459-500), default JetParams, broadcast to every member. */
dc_status dc_init_double_jet(dc_ctx* ctx);
/* n_steps x Stepper::model_step (swe.hpp:244-259) on every member. */
dc_status dc_step(dc_ctx* ctx, int32_t n_steps);
/* Stepper::flux_rhs (swe.hpp:229-239) of member m (synchronous; host outputs). */
dc_status dc_flux_rhs(dc_ctx* ctx, int32_t m, float* d_eta, float* d_hu, float* d_hv);
/* Stepper::cfl_dt (swe.hpp:212-226) of every member (synchronous; host output). */
dc_status dc_cfl_dt(dc_ctx* ctx, double* dt_out);
/* substep counts of the last model step per member (synchronous). */
dc_status dc_substeps(dc_ctx* ctx, int32_t* out);

/* ---- model error (stochastic.hpp) --------------------------------------------- */
/* perturb_state (stochastic.hpp:164-173) on every member. PHILOX: offsets and xi drawn
 * from (seed, model_error, member) at the context's draw counter, which then advances.
 * INJECTED: offsets [n_members][2] and xi [n_members][nxc*nyc] (b-outer, a-inner). */
dc_status dc_perturb(dc_ctx* ctx, int32_t mode, const int32_t* offsets, const double* xi);
/* add_q_half (stochastic.hpp:144-160) of host coarse fields on per-member offsets. */
dc_status dc_add_q_half(dc_ctx* ctx, const int32_t* offsets, const double* coarse,
                        double scale);
dc_status dc_get_draw_counter(dc_ctx* ctx, uint64_t* model_error_draw);
dc_status dc_set_draw_counter(dc_ctx* ctx, uint64_t model_error_draw);
/* StreamTag of the context's model-error draws (rng.hpp:15-23): 1 model_error (default,
 * the ensemble), 3 truth_model_error (the twin experiment's truth run). */
dc_status dc_set_model_error_tag(dc_ctx* ctx, uint64_t tag);

/* ---- observation system ------------------------------------- */
/* innovation of every member at n_obs observations -> d[m][o][2]
 * (synchronous, host output). */
dc_status dc_innovations(dc_ctx* ctx, const dc_obs* obs, int32_t n_obs, double* d_out);
/* observe_mooring without noise on member m -> y[o][2] (synchronous). */
dc_status dc_observe_mooring(dc_ctx* ctx, int32_t m, const double* xy, int32_t n,
                             double* y_out);
/* Per-member drifter copies: positions [n_members][n_d][2]. */
dc_status dc_drifters_set(dc_ctx* ctx, const double* pos, int32_t n_d);
/* advect_drifters, forward Euler at the containing cell. */
dc_status dc_drifters_advect(dc_ctx* ctx, double dt);
/* positions and winding counts [n_members][n_d][2] (synchronous). */
dc_status dc_drifters_get(dc_ctx* ctx, double* pos, int32_t* wind);
/* number of drifter copies per member (DC_ESTATE when none are set). */
dc_status dc_drifters_count(dc_ctx* ctx, int32_t* n_d);
/* restore positions and winding counts [n_members][n_d][2] (checkpoint resume). */
dc_status dc_drifters_restore(dc_ctx* ctx, const double* pos, const int32_t* wind, int32_t n_d);

/* ---- snapshots and checkpoints (state.hpp:43-116) ----------- */
/* The context's parameters and member slice. */
dc_status dc_get_config(dc_ctx* ctx, dc_config* cfg, int32_t* n_members, int64_t* member_base);
/* the model-error stream tag (dc_set_model_error_tag) and IEWPF mode (dc_iewpf_set_mode). */
dc_status dc_get_model_error_tag(dc_ctx* ctx, uint64_t* tag);
dc_status dc_iewpf_get_mode(dc_ctx* ctx, int32_t* mode);
/* save_snapshot (state.hpp:71-85) of member m to a file: "DCST" | u32 version 1 | u32 nx |
 * u32 ny | f64 t | eta f32[nx*ny] | hu | hv, little endian, byte-identical to the
 * reference writer. Synchronous. */
dc_status dc_save_snapshot(dc_ctx* ctx, int32_t m, const char* path);
/* load_snapshot (state.hpp:93-114) into member m, with the reference's checks and
 * messages (bad magic, unsupported version, implausible extents, truncated stream);
 * extents must equal the context grid (DC_EINVAL otherwise). Synchronous. */
dc_status dc_load_snapshot(dc_ctx* ctx, int32_t m, const char* path);
/* Checkpoint directory (SPEC.md ensemble_engine External Interfaces):
 * dir/ensemble/particle_<i>.dcst for every member (global id i), when drifter copies are
 * set dir/ensemble/particle_<i>.drifters ("drifter,x,y,wind_x,wind_y" per line, %.17g),
 * dir/rng_state_<first id>.txt (master seed, model-error draw counter and stream tag,
 * filter cycle, IEWPF mode: the whole counter-based RNG and filter state of the slice)
 * and dir/meta.txt (parameter echo). The directory and dir/ensemble are created if absent.
 * Restoring reproduces the uninterrupted run bit for bit, drifters
 * included; load also accepts the single-context name dir/rng_state.txt. */
dc_status dc_checkpoint_save(dc_ctx* ctx, const char* dir, uint64_t filter_cycle);
dc_status dc_checkpoint_load(dc_ctx* ctx, const char* dir, uint64_t* filter_cycle);

/* ---- twin experiment either side of the path ------------------- */
/* One observation record (SPEC.md ObservationRecord + file grammar). */
typedef struct dc_obs_record {
    double time;      /* s */
    int32_t kind;     /* 0 drifter, 1 mooring */
    int32_t id;       /* platform id */
    double x, y;      /* m */
    double y_hu, y_hv;
} dc_obs_record;
/* Observation noise eps ~ N(0, diag(r_hu, r_hv)) of platforms
 * (kind, ids[i]) at observation index obs_index: counter-based Philox keyed by
 * stream_seed(seed, obs_noise, kind << 32 | id) (rng.hpp:21,35-40), one normal pair per
 * index. eps_out[n][2]. Synchronous. */
dc_status dc_obs_noise(dc_ctx* ctx, int32_t kind, const int32_t* ids, int32_t n,
                       uint64_t obs_index, double r_hu, double r_hv, double* eps_out);
/* observe_drifter of n truth drifters: y = (dx/dt_obs * H_eq,
 * dy/dt_obs * H_eq) + eps, displacement by the minimal periodic image; eps may be NULL.
 * Positions [n][2] wrapped into the domain. Synchronous. */
dc_status dc_observe_drifters(dc_ctx* ctx, const double* prev_xy, const double* cur_xy,
                              int32_t n, double dt_obs, const double* eps, double* y_out);
/* Standard particle-filter log-likelihood -1/2 d^T R^-1 d (R = diag(r_hu, r_hv)) of every
 * member with the eta-compensated innovations -> loglik[n_members];
 * failed members get -inf. Synchronous. */
dc_status dc_pf_loglik(dc_ctx* ctx, const dc_obs* obs, int32_t n_obs, double r_hu, double r_hv,
                       double* loglik_out);
/* Normalised weights from n log-likelihoods (all ranks' values, global particle order);
 * DC_ECOLLAPSE when every exp(loglik) underflows ("ensemble collapse"), with
 * the max log-weight in *max_loglik. Host only. */
dc_status dc_pf_weights(const double* loglik, int32_t n, double* w_out, double* max_loglik);
/* residual_resample: floor(n w_i) copies, residual slots by multinomial
 * draws (Philox keyed by stream_seed(seed, resample, 0), counter {slot, 0, cycle}) ->
 * idx_out[n], ascending. Host only. */
dc_status dc_residual_resample(const double* w, int32_t n, uint64_t seed, uint64_t cycle,
                               int32_t* idx_out);
/* Resampling by copy on the device: member m <- member idx[m] (fields, time, drifter
 * copies), local indices. Synchronous. */
dc_status dc_resample_members(dc_ctx* ctx, const int32_t* idx);
/* Resampling across ranks: a member's whole state -- fields, time,
 * drifter copies -- packed into / unpacked from a device buffer of dc_member_bytes bytes
 * (stream-ordered device copies on the context stream), so ranks can exchange resampled
 * members over NCCL point-to-point. Import invalidates the fused CFL statistics. */
dc_status dc_member_bytes(dc_ctx* ctx, uint64_t* bytes);
dc_status dc_member_export(dc_ctx* ctx, int32_t m, void* d_dst);
dc_status dc_member_import(dc_ctx* ctx, int32_t m, const void* d_src);
/* forecast_error of the drifter copies against
 * truth positions [n_d][2]: E = sqrt(mean_d E_d), E_d = mean over members of the squared
 * minimal-image distance to truth; RMSE likewise about the ensemble mean of the unwrapped
 * positions. Ed / Rd ([n_d]) may be NULL. Synchronous. */
dc_status dc_forecast_error(dc_ctx* ctx, const double* truth_xy, double* E, double* RMSE,
                            double* Ed, double* Rd);
/* Multi-GPU forecast statistics: each rank copies its drifter ensemble
 * into device buffers ([n_members][n_d][2] fp64 positions, int32 winding counts) with
 * dc_drifters_get_device (stream-ordered on the context stream), the ranks gather them
 * in member-id order (NCCL), and one rank evaluates forecast_error over all members with
 * dc_forecast_error_gathered on `stream` of `device` -- bitwise equal to dc_forecast_error
 * of one context holding every member. Both synchronous on return of the statistics. */
dc_status dc_drifters_get_device(dc_ctx* ctx, double* d_pos, int32_t* d_wind);
dc_status dc_forecast_error_gathered(const dc_config* cfg, int32_t device, void* stream,
                                     int32_t n_members, int32_t n_d, const double* d_pos,
                                     const int32_t* d_wind, const double* truth_xy, double* E,
                                     double* RMSE, double* Ed, double* Rd);
/* Observation file: UTF-8 lines "time,kind,id,x,y,y_hu,y_hv" with kind
 * "drifter" | "mooring" and %.17g numbers (exact round trip). read: *n_out = records in
 * the file; recs may be NULL to count; DC_EINVAL if capacity is too small. Host only. */
dc_status dc_obs_file_write(const char* path, const dc_obs_record* recs, int32_t n,
                            int32_t append);
dc_status dc_obs_file_read(const char* path, dc_obs_record* recs, int32_t capacity,
                           int32_t* n_out);
/* Trajectory output: "time,particle,drifter,x,y,wind_x,wind_y" for every
 * member's drifter copies, global particle ids. Synchronous. */
dc_status dc_trajectory_write(dc_ctx* ctx, const char* path, double time, int32_t append);

/* generate_truth on device `device`: a one-member truth run on the
 * truth_model_error stream (model error after every model step), platforms inserted at
 * insert_time (drifters on a drifters_x x drifters_y lattice, advected in the truth;
 * moorings on a moorings_x x moorings_y lattice), one record per platform every
 * obs_interval (a multiple of model_dt) with eps ~ N(0, diag(r_hu, r_hv)). Writes
 * dir/observations.txt and dir/truth_<t>.dcst (t = 0, every snapshot_interval or the end);
 * dir must exist. *n_records = records written. */
typedef struct dc_truth_plan {
    double duration, insert_time, obs_interval, snapshot_interval; /* s */
    int32_t drifters_x, drifters_y;  /* 8 x 8 */
    int32_t moorings_x, moorings_y;  /* 20 x 12 (0: none) */
    double r_hu, r_hv;               /* observation error variances (R = I in the paper) */
} dc_truth_plan;
dc_status dc_generate_truth(const dc_config* cfg, const dc_truth_plan* plan, const char* dir,
                            int32_t device, int64_t* n_records);

/* ---- IEWPF --------------------------------------------------- */
/* precompute_S on the host in fp64: HQH^T and S = (HQH^T+R)^-1,
 * row-major 2x2. Context-free. */
dc_status dc_precompute_S(const dc_config* cfg, double r_hu, double r_hv, double* hqht,
                          double* S);
/* precompute_local_svd: 49x49 block and U Sigma^{1/2} (row-major).
 * Context-free; symmetric eigen-decomposition (the block is symmetric PSD). */
dc_status dc_precompute_local_svd(const dc_config* cfg, const double* S, double* block,
                                  double* usig);
/* Stages 1-3 for the context's particles: innovations, pulls (+phi, c), perpendicular
 * pair (gamma, zeta). Writes this slice's (c_i, zeta_i) pairs to cz_out
 * ([n_members][2], DEVICE pointer if cz_out_is_device, else host, synchronous).
 * cycle selects the filter-stream draw. n_total: global ensemble size N_e. */
dc_status dc_iewpf_begin(dc_ctx* ctx, const dc_obs* obs, int32_t n_obs, const double* S,
                         const double* usig, uint64_t cycle, int32_t n_total, void* cz_out,
                         int32_t cz_out_is_device);
/* Stages 4-6 given ALL particles' (c_i, zeta_i) ([n_total][2], device pointer if
 * cz_is_device): barrier scalars, alpha, P^{1/2} posterior update. */
dc_status dc_iewpf_finish(dc_ctx* ctx, const void* cz_all, int32_t cz_is_device);
/* Single-context convenience: begin + finish without a collective (n_total = n_members). */
/* Select the IEWPF variant for the following analyses (default DC_IEWPF_TWO_STAGE).
 * One-stage: w_target = max_i c_i, c*_i = w_target - c_i, posterior
 * psi^a + alpha^1/2 P^1/2 xi; the reported beta is 0. */
dc_status dc_iewpf_set_mode(dc_ctx* ctx, int32_t mode);
dc_status dc_iewpf_assimilate(dc_ctx* ctx, const dc_obs* obs, int32_t n_obs, const double* S,
                              const double* usig, uint64_t cycle);
/* Diagnostics of the last analysis (synchronous): per particle + (w_target, beta). */
dc_status dc_iewpf_diagnostics(dc_ctx* ctx, dc_particle_diag* per_member, double* w_beta);

/* Per-cycle diagnostics dump (SPEC.md iewpf_filter External Interfaces): lines
 * "cycle,particle,c,gamma,zeta,alpha,beta,w_target" of the last analysis, global particle
 * ids, %.17g. Synchronous. */
dc_status dc_iewpf_diagnostics_write(dc_ctx* ctx, const char* path, uint64_t cycle,
                                     int32_t append);

/* ---- pipelined per-cycle readback ----------------------------------------------
 * dc_readback_enqueue queues, behind the work already on the context stream, copies of
 * the cycle's outputs into one of two pinned slots -- `what` = DC_READBACK_* bits: the
 * particle diagnostics + (w_target, beta) of dc_iewpf_diagnostics, the drifter ensemble
 * of dc_drifters_get, and forecast_error against truth_xy [n_d][2] (copied at the call) --
 * and returns at once. dc_readback_wait(slot) blocks until that slot's copies landed and
 * unpacks them (NULL outputs are skipped); values equal the synchronous calls' bit for
 * bit. A driver enqueues cycle c, queues cycle c+1, then waits for c: the device never
 * idles on the host. Device errors of the queued work surface at the wait. */
#define DC_READBACK_DIAG 1
#define DC_READBACK_DRIFTERS 2
#define DC_READBACK_FORECAST_ERROR 4
dc_status dc_readback_enqueue(dc_ctx* ctx, int32_t slot, int32_t what, const double* truth_xy);
dc_status dc_readback_wait(dc_ctx* ctx, int32_t slot, dc_particle_diag* per_member,
                           double* w_beta, double* pos, int32_t* wind, double* E, double* RMSE);

/* ---- one data-assimilation cycle ----------------------------- */
/* n_steps model steps; model error (PHILOX) after each but the last; drifters advected
 * by model_dt before each step when drifters are set; then the IEWPF analysis
 * (single-context). Stream-ordered, no host sync inside. */
dc_status dc_da_cycle(dc_ctx* ctx, int32_t n_steps, const dc_obs* obs, int32_t n_obs,
                      const double* S, const double* usig, uint64_t cycle);

/* ---- multi-GPU: one process / context per GPU, NCCL over NVLink ---- */
/* Ranks hold contiguous particle ranges in rank order (dc_create's member_base); the
 * host driver creates one NCCL id on rank 0 (dc_comm_unique_id), broadcasts its 128
 * bytes to every rank (MPI_Bcast, a shared file, torch.distributed, ...) and each rank
 * attaches its context (collective: blocks until all ranks joined; checks the partition
 * covers [0, n_total)). While attached, dc_iewpf_assimilate / dc_da_cycle exchange the
 * (c_i, zeta_i) pairs of all ranks at the IEWPF barrier, and dc_forecast_error /
 * dc_readback_enqueue(FORECAST_ERROR) gather every rank's drifter ensemble to rank 0
 * (the other ranks report no statistics: NaN / untouched) -- NCCL send/recv on the
 * context stream, no host synchronisation. Results are bitwise independent of the
 * number of ranks. NCCL is loaded at run time (libnccl.so.2); failures -> DC_ENCCL.
 * Replaces: the spec's worker-pool barrier. */
#define DC_COMM_ID_BYTES 128
dc_status dc_comm_unique_id(uint8_t* id_out);
dc_status dc_comm_attach(dc_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world,
                         int64_t n_total);
dc_status dc_comm_detach(dc_ctx* ctx);
dc_status dc_comm_info(dc_ctx* ctx, int32_t* rank, int32_t* world, int64_t* n_total);

/* ---- instrumentation ------------------------------------------------------------ */
/* number of kernels this context has launched (host-side counter). */
int64_t dc_kernel_launches(dc_ctx* ctx);
/* counters since creation (synchronous): [0] kernels launched, [1] member-substeps
 * (cell-updates / (nx*ny)), [2] substep-loop iterations. */
dc_status dc_counters(dc_ctx* ctx, uint64_t* out);
/* instrumentation for the roofline: n_substeps substeps launched one by one with CUDA
 * events around each stage kernel; ms_out[0..1] = mean stage-1 / stage-2 duration.
 * Advances the state (n_substeps substeps of a model step). */
dc_status dc_time_stages(dc_ctx* ctx, int32_t n_substeps, double* ms_out);
/* Per-kernel profile of everything the calling thread launches between begin and end
 * (any context): each kernel is bracketed by CUDA events on its own stream, and its
 * algorithmic HBM bytes (the data it must read and write once) are
 * accumulated per kernel name. Inside the window dc_step runs its host-driven substep
 * loop, so the stage kernels are timed individually. dc_profile_end synchronises and
 * writes up to cap entries (first-launch order); *n_out = number of distinct kernels. */
typedef struct dc_kernel_time {
    char name[40];
    int64_t launches;
    double ms;     /* summed device time of the launches */
    double bytes;  /* summed algorithmic bytes of the launches */
} dc_kernel_time;
dc_status dc_profile_begin(dc_ctx* ctx);
dc_status dc_profile_end(dc_ctx* ctx, dc_kernel_time* out, int32_t cap, int32_t* n_out);
/* the cudaStream_t the context runs on. */
void* dc_stream(dc_ctx* ctx);
/* Memory checker (no compute-sanitizer on the GPU pool): with DC_GUARD=1 in the
 * environment every device buffer of the library is allocated with 64 KB guard bands
 * (byte pattern) on both sides and its contents poisoned (0xFF bytes: NaN floats) before
 * first use. Synchronises the device and verifies every live guard band: DC_ECUDA and a
 * description (allocation site, side, offset) when a kernel wrote out of bounds; DC_OK
 * (n_bad = 0) otherwise or without DC_GUARD. */
dc_status dc_check_guards(char* msg, int32_t cap, int32_t* n_bad);
/* Exhaustive device self-check of the branch-free IEEE sqrt / reciprocal used by the
 * stencil against the CUDA intrinsics over all positive normal floats (synchronous).
 * counts[0..1] = sqrt / rcp mismatches, counts[2..3] = first mismatching operand bits. */
dc_status dc_selftest_math(int32_t device, uint64_t* counts);

#ifdef __cplusplus
}
#endif

#endif /* DRIFTCAST_GPU_H */
