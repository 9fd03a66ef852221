#!/usr/bin/env python
"""bench.py -- IEWPF data-assimilation cycle throughput on B200 (driver contract).

Workload (default, BASELINE.json configs[4] -- the north-star scale, the largest config
that fits one GPU): the double jet refined 2x per axis, 1000x600 cells (dx=dy=1110 m),
1000 members in total, 64 drifter observations every 5 min, drifter forecast copies in
every member. One bench "step" = one full IEWPF cycle: 5 model steps
of 60 s (CFL substeps on the device), Philox model error after the first 4, drifters
advected in every member each step, then the two-stage IEWPF analysis.

  N GPUs = one process per GPU (torchrun), contiguous particle ranges. Default strong
           scaling: --members-total (1000) split over the ranks; --members M gives weak
           scaling (M per rank). The only collectives are inside the library
           (dc_comm_attach: NCCL over NVLink): the (c_i, zeta_i) exchange at the IEWPF
           barrier and the drifter gather to rank 0 for the forecast statistics.
           torch.distributed (gloo) only carries host plumbing: the NCCL id, the truth
           observations, barriers and the max-over-ranks timing.
  value  = ensemble cell-updates/s (one cell of one member through one SSP-RK2
           substep), device-timed with CUDA events over K cycles, state resident in HBM
  e2e    = the same metric through the C ABI with host buffers: the cycle's observation
           records copied host->device inside the call, per-particle diagnostics, drifter
           positions and forecast statistics E(t)/RMSE(t) read back device->host every
           cycle into pinned slots (cycle c read while c+1 runs), wall-clock timed
  roofline = the dominant kernel (the SWE stage pair) plus a per-kernel table from a
           profile window (dc_profile_begin/end: CUDA events around every launch of 2
           cycles, algorithmic bytes from the launchers) with per-stage shares
  secondary = configs[1] (500x300, 100 members, the paper's setup) at N=1

--impl reference times the reference's own CPU operators (oracle/_ref, compiled from
/root/reference headers: Stepper::model_step + perturb_state, threaded over all host
cores) plus this repo's CPU restatement of the analysis (no reference code exists for
it), on a bounded member sample of the same workload per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ensemble cell-updates/s (IEWPF DA cycle)"
UNIT = "cell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--members-total", type=int, default=1000,
                    help="ensemble size split over the ranks (strong scaling)")
    ap.add_argument("--members", type=int, default=None,
                    help="members per GPU (weak scaling; overrides --members-total)")
    ap.add_argument("--nx", type=int, default=1000)
    ap.add_argument("--ny", type=int, default=600)
    ap.add_argument("--obs", default="drifters", choices=["drifters", "moorings"])
    ap.add_argument("--fast", action="store_true", help="FMA build of the stencil")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs[1] line")
    ap.add_argument("--cpu-members", type=int, default=64,
                    help="member subset of the CPU baseline (scaled linearly)")
    ap.add_argument("--cpu-budget-s", type=float, default=150.0,
                    help="CPU-baseline time budget: up to 5 repetitions within it")
    ap.add_argument("--comm", action="store_true",
                    help="use the library NCCL communicator even at N=1")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def partition(total, world, rank):
    """contiguous particle range of a rank."""
    return total * rank // world, total * (rank + 1) // world


def platforms(cfg, kind):
    """Observation platforms: 64 drifters on an 8x8 lattice or 240 moorings on 12x20,
    25 cells apart where the grid allows."""
    lx, ly = cfg.nx * cfg.dx, cfg.ny * cfg.dy
    if kind == "moorings":
        nxp, nyp = 20, 12
    else:
        nxp, nyp = 8, 8
    xs = (np.arange(nxp) + 0.5) / nxp * lx
    ys = (np.arange(nyp) + 0.5) / nyp * ly
    X, Y = np.meshgrid(xs, ys)
    return np.stack([X.ravel(), Y.ravel()], axis=1)


def synthetic_observations(pkg, cfg, n_cycles, kind, device, stream=None):
    """Twin-experiment observations from the library's own generate_truth
    on this GPU: the truth on the truth_model_error stream with model error every step,
    64 drifters (displacement observations, observe_drifter) or 240 moorings
    (observe_mooring) every 300 s from t = 0, eps ~ N(0, R=I) on the obs_noise streams,
    written to and read back from the observation file. Returns [n_cycles][n_obs][4]
    (x, y, y_hu, y_hv)."""
    import shutil
    import tempfile
    d = tempfile.mkdtemp(prefix="dc_truth_")
    try:
        drifters, moorings = ((8, 8), (0, 0)) if kind == "drifters" else ((0, 0), (20, 12))
        pkg.generate_truth(cfg, d, duration=300.0 * n_cycles, insert_time=0.0,
                           obs_interval=300.0, snapshot_interval=0.0, drifters=drifters,
                           moorings=moorings, device=device)
        recs = pkg.read_obs_file(os.path.join(d, "observations.txt"))
    finally:
        shutil.rmtree(d, ignore_errors=True)
    by_t = {}
    for t, _, _, x, y, yh, yv in recs:
        by_t.setdefault(t, []).append((x, y, yh, yv))
    return np.array([by_t[t] for t in sorted(by_t)][:n_cycles])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": float(max(power)) if power else None}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


# FP32 lane operations per cell of the exact stage kernels: predicated-on FFMA2/FADD2/FMUL2
# (2 each) + FFMA/FADD/FMUL (1) executed per member cell in the ncu source page of the
# final round-2 build's capture (profiles/r2_swe_stage_ncu.json: 201.8 / 224.0 at
# 1000x600), less the 256-for-252-column window halo (x 1000/1024): the work one output
# cell needs. Stage 1, stage 2. (The power-of-two folds and the carried y slopes removed
# ~6 % of them: 210.5 / 232.5 before.)
FP32_OPS_PER_CELL = (197.1, 218.7)

# cycle stages ("stage shares") of every kernel name the profiler reports
STAGE_OF = {
    "swe_stage_pair<1>": "forecast", "swe_stage_pair<2>": "forecast", "fix_ghosts": "forecast",
    "reset_stats": "forecast", "cfl_scan": "forecast", "step_begin": "forecast",
    "count_iters": "forecast", "philox_soar": "model_error", "philox_noise": "model_error",
    "q_half_apply": "model_error", "drifters": "drifters", "forecast_error": "drifters",
}


def config_dict(args, world, nx, ny, members_per_gpu, total, n_obs):
    """The workload description both arms print (identical for the same invocation)."""
    obs = ("64 drifter obs" if args.obs == "drifters" else "240 moored-buoy obs")
    if (nx, ny) == (500, 300):
        which = "configs[1]" if args.obs == "drifters" else "configs[2]"
        name = f"{which}: double-jet IEWPF 500x300 (dx=2220 m)"
    elif (nx, ny) == (1000, 600):
        name = "configs[4]: double jet refined 2x per axis (1000x600, dx=1110 m), IEWPF"
    else:
        name = f"custom: double-jet IEWPF {nx}x{ny}"
    scaling = "weak" if args.members is not None else "strong"
    pitch = (nx + 4 + 31) // 32 * 32
    state_mb = 6 * members_per_gpu * (ny + 4) * pitch * 4 / 1e6
    return {"workload": f"{name}, {total} members in total ({members_per_gpu}/GPU, {scaling} "
                        f"scaling), {obs} every 5 min, drifter forecast copies in every member",
            "nx": nx, "ny": ny, "members_total": total, "members_per_gpu": members_per_gpu,
            "n_obs": int(n_obs), "obs": args.obs,
            "cycle": "5 x 60 s steps, model error after 4, IEWPF analysis",
            "exact_fp": not args.fast, "parallelism": f"ensemble dp{world}",
            "l2": f"inputs larger than L2: state + stage buffers {state_mb:.0f} MB per GPU vs "
                  "126 MB L2"}


def fp32_roofline(ms1, ms2, cells, clocks):
    """Achieved FP32 lane-ops/s of the two stage kernels against B200's FP32 peak
    (148 SMs x 128 lanes x SM clock under load)."""
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = 148 * 128 * mhz * 1e6 / 1e12
    achieved = (FP32_OPS_PER_CELL[0] + FP32_OPS_PER_CELL[1]) * cells / ((ms1 + ms2) / 1e3) / 1e12
    return {"achieved": achieved, "peak": peak, "unit": "T lane-ops/s", "frac": achieved / peak,
            "ops_per_cell_update": sum(FP32_OPS_PER_CELL),
            "peak_basis": f"148 SMs x 128 FP32 lanes x {mhz:.0f} MHz"}


def profiled_traffic():
    """dram bytes per SWE stage launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "swe_stage_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def kernel_table(prof, n_cycles, peak, cycle_ms):
    """Per-kernel roofline rows + stage shares from a dc_profile window of n_cycles."""
    total = sum(ms for _, _, ms, _ in prof) or 1.0
    rows, stages = [], {}
    for name, n, ms, nbytes in prof:
        per_ms = ms / max(1, n)
        gbs = (nbytes / max(1, n)) / (per_ms / 1e3) / 1e9 if per_ms > 0 else 0.0
        rows.append({"kernel": name, "launches_per_cycle": n / n_cycles,
                     "us_per_launch": per_ms * 1e3, "bytes_per_launch": nbytes / max(1, n),
                     "achieved_gbs": gbs, "frac": gbs / peak, "share": ms / total})
        st = STAGE_OF.get(name, "analysis")
        stages[st] = stages.get(st, 0.0) + ms / total
    rows.sort(key=lambda r: -r["share"])
    return {"kernels": rows, "stage_shares": stages,
            "kernel_ms_per_cycle": total / n_cycles, "cycle_ms_graph_path": cycle_ms,
            "basis": "dc_profile window: CUDA events around every launch on its stream over "
                     f"{n_cycles} cycles (stage kernels launched one by one); shares of the "
                     "summed kernel time; algorithmic bytes per launch from the launchers "
                     "(DESIGN.md §4)"}


# ------------------------------------------------------------------------------------
# CPU side: the reference's operators (oracle/_ref) + the analysis restatement
# ------------------------------------------------------------------------------------
def cpu_truth_obs(p, kind):
    """The first cycle's observations of the twin experiment (t = 300 s) replayed on the
    CPU restatement (the GPU generate_truth equals this bit for bit,
    test_generate_truth_matches_oracle)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle
    orc = Oracle()
    s = orc.init_double_jet(p)
    cfgl = type("c", (), {"nx": p.nx, "ny": p.ny, "dx": p.dx, "dy": p.dy})
    pos = platforms(cfgl, kind)
    prev = pos.copy()
    for step in range(5):
        if kind == "drifters":
            orc.advect_drifters(p, s, pos, 60.0)
        orc.model_step(p, s, 1)
        orc.perturb_philox_tag(p, s, 3, 0, step)
    n = len(pos)
    if kind == "drifters":
        eps = orc.obs_noise(p, 0, np.arange(n), 0, 1.0, 1.0)
        y = orc.observe_drifters(p, prev, pos, 300.0, eps)
        return np.hstack([pos, y])
    eps = orc.obs_noise(p, 1, np.arange(n), 0, 1.0, 1.0)
    y = np.array([orc.observe_mooring(p, s, pos[i, 0], pos[i, 1]) for i in range(n)]) + eps
    return np.hstack([pos, y])


def eigh_usig(block):
    """U Sigma^1/2 of the 49x49 local block by eigh, as the GPU arm's
    dc_precompute_local_svd constructs it."""
    w, U = np.linalg.eigh(block)
    return U * np.sqrt(np.maximum(w, 0.0))[None, :]


def cpu_reference_sample(p, obs, n_members, threads, base_state, usig, S):
    """One IEWPF cycle of a member sample on the CPU: the reference's forecast
    (Stepper::model_step + perturb_state, threaded) + the restated analysis (threaded
    over member slices). Returns (seconds, cell-updates, kind)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle, Ref, State, have_ref
    orc = Oracle()
    n = p.nx * p.ny
    e = np.repeat(base_state.eta[None], n_members, 0).copy()
    u = np.repeat(base_state.hu[None], n_members, 0).copy()
    v = np.repeat(base_state.hv[None], n_members, 0).copy()
    pa = np.array([1, 1, 1, 1, 0], np.uint8)
    s0 = State(e[0].copy(), u[0].copy(), v[0].copy())
    if have_ref():
        ref = Ref()
        subs = len(ref.model_step_dts(p, s0))
        t0 = time.perf_counter()
        ref.forecast_threads(p, e, u, v, 5, pa, threads)
        kind = "reference"
    else:
        subs = len(orc.model_step(p, s0, 1))
        t0 = time.perf_counter()
        for m in range(n_members):
            s = State(e[m], u[m], v[m])
            for k in range(5):
                orc.model_step(p, s, 1)
                if k < 4:
                    orc.perturb_philox(p, s, m, k)
        kind = "port"
    per = max(1, (n_members + threads - 1) // threads)
    jobs = []
    for lo in range(0, n_members, per):
        hi = min(n_members, lo + per)
        jobs.append(threading.Thread(target=orc.iewpf_assimilate,
                                     args=(p, e[lo:hi], u[lo:hi], v[lo:hi], obs, S, usig, 0),
                                     kwargs={"member_base": lo}))
    for j in jobs:
        j.start()
    for j in jobs:
        j.join()
    dt = time.perf_counter() - t0
    return dt, n_members * 5 * subs * n, kind


def cpu_setup(nx, ny, kind, obs=None):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle, make_params
    dx = 2220.0 * 500 / nx
    p = make_params(nx=nx, ny=ny, dx=dx, dy=dx)
    orc = Oracle()
    base = orc.init_double_jet(p)
    if obs is None:
        obs = cpu_truth_obs(p, kind)
    _, S = orc.precompute_S(p)
    usig = eigh_usig(orc.local_block(p, S))
    return p, base, obs, S, usig


def cpu_baseline(nx, ny, kind, obs, members, budget_s):
    """Median over up to 5 repetitions (within budget_s) of one cycle of a member subset,
    scaled linearly to the ensemble (members are independent between analyses and the
    metric is per-member intensive). BASELINE.md §2."""
    p, base, obs, S, usig = cpu_setup(nx, ny, kind, obs)
    threads = os.cpu_count() or 1
    times, cu, kind_run = [], 0, "reference"
    while len(times) < 5:
        dt, cu, kind_run = cpu_reference_sample(p, obs, members, threads, base, usig, S)
        times.append(dt)
        if sum(times) + dt > budget_s:
            break
    med = float(np.median(times))
    return {"value": cu / med, "unit": UNIT, "cores": threads, "kind": kind_run,
            "cpu": cpu_model(), "reps": len(times), "rep_s": times,
            "sample": f"{members}-member subset x 1 IEWPF cycle (5 model steps, 4 perturbs, "
                      f"{len(obs)} truth obs, eigh U Sigma^1/2) per repetition, median of "
                      f"{len(times)}; scaled linearly to the full ensemble (cell-updates/s is "
                      f"per-member intensive); forecast on the reference operators over "
                      f"{threads} threads, analysis via the CPU restatement"}


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the CPU reference, one bounded member sample of the
    same workload per step; other ranks exit without work."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = max(2, min(threads, 16))
    p, base, obs, S, usig = cpu_setup(args.nx, args.ny, args.obs)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_reference_sample(p, obs, sample, threads, base, usig, S)
    times, cus, kind = [], 0, "reference"
    for _ in range(args.steps):
        dt, cus, kind = cpu_reference_sample(p, obs, sample, threads, base, usig, S)
        times.append(dt)
    med = float(np.median(times))
    val = cus / med
    total = args.members * world if args.members is not None else args.members_total
    mpg = args.members if args.members is not None else partition(total, world, 0)[1]
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.members is not None else "strong",
        "vs_baseline": None, "dtype": "f32 state / f64 covariance", "data": "synthetic",
        "config": config_dict(args, world, args.nx, args.ny, mpg, total, len(obs)),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": kind,
                         "cpu": cpu_model(),
                         "sample": f"{sample} members x 1 IEWPF cycle per step (forecast via "
                                   f"the reference operators, analysis via the CPU "
                                   f"restatement with the eigh U Sigma^1/2 factor; truth "
                                   f"observations of the twin experiment; {threads} threads); "
                                   f"median over {args.steps} steps; cell-updates/s is "
                                   "per-member intensive"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------
# GPU side
# ------------------------------------------------------------------------------------
class Plumbing:
    """Host-side rank plumbing over torch.distributed (gloo): barriers, broadcasts of host
    arrays, max/sum reductions. No data-path traffic goes through it."""

    def __init__(self, world):
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def bcast_array(self, a, rank):
        if not self.dist:
            return a
        import torch
        shp = torch.tensor(list(a.shape) if rank == 0 else [0, 0, 0], dtype=torch.int64)
        self.dist.broadcast(shp, 0)
        t = torch.from_numpy(np.ascontiguousarray(a)) if rank == 0 else \
            torch.zeros(tuple(int(x) for x in shp), dtype=torch.float64)
        self.dist.broadcast(t, 0)
        return t.numpy()

    def bcast_bytes(self, b, rank, n=128):
        if not self.dist:
            return b
        import torch
        t = torch.tensor(list(b), dtype=torch.uint8) if rank == 0 else torch.zeros(n, dtype=torch.uint8)
        self.dist.broadcast(t, 0)
        return bytes(t.tolist())

    def max_sum(self, tmax, total):
        if not self.dist:
            return tmax, total
        import torch
        a = torch.tensor([tmax], dtype=torch.float64)
        b = torch.tensor([total], dtype=torch.float64)
        self.dist.all_reduce(a, op=self.dist.ReduceOp.MAX)
        self.dist.all_reduce(b, op=self.dist.ReduceOp.SUM)
        return float(a.item()), float(b.item())

    def all_gather_host(self, t):
        import torch
        parts = [torch.zeros_like(t) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(parts, t)
        return torch.cat(parts)

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


def run_config(pkg, args, pl, rank, world, local, nx, ny, M, base, total, K, W, profile=True,
               clocks=True):
    """K timed cycles (device), K e2e cycles (wall clock, host buffers), a profile window;
    returns the metrics of this rank (max/sum over ranks applied)."""
    import torch
    stream = torch.cuda.Stream(device=local)
    dx = 2220.0 * 500 / nx  # the double-jet domain is fixed; refining shrinks dx
    cfg = pkg.Config(nx=nx, ny=ny, dx=dx, dy=dx, exact_fp=not args.fast)
    n_prof = 2 if profile else 0
    n_cycles = W + 2 * K + n_prof
    obs_all = None
    if rank == 0:
        obs_all = synthetic_observations(pkg, cfg, n_cycles + 1, args.obs, local)
    obs_all = pl.bcast_array(obs_all, rank)  # the truth is generated once, on rank 0
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    # host-staged test path (two ranks sharing one GPU, where NCCL cannot run): the
    # (c, zeta) pairs and drifters gathered through gloo between iewpf_begin / _finish
    staged = world > 1 and os.environ.get("DC_BENCH_BACKEND") == "gloo"
    ens = pkg.Ensemble(cfg, M, member_base=base, device=local, stream=stream.cuda_stream)
    use_comm = (world > 1 and not staged) or args.comm
    if use_comm:
        nid = pkg.comm_unique_id() if rank == 0 else bytes(128)
        nid = pl.bcast_bytes(nid, rank)
        ens.comm_attach(nid, rank, world, total)
    ens.init_double_jet()
    drift0 = platforms(cfg, "drifters")
    n_d = len(drift0)
    ens.drifters_set(drift0[None].repeat(M, 0))
    if staged:
        cz_local = torch.zeros((M, 2), dtype=torch.float64, device=f"cuda:{local}")
        cz_all = torch.zeros((total, 2), dtype=torch.float64, device=f"cuda:{local}")

    def cycle(c):
        obs = obs_all[c]
        if not staged:
            ens.da_cycle(5, obs, S, usig, c)
            return
        with torch.cuda.stream(stream):
            ens.da_cycle(5, np.zeros((0, 4)), S, usig, c)  # forecast + drifters only
            ens.iewpf_begin(obs, S, usig, c, total, cz_ptr=cz_local.data_ptr())
            cz_all.copy_(pl.all_gather_host(cz_local.cpu()))
            ens.iewpf_finish(cz_ptr=cz_all.data_ptr())

    clk = ClockSampler(local) if clocks else None
    if clk:
        clk.start()
    for c in range(W):
        cycle(c)
    ens.sync()
    pl.barrier()
    l0, cs0, _ = ens.counters()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(local)
    pl.barrier()
    ev0.record(stream)
    for c in range(W, W + K):
        cycle(c)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize(local)
    pl.barrier()
    ms = ev0.elapsed_time(ev1)
    l1, cs1, _ = ens.counters()
    ens.sync()
    cell_updates = (cs1 - cs0) * nx * ny
    ms, cell_updates = pl.max_sum(ms, float(cell_updates))
    value = cell_updates / (ms / 1e3)

    # ---- end to end through the C ABI with host buffers ----
    diag_bytes = M * 4 + M * 8 * 8 + 16  # err flags + per-particle scalars + (w, beta)
    drift_bytes = M * n_d * 2 * (8 + 4)
    obs_bytes = obs_all.shape[1] * 32
    truth_ok = args.obs == "drifters" and obs_all.shape[1] == n_d
    fe_bytes = 16 * n_d if truth_ok and rank == 0 else 0  # E_d, RMSE_d per drifter
    truth_bytes = 16 * n_d if truth_ok and rank == 0 else 0  # truth positions H2D
    gather_note = None
    if truth_ok and staged:
        gather_note = "host-staged drifter gather (test path)"
        lpos = torch.empty((M, n_d, 2), dtype=torch.float64, device=f"cuda:{local}")
        lwind = torch.empty((M, n_d, 2), dtype=torch.int32, device=f"cuda:{local}")
        gpos = torch.empty((total, n_d, 2), dtype=torch.float64, device=f"cuda:{local}")
        gwind = torch.empty((total, n_d, 2), dtype=torch.int32, device=f"cuda:{local}")

        def staged_stats(c):
            ens.drifters_to_device(lpos.data_ptr(), lwind.data_ptr())
            gpos.copy_(pl.all_gather_host(lpos.cpu()))
            gwind.copy_(pl.all_gather_host(lwind.cpu()))
            if rank == 0:
                pkg.forecast_error_gathered(cfg, total, n_d, gpos.data_ptr(), gwind.data_ptr(),
                                            obs_all[c][:, :2], device=local,
                                            stream=stream.cuda_stream)

    pl.barrier()
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e2e_cu0 = ens.counters()[1]
    ev2.record(stream)
    # each cycle's outputs (per-particle diagnostics + (w, beta), the drifter forecast
    # ensemble, E(t) / RMSE(t) against the truth drifters -- gathered to rank 0 by the
    # library at N > 1) go D2H into a pinned slot queued behind the cycle; the host reads
    # cycle c while cycle c+1 runs
    for i, c in enumerate(range(W + K, W + 2 * K)):
        cycle(c)
        if truth_ok and not staged:
            ens.readback_enqueue(i % 2, truth_xy=obs_all[c][:, :2])
        else:
            ens.readback_enqueue(i % 2)
            if truth_ok:
                staged_stats(c)
        if i > 0:
            ens.readback_wait((i - 1) % 2)
    ev3.record(stream)
    ens.readback_wait((K - 1) % 2)
    torch.cuda.synchronize(local)
    wall = time.perf_counter() - t0
    e2e_dev_ms = ev2.elapsed_time(ev3)  # the same region on the device clock
    e2e_cu = (ens.counters()[1] - e2e_cu0) * nx * ny
    wall, e2e_cu = pl.max_sum(wall, float(e2e_cu))
    e2e_value = e2e_cu / wall
    clk_res = clk.stop() if clk else None

    # ---- per-kernel profile window (2 cycles, every launch bracketed by events) ----
    prof = None
    if profile:
        pl.barrier()
        ens.profile_begin()
        for c in range(W + 2 * K, W + 2 * K + n_prof):
            cycle(c)
        prof = ens.profile_end()
    ens.sync()
    ens.close()
    return {"value": value, "ms": ms, "K": K, "cell_updates": cell_updates,
            "launches": int(l1 - l0), "e2e_value": e2e_value, "e2e_ms": wall * 1e3 / K,
            "e2e_dev_ms": e2e_dev_ms / K,
            "h2d": obs_bytes + truth_bytes, "d2h": diag_bytes + drift_bytes + fe_bytes,
            "n_obs": obs_all.shape[1], "obs0": obs_all[0], "prof": prof, "n_prof": n_prof,
            "clocks": clk_res, "cells": M * nx * ny, "comm": use_comm, "gather": gather_note}


def roofline_block(r, peak, peak_src):
    """The dominant kernel (the SWE stage pair, one substep = one launch of each stage)
    + the per-kernel table."""
    by = {name: (n, ms, b) for name, n, ms, b in r["prof"]}
    n1, ms1, b1 = by["swe_stage_pair<1>"]
    n2, ms2, b2 = by["swe_stage_pair<2>"]
    t1, t2 = ms1 / n1, ms2 / n2  # ms per launch
    achieved = (b1 / n1 + b2 / n2) / ((t1 + t2) / 1e3) / 1e9
    cells = r["cells"]
    tbl = kernel_table(r["prof"], r["n_prof"], peak, r["ms"] / r["K"])
    tr = profiled_traffic()
    traffic = None
    if tr and tr.get("dram_bytes_per_cell_pair"):
        # DRAM bytes of one stage-1 + one stage-2 launch per cell (intensive in the member
        # count: the state is far larger than L2 either way), scaled to this launch size
        traffic = tr["dram_bytes_per_cell_pair"] * cells / 2.0
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_note": ("mean DRAM bytes of a stage launch (ncu --set full, "
                             f"{(tr or {}).get('source')}), per launch like achieved"
                             if traffic is not None else "no ncu capture committed"),
            "kernel": "swe_stage_pair<1>+<2> (one SSP-RK2 substep: 24 B/cell stage 1, 36 B/cell "
                      "stage 2 algorithmic, SURVEY.md §8d)",
            "stage_ms": [t1, t2], "peak_source": peak_src,
            "note": "the stage kernel is FP32-pipe bound, not HBM bound (DESIGN.md §4): see "
                    "fp32 for the binding roofline",
            "fp32": fp32_roofline(t1, t2, cells, r["clocks"]),
            "single_sweep_24B": {"achieved": 24.0 * cells / ((t1 + t2) / 1e3) / 1e9,
                                 "frac": 24.0 * cells / ((t1 + t2) / 1e3) / 1e9 / peak},
            **tbl}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_1910_01031_b200 as pkg

    # DC_BENCH_DEVICE exists only to run several ranks on a single-GPU box (test path)
    if os.environ.get("DC_BENCH_DEVICE") is not None:
        local = int(os.environ["DC_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    pl = Plumbing(world)
    if args.members is not None:
        total = args.members * world
        base, M = rank * args.members, args.members
    else:
        total = args.members_total
        lo, hi = partition(total, world, rank)
        base, M = lo, hi - lo
    K, W = args.steps, args.warmup
    r = run_config(pkg, args, pl, rank, world, local, args.nx, args.ny, M, base, total, K, W)
    sec = None
    if world == 1 and not args.no_secondary and (args.nx, args.ny) != (500, 300):
        s = run_config(pkg, args, pl, rank, world, local, 500, 300, 100, 0, 100, K, W,
                       profile=True, clocks=False)
        sec = s
    if rank != 0:
        pl.close()
        return
    peaks, peak_src = load_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.nx, args.ny, args.obs, r["obs0"], args.cpu_members,
                               args.cpu_budget_s)
        except Exception as ex:  # the checker is optional on the box; never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": f"{type(ex).__name__}: {ex}"}
    roof = roofline_block(r, peak, peak_src)
    line = {
        "metric": METRIC,
        "value": r["value"],
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": r["ms"] / K,
        "higher_is_better": True,
        "scaling": "weak" if args.members is not None else "strong",
        "vs_baseline": None,
        "dtype": "f32 state (SWE stencil) / f64 covariance + filter scalars",
        "data": "synthetic: double-jet IC, Philox model error, generate_truth twin experiment with "
                f"{r['n_obs']} {args.obs}, R=I",
        "config": config_dict(args, world, args.nx, args.ny, M, total, r["n_obs"]),
        "cycle_ms": r["ms"] / K,
        "e2e": {"value": r["e2e_value"], "unit": UNIT, "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"], "ms_per_step": r["e2e_ms"],
                "device_ms_per_step": r["e2e_dev_ms"]},
        "gpu_launches": r["launches"],
        "collectives": ("library NCCL (dc_comm_attach): (c_i, zeta_i) exchange at the IEWPF "
                        "barrier + drifter gather to rank 0" if r["comm"] else
                        (r["gather"] or "none (single context)")),
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": r["clocks"],
    }
    if sec is not None:
        sroof = roofline_block(sec, peak, peak_src)
        line["secondary"] = {
            "config": config_dict(args, 1, 500, 300, 100, 100, sec["n_obs"]),
            "value": sec["value"], "unit": UNIT, "cycle_ms": sec["ms"] / K,
            "e2e": {"value": sec["e2e_value"], "unit": UNIT, "ms_per_step": sec["e2e_ms"],
                    "h2d_bytes_per_step": sec["h2d"], "d2h_bytes_per_step": sec["d2h"]},
            "gpu_launches": sec["launches"],
            "roofline": {k: sroof[k] for k in ("achieved", "peak", "frac", "stage_ms", "fp32",
                                               "stage_shares", "kernel_ms_per_cycle")},
        }
    print(json.dumps(line), flush=True)
    pl.close()


if __name__ == "__main__":
    main()
