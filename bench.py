#!/usr/bin/env python
"""bench.py -- IEWPF data-assimilation cycle throughput on B200 (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on for one GPU):
double-jet ensemble, 500x300 cells (dx=dy=2220 m), 100 members per GPU, 64 drifter
observations every 5 min. One bench "step" = one full IEWPF cycle:
5 model steps of 60 s (CFL substeps on the device), Philox model error after the first
4, drifters advected in every member each step, then the two-stage IEWPF analysis.

  value  = ensemble cell-updates/s (one cell of one member through one SSP-RK2
           substep), device-timed with CUDA events over K cycles, state resident in HBM
  e2e    = the same metric through the C ABI with host buffers: the cycle's observation
           records (and the truth drifter positions) copied host->device inside the calls,
           per-particle diagnostics, drifter positions and forecast statistics read back
           device->host every cycle into pinned slots (cycle c read while c+1 runs),
           wall-clock timed
  N > 1  = one process per GPU (torchrun), 100 members per rank (weak scaling); the
           only collective is the NCCL all-gather of (c_i, zeta_i) at the IEWPF barrier.

--impl reference times the reference's own CPU operators (oracle/_ref, compiled from
/root/reference headers: Stepper::model_step + perturb_state, threaded over all host
cores) plus this repo's CPU restatement of the analysis (no reference code exists for
it), on a bounded sample of the same workload.
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
    ap.add_argument("--members", type=int, default=100, help="members per GPU")
    ap.add_argument("--nx", type=int, default=500)
    ap.add_argument("--ny", type=int, default=300)
    ap.add_argument("--obs", default="drifters", choices=["drifters", "moorings"])
    ap.add_argument("--fast", action="store_true", help="FMA build of the stencil")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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


def synthetic_observations(pkg, cfg, n_cycles, kind, device, stream):
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


def reduce_max_sum(dist, backend, local, tmax, total):
    """max over ranks of a time, sum over ranks of a count."""
    import torch
    dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    a = torch.tensor([tmax], dtype=torch.float64, device=dev)
    b = torch.tensor([total], dtype=torch.float64, device=dev)
    dist.all_reduce(a, op=dist.ReduceOp.MAX)
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    return float(a.item()), float(b.item())


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


# FP32 lane operations per cell of the exact stage kernels, counted from their SASS
# (FFMA2/FADD2/FMUL2 = 2, FFMA/FADD/FMUL = 1; tools/sass_hist.py): stage 1, stage 2
FP32_OPS_PER_CELL = (208.0, 229.0)


def workload_name(args, M):
    """Which BASELINE.json config this run is (configs[1] is the default)."""
    obs = ("64 drifter obs" if args.obs == "drifters" else "240 moored-buoy obs")
    if (args.nx, args.ny) == (500, 300):
        which = "configs[1]" if args.obs == "drifters" else "configs[2]"
        return (f"{which}: double-jet IEWPF 500x300, {M} members/GPU, {obs} every 5 min, "
                "drifter forecast copies in every member")
    if (args.nx, args.ny) == (1000, 600):
        return (f"configs[4]: double jet refined 2x per axis (1000x600, dx=1110 m), IEWPF, "
                f"{M} members/GPU, {obs} every 5 min")
    return f"custom: double-jet IEWPF {args.nx}x{args.ny}, {M} members/GPU, {obs}"


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
            return json.load(f).get("dram_bytes_per_launch")
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


def cpu_reference_sample(cfg_params, obs, n_members, threads, base_state):
    """The reference's CPU forecast (Stepper::model_step + perturb_state, threaded) for a
    bounded member sample + the restated analysis on that sample. Returns
    (seconds, cell-updates)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle, Ref, State, have_ref
    p = cfg_params
    orc = Oracle()
    n = p.nx * p.ny
    e = np.repeat(base_state.eta[None], n_members, 0).copy()
    u = np.repeat(base_state.hu[None], n_members, 0).copy()
    v = np.repeat(base_state.hv[None], n_members, 0).copy()
    pa = np.array([1, 1, 1, 1, 0], np.uint8)
    # substeps of one model step (identical across members for the jet at this horizon)
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
    _, S = orc.precompute_S(p)
    usig = np.linalg.cholesky(orc.local_block(p, S))
    # analysis: member slices on all threads (ctypes releases the GIL); each slice runs
    # the full six stages, so the work equals one N_e = n_members analysis
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


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the CPU reference on a bounded sample per step."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from checkers import Oracle, make_params
    p = make_params(nx=args.nx, ny=args.ny, dx=2220.0 * 500 / args.nx, dy=2220.0 * 500 / args.nx)
    threads = os.cpu_count() or 1
    sample = max(2, threads)
    orc = Oracle()
    base = orc.init_double_jet(p)
    rng = np.random.default_rng(0)
    pos = platforms(type("c", (), {"nx": p.nx, "ny": p.ny, "dx": p.dx, "dy": p.dy}), args.obs)
    obs = np.hstack([pos, rng.normal(0, 20, size=(len(pos), 2))])
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_reference_sample(p, obs, sample, threads, base)
    times, cus, kind = [], 0, "reference"
    for _ in range(args.steps):
        dt, cu, kind = cpu_reference_sample(p, obs, sample, threads, base)
        times.append(dt)
        cus = cu
    med = float(np.median(times))
    val = cus / med
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 state / f64 covariance", "data": "synthetic",
        "config": {"workload": workload_name(args, args.members),
                   "cycle": "5 x 60 s steps, model error after 4, IEWPF analysis",
                   "members_sampled": sample, "nx": p.nx, "ny": p.ny, "obs": args.obs},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": kind, "cpu": cpu_model(),
                         "sample": f"{sample} members x 1 IEWPF cycle per step (forecast via "
                                   f"the reference operators, analysis via the CPU "
                                   f"restatement; both on {threads} threads)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist  # noqa: F401  (ranks other than 0 just exit)
        run_reference(args, rank, world)
        return

    import torch
    import paper_1910_01031_b200 as pkg

    # DC_BENCH_DEVICE / DC_BENCH_BACKEND=gloo exist only to exercise the multi-rank logic
    # on a single-GPU box (ranks share the device, the all-gather is staged via the host);
    # the product path is one GPU per rank over NCCL.
    if os.environ.get("DC_BENCH_DEVICE") is not None:
        local = int(os.environ["DC_BENCH_DEVICE"])
    backend = os.environ.get("DC_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or (os.environ.get("DC_BENCH_FORCE_SPLIT") == "1" and "RANK" in os.environ):
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.Stream()
    dx = 2220.0 * 500 / args.nx  # the double-jet domain is fixed; refining shrinks dx
    cfg = pkg.Config(nx=args.nx, ny=args.ny, dx=dx, dy=dx, exact_fp=not args.fast)
    M = args.members
    K, W = args.steps, args.warmup
    total = M * world
    with torch.cuda.stream(stream):
        obs_all = synthetic_observations(pkg, cfg, W + 2 * K + 1, args.obs, local, stream.cuda_stream)
        _, S = pkg.precompute_S(cfg)
        _, usig = pkg.precompute_local_svd(cfg, S)
        ens = pkg.Ensemble(cfg, M, member_base=rank * M, device=local, stream=stream.cuda_stream)
        ens.init_double_jet()
        drift0 = platforms(cfg, "drifters")
        ens.drifters_set(drift0[None].repeat(M, 0))
        cz_local = torch.zeros((M, 2), dtype=torch.float64, device=f"cuda:{local}")
        cz_all = torch.zeros((total, 2), dtype=torch.float64, device=f"cuda:{local}")

        split = world > 1 or os.environ.get("DC_BENCH_FORCE_SPLIT") == "1"

        def cycle(c):
            obs = obs_all[c]
            if not split:
                ens.da_cycle(5, obs, S, usig, c)
            else:
                ens.da_cycle(5, np.zeros((0, 4)), S, usig, c)  # forecast + drifters only
                ens.iewpf_begin(obs, S, usig, c, total, cz_ptr=cz_local.data_ptr())
                if dist is None:  # single process forced through the split path
                    cz_all.copy_(cz_local)
                elif backend == "nccl":
                    dist.all_gather_into_tensor(cz_all, cz_local)
                else:  # host-staged test path
                    host = cz_local.cpu()
                    parts = [torch.zeros_like(host) for _ in range(world)]
                    dist.all_gather(parts, host)
                    cz_all.copy_(torch.cat(parts))
                ens.iewpf_finish(cz_ptr=cz_all.data_ptr())

        clk = ClockSampler(local)
        clk.start()
        for c in range(W):
            cycle(c)
        ens.sync()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        l0, cs0, _ = ens.counters()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        for c in range(W, W + K):
            cycle(c)
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        l1, cs1, _ = ens.counters()
        ens.sync()
        cell_updates = (cs1 - cs0) * cfg.nx * cfg.ny
        if dist:
            ms, cell_updates = reduce_max_sum(dist, backend, local, ms, float(cell_updates))
        value = cell_updates / (ms / 1e3)

        # ---- end to end through the C ABI with host buffers ----
        # pipelined readback slots: err flags + the raw per-particle scalars + (w, beta)
        diag_bytes = M * 4 + M * 8 * 8 + 16
        n_d = len(drift0)
        drift_bytes = M * n_d * 2 * (8 + 4)
        obs_bytes = obs_all.shape[1] * 32
        # forecast statistics against the truth drifters: one rank holds
        # every member's drifters after an all-gather in member-id order
        truth_ok = args.obs == "drifters" and obs_all.shape[1] == n_d
        fe_bytes = 16 * n_d if truth_ok and rank == 0 else 0  # E_d, RMSE_d per drifter
        truth_bytes = 16 * n_d if truth_ok and rank == 0 else 0  # truth positions H2D
        if truth_ok and dist is not None:
            dev = f"cuda:{local}"
            lpos = torch.empty((M, n_d, 2), dtype=torch.float64, device=dev)
            lwind = torch.empty((M, n_d, 2), dtype=torch.int32, device=dev)
            gpos = torch.empty((total, n_d, 2), dtype=torch.float64, device=dev)
            gwind = torch.empty((total, n_d, 2), dtype=torch.int32, device=dev)

        def forecast_stats(c):
            truth = obs_all[c][:, :2]
            if dist is None:
                return ens.forecast_error(truth)
            ens.drifters_to_device(lpos.data_ptr(), lwind.data_ptr())
            if backend == "nccl":
                dist.all_gather_into_tensor(gpos, lpos)
                dist.all_gather_into_tensor(gwind, lwind)
            else:  # host-staged test path
                for src, dst in ((lpos, gpos), (lwind, gwind)):
                    host = src.cpu()
                    parts = [torch.zeros_like(host) for _ in range(world)]
                    dist.all_gather(parts, host)
                    dst.copy_(torch.cat(parts))
            if rank == 0:
                return pkg.forecast_error_gathered(cfg, total, n_d, gpos.data_ptr(),
                                                   gwind.data_ptr(), truth, device=local,
                                                   stream=stream.cuda_stream)
            return None

        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        e2e_cu0 = ens.counters()[1]
        # each cycle's outputs (per-particle diagnostics + (w, beta), the drifter forecast
        # ensemble, E(t) / RMSE(t) against the truth drifters) go D2H into a pinned slot
        # queued behind the cycle; the host reads cycle c while cycle c+1 runs
        for i, c in enumerate(range(W + K, W + 2 * K)):
            cycle(c)
            if truth_ok and dist is None:
                ens.readback_enqueue(i % 2, truth_xy=obs_all[c][:, :2])
            else:
                ens.readback_enqueue(i % 2)
                if truth_ok:
                    forecast_stats(c)  # ranks gather drifters, rank 0 evaluates (synchronous)
            if i > 0:
                ens.readback_wait((i - 1) % 2)
        ens.readback_wait((K - 1) % 2)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_cu = (ens.counters()[1] - e2e_cu0) * cfg.nx * cfg.ny
        if dist:
            wall, e2e_cu = reduce_max_sum(dist, backend, local, wall, float(e2e_cu))
        e2e_value = e2e_cu / wall
        clocks = clk.stop()  # sampled from warm-up through the timed and e2e regions

        # ---- roofline of the dominant kernel (SWE stage), CUDA events per launch ----
        ms1, ms2 = ens.time_stages(7)
        cells = M * cfg.nx * cfg.ny
        bytes1, bytes2 = 24.0 * cells, 36.0 * cells  # algorithmic (60 B/cell-update)
        achieved = (bytes1 + bytes2) / ((ms1 + ms2) / 1e3) / 1e9
        peaks, peak_src = load_peaks()
        peak = float(peaks.get("hbm_gbs", 6650.0))
        traffic = profiled_traffic()
        ens.sync()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            from checkers import Oracle, make_params
            p = make_params(nx=cfg.nx, ny=cfg.ny, dx=cfg.dx, dy=cfg.dy)
            threads = os.cpu_count() or 1
            sample = max(2, min(threads, 16))
            base = Oracle().init_double_jet(p)
            dt, cu, kind = cpu_reference_sample(p, obs_all[0], sample, threads, base)
            cpu = {"value": cu / dt, "unit": UNIT, "cores": threads, "kind": kind, "cpu": cpu_model(),
                   "sample": f"{sample} members x 1 IEWPF cycle (5 model steps, 4 perturbs, "
                             f"{obs_all.shape[1]} obs): forecast on the reference operators "
                             f"over {threads} threads, analysis via the CPU restatement"}
        except Exception as ex:  # the checker is optional on the box; never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": f"{type(ex).__name__}: {ex}"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 state (SWE stencil) / f64 covariance + filter scalars",
        "data": "synthetic: double-jet IC, Philox model error, generate_truth twin experiment with "
                f"{obs_all.shape[1]} {args.obs}, R=I",
        "config": {"workload": workload_name(args, M),
                   "nx": cfg.nx, "ny": cfg.ny, "members_per_gpu": M, "members_total": total,
                   "n_obs": int(obs_all.shape[1]), "obs": args.obs, "cycle": "5 x 60 s steps, "
                   "model error after 4, IEWPF analysis", "exact_fp": not args.fast,
                   "parallelism": f"ensemble dp{world}",
                   "l2": f"inputs larger than L2: the state + stage buffers are 6 x {M} x {cfg.ny} x "
                         f"{(cfg.nx + 31) // 32 * 32} x 4 B = "
                         f"{6 * M * cfg.ny * ((cfg.nx + 31) // 32 * 32) * 4 / 1e6:.0f} MB vs 126 MB L2"},
        "cycle_ms": ms / K,
        "cell_model_steps_per_s": value / max(1.0, cell_updates / (K * 5 * total * cfg.nx * cfg.ny)),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": obs_bytes + truth_bytes,
                "d2h_bytes_per_step": diag_bytes + drift_bytes + fe_bytes,
                "ms_per_step": wall * 1e3 / K},
        "gpu_launches": int(l1 - l0),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "swe_stage (SSP-RK2 stage, 24 B/cell stage 1, 36 B/cell stage 2)",
                     "stage_ms": [ms1, ms2], "peak_source": peak_src,
                     "note": "the stage kernel is FP32-pipe bound, not HBM bound (DESIGN.md "
                             "§4): see fp32 for the binding roofline",
                     "fp32": fp32_roofline(ms1, ms2, cells, clocks),
                     # the 24 B/cell-update lower bound of a single-sweep
                     # substep (read psi, write psi), at the same substep time
                     "single_sweep_24B": {"achieved": 24.0 * cells / ((ms1 + ms2) / 1e3) / 1e9,
                                          "frac": 24.0 * cells / ((ms1 + ms2) / 1e3) / 1e9 / peak}},
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
