"""Host-side timing of bench.py's end-to-end loop, call by call (configs[1]).

Prints the mean wall time of each public call in one e2e cycle, to find where the
end-to-end number loses time against the device-timed cycle.
Usage (GPU box): python tools/e2e_probe.py [--cycles 10]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1910_01031_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--members", type=int, default=100)
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    cfg = pkg.Config(nx=500, ny=300)
    n = 3 + 2 * a.cycles
    with torch.cuda.stream(stream):
        obs_all = bench.synthetic_observations(pkg, cfg, n + 1, "drifters", 0, stream.cuda_stream)
        _, S = pkg.precompute_S(cfg)
        _, usig = pkg.precompute_local_svd(cfg, S)
        ens = pkg.Ensemble(cfg, a.members, device=0, stream=stream.cuda_stream)
        ens.init_double_jet()
        ens.drifters_set(bench.platforms(cfg, "drifters")[None].repeat(a.members, 0))
        for c in range(3):
            ens.da_cycle(5, obs_all[c], S, usig, c)
        ens.sync()
        names = ["da_cycle(enqueue)", "sync after cycle", "iewpf_diagnostics",
                 "forecast_error", "drifters_get"]
        acc = {k: 0.0 for k in names}
        # pass 1: the bench's e2e loop, each call timed
        for c in range(3, 3 + a.cycles):
            t0 = time.perf_counter()
            ens.da_cycle(5, obs_all[c], S, usig, c)
            t1 = time.perf_counter()
            ens.iewpf_diagnostics()
            t2 = time.perf_counter()
            ens.forecast_error(obs_all[c][:, :2])
            t3 = time.perf_counter()
            ens.drifters_get()
            t4 = time.perf_counter()
            acc["da_cycle(enqueue)"] += t1 - t0
            acc["iewpf_diagnostics"] += t2 - t1
            acc["forecast_error"] += t3 - t2
            acc["drifters_get"] += t4 - t3
        for k in names:
            print(f"e2e loop  {k:22s} {1e3 * acc[k] / a.cycles:8.3f} ms")
        # pass 2: enqueue, then an explicit sync, then the reads
        acc = {k: 0.0 for k in names}
        for c in range(3 + a.cycles, 3 + 2 * a.cycles):
            t0 = time.perf_counter()
            ens.da_cycle(5, obs_all[c], S, usig, c)
            t1 = time.perf_counter()
            ens.sync()
            t2 = time.perf_counter()
            ens.iewpf_diagnostics()
            t3 = time.perf_counter()
            ens.forecast_error(obs_all[c][:, :2])
            t4 = time.perf_counter()
            ens.drifters_get()
            t5 = time.perf_counter()
            for k, v in zip(names, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
                acc[k] += v
        for k in names:
            print(f"synced    {k:22s} {1e3 * acc[k] / a.cycles:8.3f} ms")
        ens.close()


if __name__ == "__main__":
    main()
