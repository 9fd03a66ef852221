"""Profiling driver: one warm-up + one measured IEWPF cycle of the bench workload
(--members, --nx x --ny, 64 drifters or 240 moorings) with synthetic observations made on
the host, so every kernel launch belongs to the ensemble (no truth run). Use with
DC_NO_GRAPH=1 so ncu sees the stage kernels as individual launches."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--obs", default="drifters", choices=["drifters", "moorings"])
    ap.add_argument("--members", type=int, default=100)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--nx", type=int, default=500)
    ap.add_argument("--ny", type=int, default=300)
    a = ap.parse_args()
    import paper_1910_01031_b200 as pkg
    from bench import platforms
    dx = 2220.0 * 500 / a.nx
    cfg = pkg.Config(nx=a.nx, ny=a.ny, dx=dx, dy=dx)
    ens = pkg.Ensemble(cfg, a.members)
    ens.init_double_jet()
    pos = platforms(cfg, a.obs)
    ens.drifters_set(platforms(cfg, "drifters")[None].repeat(a.members, 0))
    rng = np.random.default_rng(0)
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    for c in range(a.cycles):
        obs = np.hstack([pos, rng.normal(0, 20, size=(len(pos), 2))])
        ens.da_cycle(5, obs, S, usig, c)
    ens.sync()
    print("cycles done", a.cycles)


if __name__ == "__main__":
    main()
