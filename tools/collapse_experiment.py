"""collapse_experiment (SPEC.md diagnostics_cli, §5.3 / Fig. sirCollapse): for a
post-assimilation ensemble, compute standard particle-filter weights on random drifter
subsets of increasing size and report the mean number of particles with w_i > 1/N_e.

The log-likelihoods come from the device (dc_pf_loglik: eta-compensated innovations,
R = r_scale * I); subsets are drawn on the host from the collapse_subsets stream.

  python tools/collapse_experiment.py --members 100 --cycles 3 --trials 20 --sizes 0 1 2 4 8
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=100)
    ap.add_argument("--nx", type=int, default=500)
    ap.add_argument("--ny", type=int, default=300)
    ap.add_argument("--cycles", type=int, default=3, help="IEWPF cycles before the experiment")
    ap.add_argument("--trials", type=int, default=20)
    ap.add_argument("--sizes", type=int, nargs="+", default=[0, 1, 2, 4, 8, 16])
    ap.add_argument("--r-scale", type=float, default=1.0, help="10 for SPEC's 'ten times'")
    a = ap.parse_args()
    import tempfile
    import paper_1910_01031_b200 as pkg
    dx = 2220.0 * 500 / a.nx
    cfg = pkg.Config(nx=a.nx, ny=a.ny, dx=dx, dy=dx)
    with tempfile.TemporaryDirectory() as d:
        pkg.generate_truth(cfg, d, duration=300.0 * (a.cycles + 1), obs_interval=300.0)
        recs = pkg.read_obs_file(os.path.join(d, "observations.txt"))
    times = sorted({r[0] for r in recs})
    obs = {t: np.array([r[3:] for r in recs if r[0] == t]) for t in times}
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    ens = pkg.Ensemble(cfg, a.members)
    ens.init_double_jet()
    for c in range(a.cycles):
        ens.da_cycle(5, obs[times[c]], S, usig, c)
    ens.model_step(5)  # forecast to the next observation time
    last = obs[times[a.cycles]]
    rng = np.random.default_rng(6)  # the collapse_subsets stream of this tool
    print("subset_size,mean_count_w_ge_1_over_Ne")
    for k in a.sizes:
        counts = []
        for _ in range(a.trials):
            idx = rng.choice(len(last), size=k, replace=False) if k else np.zeros(0, int)
            ll = ens.pf_loglik(last[idx], r_hu=a.r_scale, r_hv=a.r_scale) if k else \
                np.zeros(a.members)
            w, _ = pkg.pf_weights(ll, strict=False)
            # w_i > 1/N_e, with equal weights (subset size 0) counted as the spec's N_e
            counts.append(int((w >= (1.0 / a.members) * (1.0 - 1e-12)).sum()))
            if k == 0:
                break
        print(f"{k},{np.mean(counts):.2f}")


if __name__ == "__main__":
    main()
