"""Quick forecast throughput probe (development aid, not the bench contract).

Times model_step (+ optional perturb) over N members with CUDA events on the library's
stream and prints cell-updates/s.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=100)
    ap.add_argument("--nx", type=int, default=500)
    ap.add_argument("--ny", type=int, default=300)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--fast", action="store_true")
    ap.add_argument("--perturb", action="store_true")
    a = ap.parse_args()
    import torch
    from paper_1910_01031_b200 import Config, Ensemble

    cfg = Config(nx=a.nx, ny=a.ny, dx=2220.0 * 500 / a.nx, dy=2220.0 * 500 / a.nx,
                 exact_fp=not a.fast)
    s = torch.cuda.Stream()
    ens = Ensemble(cfg, a.members, stream=s.cuda_stream)
    ens.init_double_jet()
    for _ in range(3):
        ens.model_step(1)
        if a.perturb:
            ens.perturb_state()
    ens.sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ens.kernel_launches()
    ev0.record(s)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        ens.model_step(1)
        if a.perturb:
            ens.perturb_state()
    ev1.record(s)
    ev1.synchronize()
    wall = time.perf_counter() - t0
    ms = ev0.elapsed_time(ev1)
    subs = ens.substeps()
    cells = a.nx * a.ny * a.members
    cu = cells * float(subs.mean()) * a.steps
    print(f"members={a.members} grid={a.nx}x{a.ny} exact={not a.fast} perturb={a.perturb}")
    print(f"substeps/step={subs.mean():.2f}  device ms={ms:.3f} wall ms={wall*1e3:.3f}")
    print(f"cell-updates/s = {cu / (ms / 1e3):.4e}   ms/model-step = {ms / a.steps:.4f}")
    print(f"HBM-equivalent (60 B/cell-update) = {cu * 60 / (ms / 1e3) / 1e9:.1f} GB/s")
    print(f"kernels launched in timed region: {ens.kernel_launches() - l0}")
    ens.sync()


if __name__ == "__main__":
    main()
