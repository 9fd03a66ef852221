"""Tiny model-step probe (development aid): 2 members of a 100x60 jet, one model step,
compared bitwise against the CPU oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    ny = int(sys.argv[2]) if len(sys.argv) > 2 else 60
    nm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    co = 5 if (nx % 5 == 0 and ny % 5 == 0) else 1
    from checkers import Oracle, make_params
    from paper_1910_01031_b200 import Config, Ensemble
    cfg = Config(nx=nx, ny=ny, c_omega=co)
    p = make_params(nx=nx, ny=ny, c_omega=co)
    orc = Oracle()
    ens = Ensemble(cfg, nm, device=0)
    ens.init_double_jet()
    ens.model_step(1)
    e, u, v, t = ens.download()
    s = orc.init_double_jet(p)
    orc.model_step(p, s, 1)
    print(nx, ny, nm, end=": ")
    for m in range(nm):
        ok = np.array_equal(e[m], s.eta) and np.array_equal(u[m], s.hu) and np.array_equal(v[m], s.hv)
        print(m, "ok" if ok else f"DIFF max {np.abs(e[m]-s.eta).max()}", end="; ")
    print()


if __name__ == "__main__":
    main()
