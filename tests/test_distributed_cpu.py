"""The N>1 decomposition on CPU with torch.distributed/gloo, world_size 2.

Each rank owns a contiguous slice of particles (global ids keep the RNG streams
independent of the partition, rng.hpp:35-40), runs stages 1-3, all-gathers the (c_i,
zeta_i) pairs -- the only collective of the path, as bench.py does over NCCL -- and runs
stages 4-6 on its slice. The gathered result must equal a single-process analysis
bit-for-bit ("identical for 1 worker and W workers").
"""
import os
import socket
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(oracle):
    from checkers import make_params
    p = make_params(nx=100, ny=60)
    n = 6
    e = np.empty((n, p.ny, p.nx), np.float32)
    u, v = np.empty_like(e), np.empty_like(e)
    for m in range(n):
        s = oracle.init_double_jet(p)
        for d in range(2):
            oracle.perturb_philox(p, s, 77 + m, d)
        e[m], u[m], v[m] = s.eta, s.hu, s.hv
    rng = np.random.default_rng(8)
    obs = np.hstack([rng.uniform(0, 1, (5, 2)) * [p.nx * p.dx, p.ny * p.dy],
                     rng.normal(0, 15, (5, 2))])
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    return p, n, e, u, v, obs, S, usig


def _worker(rank, world, port, outdir):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import torch.distributed as dist
    from checkers import Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = Oracle()
    p, n, e, u, v, obs, S, usig = _problem(oracle)
    per = n // world
    lo, hi = rank * per, (rank + 1) * per
    # stages 1-3 on a copy: this slice's (c, zeta) (n_total > slice, no barrier inputs)
    ce, cu, cv = e[lo:hi].copy(), u[lo:hi].copy(), v[lo:hi].copy()
    diag, _ = oracle.iewpf_assimilate(p, ce, cu, cv, obs, S, usig, 2, member_base=lo, n_total=n)
    cz = torch.tensor(diag[:, [0, 3]], dtype=torch.float64)
    gathered = [torch.zeros_like(cz) for _ in range(world)]
    dist.all_gather(gathered, cz)
    cz_all = torch.cat(gathered).numpy()
    se, su, sv = e[lo:hi].copy(), u[lo:hi].copy(), v[lo:hi].copy()
    oracle.iewpf_assimilate(p, se, su, sv, obs, S, usig, 2, member_base=lo, n_total=n,
                            c_all=cz_all[:, 0].copy(), zeta_all=cz_all[:, 1].copy())
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), e=se, u=su, v=sv)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_analysis_equals_single_process(oracle, tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    p, n, e, u, v, obs, S, usig = _problem(oracle)
    oracle.iewpf_assimilate(p, e, u, v, obs, S, usig, 2)
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    assert np.array_equal(np.concatenate([q["e"] for q in parts]), e)
    assert np.array_equal(np.concatenate([q["u"] for q in parts]), u)
    assert np.array_equal(np.concatenate([q["v"] for q in parts]), v)
