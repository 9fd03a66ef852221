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


# ---- resampling across ranks (paper_1910_01031_b200/resample.py) ----
def test_exchange_plan_routes_every_slot():
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1910_01031_b200.resample import exchange_plan
    per, world = 4, 3
    rng = np.random.default_rng(4)
    for _ in range(20):
        idx = np.sort(rng.integers(0, per * world, per * world))
        sent = {}
        for r in range(world):
            _, sends, _ = exchange_plan(idx, per, r)
            for dest, src in sends:
                sent.setdefault(dest, set()).add((r, src))
        for r in range(world):
            local, _, recvs = exchange_plan(idx, per, r)
            got = {}
            for sr, sl, slots in recvs:
                assert (sr, sl) in sent.get(r, set())
                for i in slots:
                    got[i] = sr * per + sl
            for i in range(per):
                g = r * per + i
                assert got.get(i, r * per + local[i]) == idx[g]
            # nothing is sent to r that r does not receive
            assert sent.get(r, set()) == {(sr, sl) for sr, sl, _ in recvs}


def _resample_worker(rank, world, port, idx, per, outdir):
    sys.path.insert(0, os.path.dirname(HERE))
    import torch
    import torch.distributed as dist
    from paper_1910_01031_b200.resample import exchange, exchange_plan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # stand-in members: 8-float rows carrying the global member id
    state = torch.arange(rank * per, (rank + 1) * per, dtype=torch.float32)[:, None].repeat(1, 8)

    def gather(li):
        state.copy_(state[torch.tensor(li)])

    exchange(exchange_plan(idx, per, rank), 8, lambda nb: torch.empty(nb),
             lambda m, b: b.copy_(state[m]), gather, lambda m, b: state[m].copy_(b), dist)
    np.save(os.path.join(outdir, f"r{rank}.npy"), state.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_resample_exchange(tmp_path):
    """Host logic of the cross-rank resampling on CPU: every slot ends up holding the
    member the global index names (ids carried by stand-in member buffers)."""
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    world, per = 2, 5
    idx = np.array([0, 0, 3, 6, 6, 6, 7, 9, 9, 9])  # both directions, duplicates, keeps
    mp.spawn(_resample_worker, args=(world, _free_port(), idx, per, str(tmp_path)),
             nprocs=world, join=True)
    got = np.concatenate([np.load(os.path.join(tmp_path, f"r{r}.npy")) for r in range(world)])
    assert np.array_equal(got[:, 0], idx) and np.all(got == got[:, :1])
