"""GPU parity at the exact BASELINE.json configurations, with the operator the product
ships (the library's eigh U Sigma^1/2 factor), and the pull / posterior compositions
pinned to the reference's OWN operators (oracle/_ref: apply_q_half_T and add_q_half,
stochastic.hpp:144-160,193-202) rather than to this repo's restatement:

  configs[0]  500x300, 10 members, 60 model steps: states and per-step substep counts vs
              the reference's Stepper (ref.model_step_dts)
  configs[2]  500x300, 240 moorings on the 20x12 lattice (25 cells apart: the 7x7 local
              blocks chain through every observation) + 64-drifter copies per member
  configs[4]  1000x600 (dx = 1110 m), 4 members, 2 DA cycles, moorings + drifter copies
  pull        per observation in ascending id: ref.apply_q_half_T(S d) -> ref.add_q_half
  posterior   z = beta^1/2 nu + alpha^1/2 xi, 7x7 U Sigma^1/2 blocks in id order, then
              ref.add_q_half on the filter offsets
  comm        dc_comm_attach at world size 1 (the NCCL path) == the single context
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from checkers import State, make_params

pytestmark = pytest.mark.gpu


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1910_01031_b200 as pkg
    return pkg


def lattice(p, nxp, nyp):
    lx, ly = p.nx * p.dx, p.ny * p.dy
    X, Y = np.meshgrid((np.arange(nxp) + 0.5) / nxp * lx, (np.arange(nyp) + 0.5) / nyp * ly)
    return np.stack([X.ravel(), Y.ravel()], 1)


def spread_states(oracle, p, n, seed):
    e = np.empty((n, p.ny, p.nx), np.float32)
    u, v = np.empty_like(e), np.empty_like(e)
    for m in range(n):
        s = oracle.init_double_jet(p)
        for d in range(3):
            oracle.perturb_philox(p, s, 1000 + m + 37 * seed, d)
        e[m], u[m], v[m] = s.eta, s.hu, s.hv
    return e, u, v


def oracle_forecast(oracle, p, e, u, v, pos, cycle, t0):
    """5 model steps with drifters + Philox model error, every member on its own thread
    (the checker's ctypes calls release the GIL)."""
    def one(m):
        s = State(e[m], u[m], v[m], t0)
        for i in range(5):
            if pos is not None:
                oracle.advect_drifters(p, s, pos[m], 60.0)
            oracle.model_step(p, s, 1)
            if i < 4:
                oracle.perturb_philox(p, s, m, 4 * cycle + i)
    with ThreadPoolExecutor(max_workers=len(e)) as ex:
        list(ex.map(one, range(len(e))))


@pytest.mark.timeout(900)
def test_configs0_forecast_60_steps_vs_reference(ref):
    """configs[0]: 10 members x 60 model steps at 500x300 on the GPU against the
    reference's own Stepper (oracle/_ref): per-step substep counts (the dt sequence of
    every member) and the states after steps 1, 10 and 60, bitwise."""
    pkg = _gpu()
    cfg = pkg.Config(nx=500, ny=300)
    p = make_params(nx=500, ny=300)
    n = 10
    base = ref.init_double_jet(p)
    e = np.empty((n, p.ny, p.nx), np.float32)
    u, v = np.empty_like(e), np.empty_like(e)
    for m in range(n):  # distinct members: the jet plus reference model-error draws
        s = State(base.eta.copy(), base.hu.copy(), base.hv.copy(), 0.0)
        ref.perturb(p, s, 1, 1, m, n_draws=2)
        e[m], u[m], v[m] = s.eta, s.hu, s.hv
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    gsubs, gstates = [], {}
    for step in range(1, 61):
        ens.model_step(1)
        gsubs.append(ens.substeps().copy())
        if step in (1, 10, 60):
            gstates[step] = ens.download()
    ens.close()

    def run(m):
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        counts, snaps = [], {}
        for step in range(1, 61):
            counts.append(len(ref.model_step_dts(p, s)))
            if step in (1, 10, 60):
                snaps[step] = (s.eta.copy(), s.hu.copy(), s.hv.copy(), s.t)
        return counts, snaps
    with ThreadPoolExecutor(max_workers=n) as ex:
        res = list(ex.map(run, range(n)))
    for m, (counts, snaps) in enumerate(res):
        assert [int(g[m]) for g in gsubs] == counts, m
        for step, (se, su, sv, st) in snaps.items():
            ge, gu, gv, gt = gstates[step]
            assert np.array_equal(ge[m], se), (m, step, np.abs(ge[m] - se).max())
            assert np.array_equal(gu[m], su) and np.array_equal(gv[m], sv), (m, step)
            assert gt[m] == st == 60.0 * step


def _pull_by_reference(ref, p, st, obs, S):
    """optimal_proposal_pull composed from the reference's operators:
    all innovations first, then per observation in ascending id apply_q_half_T(S d) on the
    aligned coarse grid and add_q_half into the float state. Returns phi."""
    H = p.h_eq
    cells = [ref.locate_cell(p, o[0], o[1]) for o in obs]
    ds = []
    for (j, k), o in zip(cells, obs):
        h = H + np.float64(st.eta[k, j])
        ds.append((o[2] * h / H - np.float64(st.hu[k, j]), o[3] * h / H - np.float64(st.hv[k, j])))
    phi = 0.0
    for (j, k), (d0, d1) in zip(cells, ds):
        sd0 = S[0, 0] * d0 + S[0, 1] * d1
        sd1 = S[1, 0] * d0 + S[1, 1] * d1
        phi += d0 * sd0 + d1 * sd1
        coarse, (oj, ok) = ref.apply_q_half_T(p, sd0, sd1, j, k, align=True)
        ref.add_q_half(p, st, oj, ok, coarse, 1.0)
    return phi


def _posterior_by_reference(ref, oracle, p, st, obs, usig, member, cycle, alpha, beta):
    """apply_P_half + the final update: z = beta^1/2 nu +
    alpha^1/2 xi on the filter stream's draw, 7x7 blocks <- U Sigma^1/2 block in ascending
    observation id (sequential fp64 sums), then the reference's add_q_half on the filter
    offsets."""
    xi, nu, _, _, (oj, ok) = oracle.perp_pair(p, member, cycle)
    c = p.c_omega
    nxc, nyc = p.nx // c, p.ny // c
    sqa, sqb = float(np.sqrt(alpha)), float(np.sqrt(beta))
    z = [sqb * float(a) + sqa * float(b) for a, b in zip(nu, xi)]
    U = usig.reshape(49, 49).tolist()

    def nearest(jj, o, n):
        v = jj - o + (c - 1) // 2
        q = v // c if v >= 0 else -((-v + c - 1) // c)
        return q % n
    for o in obs:
        j, k = ref.locate_cell(p, o[0], o[1])
        a0, b0 = nearest(j, oj, nxc), nearest(k, ok, nyc)
        idx = [((b0 + r // 7 - 3) % nyc) * nxc + (a0 + r % 7 - 3) % nxc for r in range(49)]
        bin_ = [z[i] for i in idx]
        out = []
        for r in range(49):
            s = 0.0
            row = U[r]
            for q in range(49):
                s += row[q] * bin_[q]
            out.append(s)
        for r in range(49):
            z[idx[r]] = out[r]
    ref.add_q_half(p, st, oj, ok, np.array(z), 1.0)


@pytest.mark.parametrize("nx,ny,n_obs", [(100, 60, 6), (500, 300, 12)])
def test_pull_and_posterior_pinned_to_reference_operators(ref, oracle, nx, ny, n_obs):
    """The GPU analysis against the reference's own apply_q_half_T / add_q_half composed
    per observation in ascending id: the state after the pulls (dc_iewpf_begin), phi, and
    the posterior after dc_iewpf_finish, with the library's eigh U Sigma^1/2 factor."""
    pkg = _gpu()
    cfg = pkg.Config(nx=nx, ny=ny)
    p = make_params(nx=nx, ny=ny)
    n = 3
    e, u, v = spread_states(oracle, p, n, 5)
    rng = np.random.default_rng(nx + n_obs)
    xy = rng.uniform(0, 1, (n_obs, 2)) * [p.nx * p.dx, p.ny * p.dy]
    xy[1] = xy[0] + [2 * p.dx, 3 * p.dy]  # overlapping footprints
    obs = np.hstack([xy, rng.normal(0, 20.0, (n_obs, 2))])
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    cz = ens.iewpf_begin(obs, S, usig, 2, n_total=n)
    pe, pu, pv, _ = ens.download()
    ens.iewpf_finish(cz)
    fe, fu, fv, _ = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    ens.close()
    for m in range(n):
        st = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        phi = _pull_by_reference(ref, p, st, obs, S)
        assert phi == diag[m, 1], (m, phi, diag[m, 1])
        # == (not bitwise): an untouched cell may hold -0.0 on one side
        assert np.array_equal(pe[m], st.eta) and np.array_equal(pu[m], st.hu)
        assert np.array_equal(pv[m], st.hv), m
        _posterior_by_reference(ref, oracle, p, st, obs, usig, m, 2, diag[m, 4], wb[1])
        assert np.array_equal(fe[m], st.eta), (m, np.abs(fe[m] - st.eta).max())
        assert np.array_equal(fu[m], st.hu) and np.array_equal(fv[m], st.hv), m


def _da_vs_oracle(pkg, oracle, cfg, p, n, obs_list, with_drifters, seed):
    e, u, v = spread_states(oracle, p, n, seed)
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)  # the factor the product ships
    pos = np.repeat(lattice(p, 8, 8)[None], n, 0).copy() if with_drifters else None
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    if with_drifters:
        ens.drifters_set(pos)
    for c, obs in enumerate(obs_list):
        ens.da_cycle(5, obs, S, usig, cycle=c)
    ge, gu, gv, gt = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    gp = ens.drifters_get()[0] if with_drifters else None
    ens.close()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    op = pos.copy() if with_drifters else None
    for c, obs in enumerate(obs_list):
        oracle_forecast(oracle, p, oe, ou, ov, op, c, 300.0 * c)
        od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, c)
    assert np.array_equal(wb, owb) and np.array_equal(diag, od)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
    if with_drifters:
        assert np.array_equal(gp, op)
    assert np.all(gt == 300.0 * len(obs_list))


@pytest.mark.timeout(900)
def test_configs2_moorings_500x300_bitwise(oracle):
    """configs[2] exactly: 500x300, 240 moorings on the 20x12 lattice (25 cells apart, so
    the 7x7 local blocks overlap along the whole id chain), 64 drifter copies in every
    member, 2 DA cycles, the library's eigh factor: bitwise vs the oracle."""
    pkg = _gpu()
    cfg = pkg.Config(nx=500, ny=300)
    p = make_params(nx=500, ny=300)
    moor = lattice(p, 20, 12)
    rng = np.random.default_rng(61)
    obs = [np.hstack([moor, rng.normal(0, 20.0, (240, 2))]) for _ in range(2)]
    _da_vs_oracle(pkg, oracle, cfg, p, 3, obs, True, 63)


@pytest.mark.timeout(1200)
def test_configs4_refined_grid_two_cycles_bitwise(oracle):
    """configs[4] geometry at ensemble scale: 1000x600 (dx = dy = 1110 m), 4 members, 2
    DA cycles with 240 moorings and 64 drifter copies per member, eigh factor: state,
    drifters and diagnostics bitwise vs the oracle."""
    pkg = _gpu()
    cfg = pkg.Config(nx=1000, ny=600, dx=1110.0, dy=1110.0)
    p = make_params(nx=1000, ny=600, dx=1110.0, dy=1110.0)
    moor = lattice(p, 20, 12)
    rng = np.random.default_rng(71)
    obs = [np.hstack([moor, rng.normal(0, 20.0, (240, 2))]) for _ in range(2)]
    _da_vs_oracle(pkg, oracle, cfg, p, 4, obs, True, 73)


def test_configs1_drifters_eigh_bitwise(oracle):
    """configs[1]: 500x300, 64 drifter observations on the 8x8 lattice, drifter copies,
    the library's eigh factor, 2 cycles: bitwise vs the oracle."""
    pkg = _gpu()
    cfg = pkg.Config(nx=500, ny=300)
    p = make_params(nx=500, ny=300)
    rng = np.random.default_rng(81)
    obs = [np.hstack([lattice(p, 8, 8) + 150.0 * (c + 1), rng.normal(0, 20.0, (64, 2))])
           for c in range(2)]
    _da_vs_oracle(pkg, oracle, cfg, p, 3, obs, True, 83)


def test_comm_world1_equals_single_context(oracle):
    """The multi-GPU path of the library (dc_comm_attach: NCCL send/recv of the (c, zeta)
    pairs at the barrier, drifter gather to rank 0 for the forecast statistics) at world
    size 1 gives the single context's bits: states, diagnostics and E/RMSE."""
    pkg = _gpu()
    cfg = pkg.Config(nx=100, ny=60)
    p = make_params(nx=100, ny=60)
    n = 4
    e, u, v = spread_states(oracle, p, n, 91)
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    pos = np.random.default_rng(5).uniform(0, 1, size=(n, 5, 2)) * [p.nx * p.dx, p.ny * p.dy]
    rng = np.random.default_rng(93)
    obs = [np.hstack([rng.uniform(0, 1, (5, 2)) * [p.nx * p.dx, p.ny * p.dy],
                      rng.normal(0, 20.0, (5, 2))]) for _ in range(3)]
    truth = [pos[0] + 50.0 * c for c in range(3)]
    outs = []
    for use_comm in (False, True):
        ens = pkg.Ensemble(cfg, n)
        if use_comm:
            ens.comm_attach(pkg.comm_unique_id(), 0, 1, n)
            assert ens.comm_info() == (0, 1, n)
        ens.upload(e, u, v, 0.0)
        ens.drifters_set(pos)
        res = []
        for c in range(3):
            ens.da_cycle(5, obs[c], S, usig, cycle=c)
            ens.readback_enqueue(0, truth_xy=truth[c])
            r = ens.readback_wait(0)
            res.append((r["diag"], r["w_beta"], r["E"], r["RMSE"]))
        res.append(ens.forecast_error(truth[2])[:2])
        outs.append((ens.download(), res))
        ens.close()
    (a, ra), (b, rb) = outs
    for f in range(4):
        assert np.array_equal(a[f], b[f])
    for x, y in zip(ra[:3], rb[:3]):
        assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])
        assert x[2] == y[2] and x[3] == y[3]
    assert ra[3] == rb[3]


def test_guard_banded_run_is_clean_and_bitwise():
    """The memory checker (DC_GUARD=1, csrc/guard.cu): two DA cycles with drifters and
    forecast statistics in a process whose every device buffer has 64 KB guard bands and
    0xFF-poisoned contents. No guard band may change (no out-of-bounds write anywhere on
    the path), and the results must equal an unguarded run bit for bit (no kernel reads
    uninitialised or out-of-bounds memory into a result)."""
    import json
    import os
    import subprocess
    import sys
    _gpu()
    code = r'''
import json, sys, ctypes as C
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1910_01031_b200 as pkg
from paper_1910_01031_b200 import _lib
cfg = pkg.Config(nx=100, ny=60)
_, S = pkg.precompute_S(cfg)
_, usig = pkg.precompute_local_svd(cfg, S)
ens = pkg.Ensemble(cfg, 3)
ens.init_double_jet()
pos = np.random.default_rng(1).uniform(0, 1, (3, 4, 2)) * [100 * 2220.0, 60 * 2220.0]
ens.drifters_set(pos)
rng = np.random.default_rng(2)
out = []
for c in range(2):
    obs = np.hstack([rng.uniform(0, 1, (5, 2)) * [100 * 2220.0, 60 * 2220.0], rng.normal(0, 20, (5, 2))])
    ens.da_cycle(5, obs, S, usig, c)
    ens.readback_enqueue(0, truth_xy=pos[0])
    r = ens.readback_wait(0)
    out.append([float(r["E"]), float(r["RMSE"])] + r["diag"][:, 4].tolist())
e, u, v, t = ens.download()
out.append([float(np.float64(e.sum())), float(np.float64(u.sum())), float(np.float64(v.sum()))])
msg = C.create_string_buffer(4096); n = C.c_int32()
_lib.load().dc_check_guards(msg, 4096, C.byref(n))
ens.close()
print(json.dumps({"bad": n.value, "msg": msg.value.decode(), "out": out}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for guard in ("0", "1"):
        env = dict(os.environ, DC_GUARD=guard)
        r = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res[guard] = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["1"]["bad"] == 0, res["1"]["msg"]
    assert res["1"]["out"] == res["0"]["out"]
