"""GPU parity of the observation system and the two-stage IEWPF analysis (C ABI vs the
CPU restatement in oracle/). These rows have no reference code;
the restatement follows SPEC.md/PAPER.md with the spec gaps decided in DESIGN.md §5, and
the GPU must match it BITWISE: the per-observation pull is a gather that reproduces the
sequential add_q_half roundings, the dot products use the restated fixed reduction order
and alpha uses the deterministic exp/log both sides implement.
"""
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


def setup(nx=100, ny=60, n=6, seed=0, **kw):
    pkg = _gpu()
    cfg = pkg.Config(nx=nx, ny=ny, **kw)
    p = make_params(nx=nx, ny=ny, q0=cfg.q0, seed=cfg.seed, c_omega=cfg.c_omega)
    return pkg, cfg, p


def spread_states(oracle, p, n, seed):
    """Double jet + Philox model error: n distinct members (via the oracle)."""
    e = np.empty((n, p.ny, p.nx), np.float32)
    u, v = np.empty_like(e), np.empty_like(e)
    for m in range(n):
        s = oracle.init_double_jet(p)
        for d in range(3):
            oracle.perturb_philox(p, s, 1000 + m + 37 * seed, d)
        e[m], u[m], v[m] = s.eta, s.hu, s.hv
    return e, u, v


def obs_set(p, n_obs, seed):
    rng = np.random.default_rng(seed)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    xy = rng.uniform(0, 1, size=(n_obs, 2)) * [lx, ly]
    xy[0] = [0.3 * p.dx, (p.ny - 0.5) * p.dy]          # near the periodic corner
    if n_obs > 2:
        xy[1] = xy[2] + [3 * p.dx, -2 * p.dy]           # overlapping footprints
    yv = rng.normal(0, 20.0, size=(n_obs, 2))
    return np.hstack([xy, yv])


def test_precompute_S_and_block(oracle):
    pkg, cfg, p = setup(500, 300)
    h, S = pkg.precompute_S(cfg)
    ho, So = oracle.precompute_S(p, 0, 0)
    assert np.array_equal(h, ho) and np.array_equal(S, So)
    # SURVEY.md §8a a20 probe: S = 0.881140 I at 500x300 (position independent)
    assert abs(S[0, 0] - 0.881140) < 5e-6 and abs(S[1, 1] - 0.881140) < 5e-6
    assert abs(S[0, 1]) < 1e-12
    blk, usig = pkg.precompute_local_svd(cfg, S)
    assert np.array_equal(blk, oracle.local_block(p, S))
    assert np.abs(usig @ usig.T - blk).max() < 1e-12
    # structure: 45 non-identity rows before corner inclusion -- the
    # structural pattern is the 7x7 block minus its corners; numerically the centre
    # row is exactly the identity row (the SOAR'd dipole vanishes at its own centre by
    # symmetry), so 44 rows differ from I and all lie in the pattern.
    corners = {0, 6, 42, 48}
    pattern = [r for r in range(49) if r not in corners]
    assert len(pattern) == 45
    nonid = [r for r in range(49) if np.any(blk[r] != np.eye(49)[r])]
    assert set(nonid) == set(pattern) - {24}
    assert np.array_equal(blk[24], np.eye(49)[24])


def test_innovations_bitwise(oracle):
    pkg, cfg, p = setup()
    n = 4
    e, u, v = spread_states(oracle, p, n, 1)
    obs = obs_set(p, 9, 2)
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    d = ens.innovations(obs)
    for m in range(n):
        do = oracle.innovations(p, State(e[m], u[m], v[m]), obs)
        assert np.array_equal(d[m], do)


def test_drifters_bitwise(oracle):
    pkg, cfg, p = setup()
    n, nd = 3, 17
    e, u, v = spread_states(oracle, p, n, 3)
    u += 40.0  # strong eastward transport so drifters cross the periodic edge
    rng = np.random.default_rng(5)
    pos = rng.uniform(0, 1, size=(n, nd, 2)) * [p.nx * p.dx, p.ny * p.dy]
    pos[:, 0] = [p.nx * p.dx - 1.0, 10.0]
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.drifters_set(pos)
    for _ in range(7):
        ens.advect_drifters(60.0)
    gp, gw = ens.drifters_get()
    for m in range(n):
        q = pos[m].copy()
        w = np.zeros((nd, 2), np.int32)
        s = State(e[m], u[m], v[m])
        for _ in range(7):
            oracle.advect_drifters(p, s, q, 60.0, w)
        assert np.array_equal(gp[m], q)
        assert np.array_equal(gw[m], w)
    assert gw[:, 0, 0].min() >= 1  # the edge drifter wrapped


@pytest.mark.parametrize("nx,ny,n,n_obs", [(100, 60, 6, 7), (500, 300, 4, 24)])
def test_iewpf_assimilate_bitwise(oracle, nx, ny, n, n_obs):
    pkg, cfg, p = setup(nx, ny)
    e, u, v = spread_states(oracle, p, n, 7)
    obs = obs_set(p, n_obs, 11)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S) + 0.0 * np.eye(49))
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.iewpf_assimilate(obs, S, usig, cycle=3)
    ge, gu, gv, _ = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 3)
    assert np.array_equal(wb, owb), (wb, owb)
    assert np.array_equal(diag, od), np.abs(diag - od).max(axis=0)
    for m in range(n):
        assert np.array_equal(ge[m], oe[m]), (m, np.abs(ge[m] - oe[m]).max())
        assert np.array_equal(gu[m], ou[m])
        assert np.array_equal(gv[m], ov[m])
    assert np.all((diag[:, 4] > 0) & (diag[:, 4] <= 1.0 + 1e-12))


def test_iewpf_edge_observations_bitwise(oracle):
    """Observations on the domain edges (x = 0, y = 0, just below Lx / Ly), exactly on
    cell faces and coarse-cell corners, and two observations at the same point: cell
    location, window alignment across the periodic seam and the sequential pulls all
    match the oracle bit for bit."""
    pkg, cfg, p = setup(100, 60)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    rng = np.random.default_rng(17)
    xy = np.array([[0.0, 0.0], [np.nextafter(lx, 0.0), 3.0 * p.dy],
                   [7.0 * p.dx, np.nextafter(ly, 0.0)], [5.0 * p.c_omega * p.dx, 10.0 * p.c_omega * p.dy],
                   [40.0 * p.dx, 20.0 * p.dy], [40.0 * p.dx, 20.0 * p.dy],
                   [0.5 * lx, 0.5 * ly]])
    obs = np.hstack([xy, rng.normal(0, 20.0, (len(xy), 2))])
    n = 4
    e, u, v = spread_states(oracle, p, n, 13)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.iewpf_assimilate(obs, S, usig, cycle=5)
    ge, gu, gv, _ = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    ens.close()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 5)
    assert np.array_equal(wb, owb) and np.array_equal(diag, od)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)


def test_iewpf_two_slices_equal_one(oracle):
    """The multi-GPU decomposition on one device: two contexts own members [0,3) and
    [3,6); stages 1-3 run per slice, the (c, zeta) pairs are concatenated (the NCCL
    all-gather), stages 4-6 run per slice. Result == single-context run, bitwise."""
    pkg, cfg, p = setup()
    n = 6
    e, u, v = spread_states(oracle, p, n, 9)
    obs = obs_set(p, 5, 13)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    one = pkg.Ensemble(cfg, n)
    one.upload(e, u, v, 0.0)
    one.iewpf_assimilate(obs, S, usig, cycle=1)
    ref = one.download()
    a = pkg.Ensemble(cfg, 3, member_base=0)
    b = pkg.Ensemble(cfg, 3, member_base=3)
    a.upload(e[:3], u[:3], v[:3], 0.0)
    b.upload(e[3:], u[3:], v[3:], 0.0)
    cza = a.iewpf_begin(obs, S, usig, 1, n_total=n)
    czb = b.iewpf_begin(obs, S, usig, 1, n_total=n)
    cz = np.concatenate([cza, czb])
    a.iewpf_finish(cz)
    b.iewpf_finish(cz)
    ra, rb = a.download(), b.download()
    for f in range(3):
        assert np.array_equal(np.concatenate([ra[f], rb[f]]), ref[f])


def test_da_cycle_matches_oracle(oracle):
    """One DA cycle: 5 model steps, Philox model error after the first
    4, drifters advected each step, then the analysis -- bitwise vs the oracle."""
    pkg, cfg, p = setup()
    n = 4
    e, u, v = spread_states(oracle, p, n, 15)
    obs = obs_set(p, 6, 17)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    pos = np.random.default_rng(3).uniform(0, 1, size=(n, 5, 2)) * [p.nx * p.dx, p.ny * p.dy]
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.drifters_set(pos)
    ens.da_cycle(5, obs, S, usig, cycle=0)
    ge, gu, gv, gt = ens.download()
    gp, _ = ens.drifters_get()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    op = pos.copy()
    for m in range(n):
        s = State(oe[m], ou[m], ov[m], 0.0)
        for i in range(5):
            oracle.advect_drifters(p, s, op[m], 60.0)
            oracle.model_step(p, s, 1)
            if i < 4:
                oracle.perturb_philox(p, s, m, i)
    oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 0)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
    assert np.array_equal(gp, op)
    assert np.all(gt == 300.0)


def test_iewpf_dense_platforms_bitwise(oracle):
    """A dense mooring-like lattice (blocks overlap across many dependency levels, several
    observations per level): the level-scheduled local blocks and the gathered pulls equal
    the sequential ascending-id restatement bit for bit."""
    pkg, cfg, p = setup(200, 120)
    n = 3
    e, u, v = spread_states(oracle, p, n, 9)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    X, Y = np.meshgrid((np.arange(12) + 0.5) / 12 * lx, (np.arange(7) + 0.5) / 7 * ly)
    rng = np.random.default_rng(21)
    obs = np.hstack([np.stack([X.ravel(), Y.ravel()], 1), rng.normal(0, 20.0, (84, 2))])
    obs = obs[rng.permutation(84)]  # ids not in lattice order
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.iewpf_assimilate(obs, S, usig, cycle=1)
    ge, gu, gv, _ = ens.download()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 1)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)


def test_one_stage_iewpf_bitwise(oracle):
    """the one-stage variant (target max c_i, alpha^1/2 P^1/2 xi) equals the
    restatement bit for bit."""
    pkg, cfg, p = setup()
    n = 5
    e, u, v = spread_states(oracle, p, n, 13)
    obs = obs_set(p, 6, 19)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.iewpf_set_mode(True)
    ens.iewpf_assimilate(obs, S, usig, cycle=2)
    ge, gu, gv, _ = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    oracle.lib.orc_iewpf_set_mode(1)
    try:
        od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 2)
    finally:
        oracle.lib.orc_iewpf_set_mode(0)
    assert np.array_equal(wb, owb) and wb[0] == diag[:, 0].max() and wb[1] == 0.0
    assert np.array_equal(diag, od)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)


def test_da_cycle_full_size_bitwise(oracle):
    """One DA cycle at the bench size (500x300, 64 drifters on the bench lattice, drifter
    copies in every member) for 3 members: state, drifters and diagnostics bitwise equal
    to the oracle."""
    pkg, cfg, p = setup(500, 300)
    n = 3
    e, u, v = spread_states(oracle, p, n, 23)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    X, Y = np.meshgrid((np.arange(8) + 0.5) / 8 * lx, (np.arange(8) + 0.5) / 8 * ly)
    lat = np.stack([X.ravel(), Y.ravel()], 1)
    obs = np.hstack([lat + 1234.5, np.random.default_rng(29).normal(0, 20.0, (64, 2))])
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    pos = np.repeat(lat[None], n, 0).copy()
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.drifters_set(pos)
    ens.da_cycle(5, obs, S, usig, cycle=4)
    ge, gu, gv, gt = ens.download()
    gp, _ = ens.drifters_get()
    diag, wb = ens.iewpf_diagnostics()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    op = pos.copy()
    for m in range(n):
        s = State(oe[m], ou[m], ov[m], 0.0)
        for i in range(5):
            oracle.advect_drifters(p, s, op[m], 60.0)
            oracle.model_step(p, s, 1)
            if i < 4:
                oracle.perturb_philox(p, s, m, i)
    od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 4)
    assert np.array_equal(wb, owb) and np.array_equal(diag, od)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
    assert np.array_equal(gp, op) and np.all(gt == 300.0)


@pytest.mark.parametrize("nx,ny,c", [(60, 60, 3), (110, 55, 5), (64, 48, 1), (125, 75, 5)])
def test_da_cycle_configs_bitwise(oracle, nx, ny, c):
    """DA cycles on other grids and coarsening factors (odd sizes, non-square, c_omega 1/3/5):
    bitwise vs the oracle, two cycles so the second starts from an analysed state."""
    pkg = _gpu()
    cfg = pkg.Config(nx=nx, ny=ny, c_omega=c)
    p = make_params(nx=nx, ny=ny, q0=cfg.q0, seed=cfg.seed, c_omega=c)
    n = 3
    e, u, v = spread_states(oracle, p, n, 31)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    rng = np.random.default_rng(nx + ny + c)
    obs = [np.hstack([rng.uniform(0, 1, (5, 2)) * [p.nx * p.dx, p.ny * p.dy],
                      rng.normal(0, 20.0, (5, 2))]) for _ in range(2)]
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    for cyc in range(2):
        ens.da_cycle(5, obs[cyc], S, usig, cycle=cyc)
    ge, gu, gv, _ = ens.download()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    for cyc in range(2):
        for m in range(n):
            s = State(oe[m], ou[m], ov[m], 0.0)
            for i in range(5):
                oracle.model_step(p, s, 1)
                if i < 4:
                    oracle.perturb_philox(p, s, m, 4 * cyc + i)
        oracle.iewpf_assimilate(p, oe, ou, ov, obs[cyc], S, usig, cyc)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)


def test_twenty_cycles_bitwise(oracle):
    """A long horizon: 20 DA cycles (100 model steps, 80 model-error draws, 20 analyses)
    stay bitwise equal to the oracle -- no drift accumulates anywhere on the path."""
    pkg, cfg, p = setup()
    n = 3
    e, u, v = spread_states(oracle, p, n, 41)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    rng = np.random.default_rng(43)
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    for cyc in range(20):
        obs = np.hstack([rng.uniform(0, 1, (4, 2)) * [p.nx * p.dx, p.ny * p.dy],
                         rng.normal(0, 20.0, (4, 2))])
        ens.da_cycle(5, obs, S, usig, cycle=cyc)
        for m in range(n):
            s = State(oe[m], ou[m], ov[m], 0.0)
            for i in range(5):
                oracle.model_step(p, s, 1)
                if i < 4:
                    oracle.perturb_philox(p, s, m, 4 * cyc + i)
        oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, cyc)
    ge, gu, gv, gt = ens.download()
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
    assert np.all(gt == 20 * 300.0)


def test_pipelined_readback_equals_synchronous_reads(oracle):
    """dc_readback_enqueue / dc_readback_wait (two pinned slots, cycle c read while
    cycle c+1 runs) return the same bits as the synchronous diagnostics, drifter and
    forecast-error reads of an identical ensemble."""
    pkg, cfg, p = setup()
    n = 4
    e, u, v = spread_states(oracle, p, n, 21)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    pos = np.random.default_rng(5).uniform(0, 1, size=(n, 5, 2)) * [p.nx * p.dx, p.ny * p.dy]
    obs = [obs_set(p, 6, 40 + c) for c in range(5)]
    truth = [pos[0] + c * 100.0 for c in range(5)]
    a, b = pkg.Ensemble(cfg, n), pkg.Ensemble(cfg, n)
    for ens in (a, b):
        ens.upload(e, u, v, 0.0)
        ens.drifters_set(pos)
    sync_out, pipe_out = [], []
    for c in range(5):
        a.da_cycle(5, obs[c], S, usig, cycle=c)
        d, wb = a.iewpf_diagnostics()
        gp, gw = a.drifters_get()
        E, R, _, _ = a.forecast_error(truth[c])
        sync_out.append((d, wb, gp, gw, E, R))
        b.da_cycle(5, obs[c], S, usig, cycle=c)
        b.readback_enqueue(c % 2, truth_xy=truth[c])
        if c > 0:
            pipe_out.append(b.readback_wait((c - 1) % 2))
    pipe_out.append(b.readback_wait(4 % 2))
    for (d, wb, gp, gw, E, R), r in zip(sync_out, pipe_out):
        assert np.array_equal(d, r["diag"]) and np.array_equal(wb, r["w_beta"])
        assert np.array_equal(gp, r["pos"]) and np.array_equal(gw, r["wind"])
        assert E == r["E"] and R == r["RMSE"]
    with pytest.raises(pkg.DcError):
        b.readback_wait(0)  # nothing enqueued


@pytest.mark.timeout(600)
def test_da_cycle_refined_grid_moorings_bitwise(oracle):
    """configs[4] geometry: the 4x refined grid (1000x600, dx = dy = 1110 m, 13 substeps
    per model step, N_R = 24,000) with 240 moorings on a 20x12 lattice: one DA cycle for 2
    members, state and diagnostics bitwise equal to the oracle."""
    pkg = _gpu()
    cfg = pkg.Config(nx=1000, ny=600, dx=1110.0, dy=1110.0)
    p = make_params(nx=1000, ny=600, dx=1110.0, dy=1110.0, q0=cfg.q0, seed=cfg.seed,
                    c_omega=cfg.c_omega)
    n = 2
    e, u, v = spread_states(oracle, p, n, 41)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    X, Y = np.meshgrid((np.arange(20) + 0.5) / 20 * lx, (np.arange(12) + 0.5) / 12 * ly)
    lat = np.stack([X.ravel(), Y.ravel()], 1)
    obs = np.hstack([lat, np.random.default_rng(43).normal(0, 20.0, (240, 2))])
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.da_cycle(5, obs, S, usig, cycle=2)
    ge, gu, gv, gt = ens.download()
    diag, wb = ens.iewpf_diagnostics()
    subs = ens.substeps()
    oe, ou, ov = e.copy(), u.copy(), v.copy()
    for m in range(n):
        s = State(oe[m], ou[m], ov[m], 0.0)
        for i in range(5):
            oracle.model_step(p, s, 1)
            if i < 4:
                oracle.perturb_philox(p, s, m, i)
    od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 2)
    assert np.all(subs >= 12)  # the refined grid's CFL: 13 substeps per 60 s
    assert np.array_equal(wb, owb) and np.array_equal(diag, od)
    assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
    assert np.all(gt == 300.0)


@pytest.mark.timeout(600)
def test_iewpf_observation_count_edges(oracle):
    """The observation-count range of one analysis: 1 and the maximum 1024 (every tile
    covered by every observation, 1024-deep pull folds) bitwise vs the oracle; 0, 1025
    and a non-finite position rejected with DC_EINVAL before any device work."""
    pkg, cfg, p = setup()
    n = 2
    e, u, v = spread_states(oracle, p, n, 51)
    _, S = oracle.precompute_S(p)
    usig = np.linalg.cholesky(oracle.local_block(p, S))
    for n_obs in (1, 1024):
        obs = obs_set(p, n_obs, 60 + n_obs)
        ens = pkg.Ensemble(cfg, n)
        ens.upload(e, u, v, 0.0)
        ens.iewpf_assimilate(obs, S, usig, cycle=1)
        ge, gu, gv, _ = ens.download()
        diag, wb = ens.iewpf_diagnostics()
        oe, ou, ov = e.copy(), u.copy(), v.copy()
        od, owb = oracle.iewpf_assimilate(p, oe, ou, ov, obs, S, usig, 1)
        assert np.array_equal(wb, owb) and np.array_equal(diag, od), n_obs
        assert np.array_equal(ge, oe) and np.array_equal(gu, ou) and np.array_equal(gv, ov)
        ens.close()
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    bad = [obs_set(p, 1025, 3), np.zeros((0, 4))]
    nan = obs_set(p, 4, 4)
    nan[2, 0] = np.nan
    bad.append(nan)
    for obs in bad:
        with pytest.raises(pkg.DcError) as ei:
            ens.iewpf_assimilate(obs, S, usig, cycle=1)
        assert ei.value.status == 1, ei.value  # DC_EINVAL
    ge, _, _, _ = ens.download()
    assert np.array_equal(ge, e)  # nothing was applied
