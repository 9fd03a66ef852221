"""GPU parity of the forecast path (model operator M + model error) through the C ABI.

The CUDA path is compared with the CPU restatement (oracle/liboracle.so) on the same
inputs. In the exact build (dc_config.exact_fp = 1) every float/double op follows the
reference's evaluation order without contraction, so the bar is BITWISE equality
(np.array_equal on float values: +0 == -0). The FMA build is held to the tolerance the
survey derived from the reference itself under FMA:
max|diff| <= 1e-5 * max|field| over a <= 1-day horizon.
Known answers re-hosted from proj/tests/test_swe.cpp and test_stochastic.cpp.
"""
import numpy as np
import pytest

from checkers import State, make_params

pytestmark = pytest.mark.gpu


def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1910_01031_b200 import Config, Ensemble
    return Config, Ensemble


def cfg_pair(nx=500, ny=300, exact=True, **kw):
    Config, _ = _gpu()
    if "c_omega" not in kw and (nx % 5 or ny % 5):
        kw["c_omega"] = 1
    cfg = Config(nx=nx, ny=ny, exact_fp=exact, **kw)
    p = make_params(nx=nx, ny=ny, q0=cfg.q0, seed=cfg.seed, c_omega=cfg.c_omega,
                    dx=cfg.dx, dy=cfg.dy)
    return cfg, p


def perturbed_jets(oracle, p, n, seed=0, amp_eta=0.02, amp_v=2.0):
    """Double jet plus smooth member-specific perturbations (deterministic)."""
    base = oracle.init_double_jet(p)
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:p.ny, 0:p.nx]
    eta = np.empty((n, p.ny, p.nx), np.float32)
    hu, hv = np.empty_like(eta), np.empty_like(eta)
    for m in range(n):
        kx, ky = rng.integers(1, 4, size=2)
        ph = rng.uniform(0, 2 * np.pi, size=3)
        bump = np.sin(2 * np.pi * kx * x / p.nx + ph[0]) * np.cos(2 * np.pi * ky * y / p.ny + ph[1])
        eta[m] = base.eta + (amp_eta * bump).astype(np.float32)
        hu[m] = base.hu + (amp_v * np.cos(2 * np.pi * ky * y / p.ny + ph[2])).astype(np.float32)
        hv[m] = (amp_v * bump).astype(np.float32)
    return eta, hu, hv


def test_flux_rhs_bitwise(oracle):
    _, Ensemble = _gpu()
    for nx, ny in [(500, 300), (100, 60), (16, 12)]:
        cfg, p = cfg_pair(nx, ny)
        e, u, v = perturbed_jets(oracle, p, 2, seed=nx)
        ens = Ensemble(cfg, 2)
        ens.upload(e, u, v, 0.0)
        for m in range(2):
            g = ens.flux_rhs(m)
            o = oracle.flux_rhs(p, State(e[m].copy(), u[m].copy(), v[m].copy()))
            for a, b in zip(g, o):
                assert np.array_equal(a, b), (nx, ny, m, np.abs(a - b).max())
        ens.close()


def test_lake_at_rest_exact_zero():
    """test_swe.cpp:17-44: zero tendencies, bitwise-preserved rest state, t advanced."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(16, 12)
    ens = Ensemble(cfg, 2)
    z = np.zeros((2, 12, 16), np.float32)
    lifted = z.copy()
    lifted[1] = 0.1
    ens.upload(lifted, z, z, 0.0)
    for m in range(2):
        for r in ens.flux_rhs(m):
            assert np.abs(r).max() == 0.0
    ens.model_step(1)
    e, u, v, t = ens.download()
    assert np.array_equal(e, lifted) and np.all(u == 0) and np.all(v == 0)
    assert np.all(t == 60.0)


def test_model_step_bitwise_10_members(oracle):
    """Config 1 (500x300, 10 members): 3 model steps bitwise equal to the oracle,
    including the per-member substep sequences."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair()
    n = 10
    e, u, v = perturbed_jets(oracle, p, n, seed=3)
    ens = Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.model_step(3)
    ge, gu, gv, gt = ens.download()
    subs = ens.substeps()
    for m in range(n):
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        dts = oracle.model_step(p, s, 3)
        assert np.array_equal(ge[m], s.eta), (m, np.abs(ge[m] - s.eta).max())
        assert np.array_equal(gu[m], s.hu)
        assert np.array_equal(gv[m], s.hv)
        assert gt[m] == s.t == 180.0
        assert subs[m] == len(dts)
    ens.close()


def _step_vs_oracle(oracle, nx, ny, n, steps, seed):
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(nx, ny)
    e, u, v = perturbed_jets(oracle, p, n, seed=seed)
    ens = Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.model_step(steps)
    ge, gu, gv, gt = ens.download()
    subs = ens.substeps()
    ens.close()
    for m in range(n):
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        dts = oracle.model_step(p, s, steps)
        assert np.array_equal(ge[m], s.eta), (nx, ny, m, np.abs(ge[m] - s.eta).max())
        assert np.array_equal(gu[m], s.hu), (nx, ny, m)
        assert np.array_equal(gv[m], s.hv), (nx, ny, m)
        assert gt[m] == s.t and subs[m] == len(dts)


# column counts around the 252-column CTA tile (one tile exactly, one column into a
# second tile, odd widths whose column pairs straddle the periodic seam), row counts
# with and without the short tail strips, a single member
@pytest.mark.parametrize("nx,ny,n", [(252, 40, 3), (253, 37, 2), (257, 64, 2), (101, 150, 3),
                                     (504, 301, 2), (37, 23, 1)])
def test_model_step_bitwise_shapes(oracle, nx, ny, n):
    _step_vs_oracle(oracle, nx, ny, n, 2, seed=nx + ny)


# the two substep-loop paths: the graph while-node (default) and the host-driven loop
# (DC_NO_GRAPH=1, also what a dc_profile window uses) -- both must give the same bits
@pytest.mark.parametrize("env", [{}, {"DC_NO_GRAPH": "1"}])
def test_model_step_bitwise_launch_variants(oracle, monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _step_vs_oracle(oracle, 500, 300, 3, 2, seed=11)


def test_profile_window_is_bitwise_and_complete(oracle):
    """dc_profile_begin/end: the stage kernels run one by one inside the window (host
    loop), results stay bitwise, and every launch is reported with its algorithmic bytes
    (24 / 36 B per cell for the two stages)."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(500, 300)
    e, u, v = perturbed_jets(oracle, p, 3, seed=12)
    ens = Ensemble(cfg, 3)
    ens.upload(e, u, v, 0.0)
    ens.profile_begin()
    ens.model_step(2)
    prof = {name: (n, ms, b) for name, n, ms, b in ens.profile_end()}
    ge, gu, gv, gt = ens.download()
    subs = 0
    for m in range(3):
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        dts = oracle.model_step(p, s, 2)
        subs = max(subs, len(dts))
        assert np.array_equal(ge[m], s.eta) and np.array_equal(gu[m], s.hu)
        assert np.array_equal(gv[m], s.hv)
    n1, ms1, b1 = prof["swe_stage_pair<1>"]
    n2, ms2, b2 = prof["swe_stage_pair<2>"]
    assert n1 == n2 >= subs and ms1 > 0 and ms2 > 0
    assert b1 == n1 * 24.0 * 3 * 500 * 300 and b2 == n2 * 36.0 * 3 * 500 * 300
    assert prof["step_begin"][0] == 2 and "fix_ghosts" in prof
    ens.close()


def test_model_step_fma_tolerance(oracle):
    """FMA build (exact_fp=0): the stencil contracts to FFMA, so the trajectory drifts
    from the reference at round-off level. Stated tolerance: max|diff| <= 5e-5 of
    max|field| after 10 model steps (70 substeps), measured drift ~1.7e-5 (SURVEY.md
    §8c quotes 2.9e-6 for the CPU's FMA build; nvcc contracts more expressions)."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(exact=False)
    n = 4
    e, u, v = perturbed_jets(oracle, p, n, seed=5)
    ens = Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.model_step(10)
    ge, gu, gv, _ = ens.download()
    for m in range(n):
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        oracle.model_step(p, s, 10)
        for a, b in ((ge[m], s.eta), (gu[m], s.hu), (gv[m], s.hv)):
            rel = np.abs(a.astype(np.float64) - b).max() / max(np.abs(b).max(), 1e-30)
            assert rel <= 5e-5, (m, rel)
    ens.close()


def test_cfl_dt_public_formula(oracle):
    """Stepper::cfl_dt (swe.hpp:212-226) and test_swe.cpp:46-62."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(16, 16)
    ens = Ensemble(cfg, 2)
    z = np.zeros((2, 16, 16), np.float32)
    hu = z.copy()
    hu[1] = 230.0
    ens.upload(z, hu, z, 0.0)
    dt = ens.cfl_dt()
    expect = 0.8 * 0.25 * 2220.0 / np.sqrt(9.806 * 230.0)
    assert abs(dt[0] - expect) <= 1e-3 * expect
    assert dt[1] < dt[0]
    assert dt[0] == oracle.cfl_dt(p, State(z[0], z[0], z[0]))


def test_perturb_injected_bitwise(oracle, ref):
    """perturb_state with the reference's own NoiseStream draws injected: the GPU
    reproduces the reference perturb_state bit-for-bit."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair()
    n = 3
    e, u, v = perturbed_jets(oracle, p, n, seed=9)
    ens = Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    offs, xis, refs = [], [], []
    for m in range(n):
        s = State(e[m].copy(), u[m].copy(), v[m].copy())
        o, xi = ref.perturb(p, s, 1, 1, m, 1)
        offs.append(o[0])
        xis.append(xi[0])
        refs.append(s)
    ens.perturb_state(np.array(offs), np.array(xis))
    ge, gu, gv, _ = ens.download()
    for m in range(n):
        assert np.array_equal(ge[m], refs[m].eta)
        assert np.array_equal(gu[m], refs[m].hu)
        assert np.array_equal(gv[m], refs[m].hv)


def test_perturb_philox_bitwise(oracle):
    """Counter-based Philox model error: GPU == CPU restatement, several draws."""
    _, Ensemble = _gpu()
    for nx, ny, c in [(500, 300, 5), (60, 60, 5), (30, 27, 3)]:
        cfg, p = cfg_pair(nx, ny, c_omega=c)
        n = 3
        e, u, v = perturbed_jets(oracle, p, n, seed=11)
        ens = Ensemble(cfg, n, member_base=7)
        ens.upload(e, u, v, 0.0)
        for _ in range(2):
            ens.perturb_state()
        ge, gu, gv, _ = ens.download()
        for m in range(n):
            s = State(e[m].copy(), u[m].copy(), v[m].copy())
            for d in range(2):
                oracle.perturb_philox(p, s, 7 + m, d)
            assert np.array_equal(ge[m], s.eta), (nx, m)
            assert np.array_equal(gu[m], s.hu)
            assert np.array_equal(gv[m], s.hv)
        ens.close()


@pytest.mark.parametrize("nx,ny,c,n", [(100, 305, 5, 1500), (99, 300, 3, 1500), (60, 90, 1, 4000)])
def test_perturb_column_strips_bitwise(oracle, nx, ny, c, n):
    """Enough members that q_half_apply runs as column strips of several tiles per CTA
    (the coarse-row ring, the pipeline across tiles, the TMA box re-armed per tile, a
    partial last tile at ny = 305; c_omega 5 / 3 / 1 size the ring): members at the start,
    middle and end of the ensemble bitwise equal to the CPU restatement, two draws."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair(nx, ny, c_omega=c)
    ens = Ensemble(cfg, n, member_base=3)
    ens.init_double_jet()
    for _ in range(2):
        ens.perturb_state()
    for m in (0, n // 2 + 1, n - 1):
        s = oracle.init_double_jet(p)
        for d in range(2):
            oracle.perturb_philox(p, s, 3 + m, d)
        e, u, v, _ = ens.download_member(m)
        assert np.array_equal(e, s.eta), (nx, c, m)
        assert np.array_equal(u, s.hu) and np.array_equal(v, s.hv), (nx, c, m)
    ens.close()


def test_step_perturb_sequence_bitwise(oracle):
    """Forecast with model error, 5 model steps with a Philox draw after each of the
    first 4 (the DA-cycle forecast pattern), bitwise."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair()
    n = 4
    e, u, v = perturbed_jets(oracle, p, n, seed=21)
    ens = Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    for s in range(5):
        ens.model_step(1)
        if s < 4:
            ens.perturb_state()
    ge, gu, gv, gt = ens.download()
    for m in range(n):
        st = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        for s in range(5):
            oracle.model_step(p, st, 1)
            if s < 4:
                oracle.perturb_philox(p, st, m, s)
        assert np.array_equal(ge[m], st.eta) and np.array_equal(gu[m], st.hu)
        assert np.array_equal(gv[m], st.hv) and gt[m] == st.t


def test_dry_cell_rejected():
    """test_swe.cpp:235-243: DryCellError on a dry cell."""
    _, Ensemble = _gpu()
    from paper_1910_01031_b200 import DcError
    cfg, p = cfg_pair(16, 12)
    ens = Ensemble(cfg, 1)
    z = np.zeros((1, 12, 16), np.float32)
    e = z.copy()
    e[0, 4, 3] = -231.0
    ens.upload(e, z, z, 0.0)
    with pytest.raises(DcError) as ei:
        ens.flux_rhs(0)
    assert ei.value.status == 2 and "dry cell at (3,4)" in ei.value.message
    with pytest.raises(DcError) as ei:
        ens.cfl_dt()
    assert ei.value.status == 2


def test_double_jet_init_matches(oracle):
    _, Ensemble = _gpu()
    cfg, p = cfg_pair()
    ens = Ensemble(cfg, 2)
    ens.init_double_jet()
    e, u, v, t = ens.download()
    s = oracle.init_double_jet(p)
    assert np.array_equal(e[1], s.eta) and np.array_equal(u[1], s.hu) and np.all(v == 0)


def test_branch_free_sqrt_rcp_exhaustive():
    """The stencil's branch-free sqrt / reciprocal equal __fsqrt_rn / __frcp_rn on every
    float in [2^-100, 2^100] (checked exhaustively, ~1.7e9 operands), which is what makes
    the Exact policy IEEE for every state the model admits (depths ~1e2, speeds ~1e1)."""
    _gpu()
    import ctypes as C
    from paper_1910_01031_b200 import load
    L = load()
    counts = (C.c_uint64 * 4)()
    assert L.dc_selftest_math(0, counts) == 0
    assert counts[0] == 0, f"sqrt mismatches in [2^-100,2^100]: {counts[0]} (all: {counts[2]})"
    assert counts[1] == 0, f"rcp mismatches in [2^-100,2^100]: {counts[1]} (all: {counts[3]})"


@pytest.mark.parametrize("field,value", [("hu", np.nan), ("hv", np.inf)])
def test_non_finite_state_reported_like_reference(oracle, ref, field, value):
    """A non-finite transport poisons the substep: the reference's heun sentinel
    (swe.hpp:99,416-418) throws "model_step: non-finite value after substep k"; the GPU's
    running packed sentinel reports the same error, substep and member."""
    _, Ensemble = _gpu()
    from paper_1910_01031_b200 import DcError
    cfg, p = cfg_pair(100, 60)
    eta, hu, hv = perturbed_jets(oracle, p, 3, seed=5)
    bad = {"hu": hu, "hv": hv}[field]
    bad[1, 30, 40] = value
    s = State(eta[1].copy(), hu[1].copy(), hv[1].copy(), 0.0)
    from checkers import CheckerError
    with pytest.raises(CheckerError) as er:
        ref.model_step(p, s, 1)
    ens = Ensemble(cfg, 3)
    ens.upload(eta, hu, hv, 0.0)
    with pytest.raises(DcError) as eg:
        ens.model_step(1)
        ens.sync()  # device errors surface at the next synchronising call
    assert eg.value.status == 3 and eg.value.member == 1
    assert er.value.msg in eg.value.message, (er.value.msg, eg.value.message)
    assert eg.value.message.startswith("model_step: non-finite value after substep ")


# every substep-loop variant must retire errored members and finish the step: a member
# dry at step start (never steps), one poisoned mid-substep (non-finite), all members dry
@pytest.mark.timeout(300)
@pytest.mark.parametrize("env", [{}, {"DC_NO_GRAPH": "1"}])
def test_errored_members_retire_in_every_loop_variant(oracle, monkeypatch, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, Ensemble = _gpu()
    from paper_1910_01031_b200 import DcError
    cfg, p = cfg_pair(100, 60)
    e, u, v = perturbed_jets(oracle, p, 4, seed=6)
    e[1, 10, 20] = -231.0  # dry at step start
    u[2, 30, 40] = np.nan  # non-finite after the first substep
    ens = Ensemble(cfg, 4)
    ens.upload(e, u, v, 0.0)
    with pytest.raises(DcError):
        ens.model_step(2)
        ens.sync()
    with pytest.raises(DcError):
        ens.download()
    ge, gu, gv, gt = ens.download(strict=False)
    for m in (0, 3):  # the healthy members stepped on, bitwise
        s = State(e[m].copy(), u[m].copy(), v[m].copy(), 0.0)
        oracle.model_step(p, s, 2)
        assert np.array_equal(ge[m], s.eta) and np.array_equal(gu[m], s.hu)
        assert np.array_equal(gv[m], s.hv) and gt[m] == s.t
    ens.close()
    e[:, 10, 20] = -231.0  # nobody can step
    ens = Ensemble(cfg, 4)
    ens.upload(e, u, v, 0.0)
    with pytest.raises(DcError):
        ens.model_step(1)
        ens.sync()
    ens.close()


def test_failed_member_recovers_when_overwritten(oracle):
    """A member that failed (dry cell) is healthy again once its state is overwritten --
    re-uploaded, or resampled from a healthy particle -- and then steps bitwise like the
    oracle (the reference throws per call and never poisons a particle)."""
    _, Ensemble = _gpu()
    from paper_1910_01031_b200 import DcError
    cfg, p = cfg_pair(100, 60)
    e, u, v = perturbed_jets(oracle, p, 3, seed=8)
    bad = e.copy()
    bad[1, 10, 20] = -231.0
    ens = Ensemble(cfg, 3)
    ens.upload(bad, u, v, 0.0)
    with pytest.raises(DcError):
        ens.model_step(1)
        ens.sync()
    ens.upload_member(1, e[1], u[1], v[1], 0.0)  # reload the failed particle
    ens.model_step(1)  # every member steps now (no error surfaces)
    ge, gu, gv, gt = ens.download()
    s = State(e[1].copy(), u[1].copy(), v[1].copy(), 0.0)
    oracle.model_step(p, s, 1)
    assert np.array_equal(ge[1], s.eta) and np.array_equal(gu[1], s.hu) and gt[1] == 60.0
    # resampling a failed slot from a healthy source clears it; a failed source carries its
    # error into the slots that copy it
    ens.upload(bad, u, v, 0.0)
    with pytest.raises(DcError):
        ens.model_step(1)
        ens.sync()
    ens.resample_members(np.array([0, 0, 2], np.int32))
    ens.model_step(1)
    ens.sync()
    ens.close()


@pytest.mark.timeout(600)
def test_many_members_one_context(oracle):
    """5100 members of the 500x300 jet in one context (members x strips > 65535, the old
    gridDim.y cliff of the stage grid; the stage grid is 1-D now): one model step, the
    first and last members bitwise equal to the oracle."""
    _, Ensemble = _gpu()
    cfg, p = cfg_pair()
    n = 5100
    ens = Ensemble(cfg, n)
    ens.init_double_jet()
    ens.model_step(1)
    s = oracle.init_double_jet(p)
    oracle.model_step(p, s, 1)
    for m in (0, n - 1):
        e, u, v, t = ens.download_member(m)
        assert np.array_equal(e, s.eta) and np.array_equal(u, s.hu) and np.array_equal(v, s.hv)
        assert t == 60.0
    ens.close()
