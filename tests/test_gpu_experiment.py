"""GPU parity of the §8(f) rows either side of the path (C ABI vs oracle/ and the compiled
reference): observation synthesis (noise, observe_drifter), the SIR comparison (PF
log-likelihoods, resampling by copy), the drifter forecast error, DCST snapshots
(byte-identical to the reference writer) and checkpoint/restore (bitwise resume)."""
import os

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


def setup(nx=100, ny=60):
    pkg = _gpu()
    cfg = pkg.Config(nx=nx, ny=ny)
    p = make_params(nx=nx, ny=ny, q0=cfg.q0, seed=cfg.seed, c_omega=cfg.c_omega)
    return pkg, cfg, p


def spread_states(oracle, p, n, seed):
    e = np.empty((n, p.ny, p.nx), np.float32)
    u, v = np.empty_like(e), np.empty_like(e)
    for m in range(n):
        s = oracle.init_double_jet(p)
        for d in range(2):
            oracle.perturb_philox(p, s, 500 + m + 31 * seed, d)
        e[m], u[m], v[m] = s.eta, s.hu, s.hv
    return e, u, v


def test_obs_noise_and_observe_drifters_match_oracle(oracle):
    pkg, cfg, p = setup()
    ens = pkg.Ensemble(cfg, 1)
    ids = np.arange(64, dtype=np.int32)
    for kind in (0, 1):
        for idx in (0, 5, 1 << 33):
            g = ens.obs_noise(kind, ids, idx, r_hu=1.0, r_hv=2.5)
            o = oracle.obs_noise(p, kind, ids, idx, r_hu=1.0, r_hv=2.5)
            assert np.array_equal(g, o)
    rng = np.random.default_rng(2)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    prev = rng.uniform(0, 1, (64, 2)) * [lx, ly]
    cur = (prev + rng.normal(0, 3000.0, (64, 2))) % [lx, ly]
    prev[0] = [lx - 5.0, 10.0]
    cur[0] = [7.0, ly - 3.0]
    eps = ens.obs_noise(0, ids, 3)
    for e in (None, eps):
        assert np.array_equal(ens.observe_drifters(prev, cur, 300.0, e),
                              oracle.observe_drifters(p, prev, cur, 300.0, e))


def test_pf_loglik_matches_oracle(oracle):
    pkg, cfg, p = setup()
    n = 5
    e, u, v = spread_states(oracle, p, n, 1)
    rng = np.random.default_rng(4)
    obs = np.hstack([rng.uniform(0, 1, (40, 2)) * [p.nx * p.dx, p.ny * p.dy],
                     rng.normal(0, 20.0, (40, 2))])
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    g = ens.pf_loglik(obs, r_hu=1.0, r_hv=10.0)
    o = np.array([oracle.pf_loglik(p, State(e[m], u[m], v[m]), obs, 1.0, 10.0) for m in range(n)])
    assert np.array_equal(g, o)
    w, _ = pkg.pf_weights(g, strict=False)
    assert np.isclose(w.sum(), 1.0)


def test_resample_members_by_copy(oracle):
    pkg, cfg, p = setup()
    n = 6
    e, u, v = spread_states(oracle, p, n, 2)
    pos = np.random.default_rng(8).uniform(0, 1, (n, 4, 2)) * [p.nx * p.dx, p.ny * p.dy]
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 120.0)
    ens.drifters_set(pos)
    ens.advect_drifters(60.0)
    p0, w0 = ens.drifters_get()
    idx = np.array([0, 0, 2, 3, 3, 3], np.int32)
    ens.resample_members(idx)
    ge, gu, gv, gt = ens.download()
    assert np.array_equal(ge, e[idx]) and np.array_equal(gu, u[idx]) and np.array_equal(gv, v[idx])
    p1, w1 = ens.drifters_get()
    assert np.array_equal(p1, p0[idx]) and np.array_equal(w1, w0[idx])
    assert np.all(gt == 120.0)
    ens.model_step(1)  # the resampled state steps (CFL statistics rescanned)
    assert np.all(ens.download()[3] == 180.0)


def test_forecast_error_matches_oracle(oracle):
    pkg, cfg, p = setup()
    n = 7
    e, u, v = spread_states(oracle, p, n, 3)
    rng = np.random.default_rng(9)
    pos = rng.uniform(0, 1, (5, 2)) * [p.nx * p.dx, p.ny * p.dy]
    ens = pkg.Ensemble(cfg, n)
    ens.upload(e, u, v, 0.0)
    ens.drifters_set(pos)
    for _ in range(30):
        ens.advect_drifters(600.0)
    gp, gw = ens.drifters_get()
    truth = (pos + rng.normal(0, 2000.0, pos.shape)) % [p.nx * p.dx, p.ny * p.dy]
    E, R, ed, rd = ens.forecast_error(truth)
    Eo, Ro, edo, rdo = oracle.forecast_error(p, gp, gw, truth)
    assert E == Eo and R == Ro and np.array_equal(ed, edo) and np.array_equal(rd, rdo)


def test_forecast_error_many_members_matches_oracle(oracle):
    """More members than one chunk of the per-drifter CTA (128): the chunked member-order
    folds still give the sequential sums bit for bit."""
    pkg, cfg, p = setup()
    n, n_d = 300, 5
    rng = np.random.default_rng(17)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    ens = pkg.Ensemble(cfg, n)
    ens.init_double_jet()
    ens.drifters_set(rng.uniform(0, 1, (n, n_d, 2)) * [lx, ly])
    for _ in range(40):  # the jet carries drifters across the periodic edge: windings
        ens.advect_drifters(3000.0)
    gp, gw = ens.drifters_get()
    assert np.any(gw != 0)
    truth = rng.uniform(0, 1, (n_d, 2)) * [lx, ly]
    E, R, ed, rd = ens.forecast_error(truth)
    Eo, Ro, edo, rdo = oracle.forecast_error(p, gp, gw, truth)
    assert E == Eo and R == Ro and np.array_equal(ed, edo) and np.array_equal(rd, rdo)


def test_forecast_error_gathered_slices_equal_one_context(oracle):
    """ranks hold member slices; their drifter ensembles gathered into one
    device buffer (member-id order) give forecast statistics bitwise equal to one context
    holding every member (two contexts on one GPU stand in for two ranks)."""
    import torch
    pkg, cfg, p = setup()
    n, cut = 7, 3
    e, u, v = spread_states(oracle, p, n, 5)
    rng = np.random.default_rng(21)
    pos = rng.uniform(0, 1, (6, 2)) * [p.nx * p.dx, p.ny * p.dy]
    whole = pkg.Ensemble(cfg, n)
    parts = [pkg.Ensemble(cfg, cut), pkg.Ensemble(cfg, n - cut, member_base=cut)]
    whole.upload(e, u, v, 0.0)
    parts[0].upload(e[:cut], u[:cut], v[:cut], 0.0)
    parts[1].upload(e[cut:], u[cut:], v[cut:], 0.0)
    for ens in [whole] + parts:
        ens.drifters_set(pos)
        for _ in range(3):
            ens.advect_drifters(60.0)
            ens.model_step(1)
            ens.perturb_state()
    truth = (pos + rng.normal(0, 2000.0, pos.shape)) % [p.nx * p.dx, p.ny * p.dy]
    gpos = torch.empty((n, 6, 2), dtype=torch.float64, device="cuda")
    gwind = torch.empty((n, 6, 2), dtype=torch.int32, device="cuda")
    parts[0].drifters_to_device(gpos[:cut].data_ptr(), gwind[:cut].data_ptr())
    parts[1].drifters_to_device(gpos[cut:].data_ptr(), gwind[cut:].data_ptr())
    for ens in parts:
        ens.sync()
    E, R, ed, rd = pkg.forecast_error_gathered(cfg, n, 6, gpos.data_ptr(), gwind.data_ptr(),
                                               truth)
    Ew, Rw, edw, rdw = whole.forecast_error(truth)
    assert E == Ew and R == Rw and np.array_equal(ed, edw) and np.array_equal(rd, rdw)
    wp, ww = whole.drifters_get()
    assert np.array_equal(gpos.cpu().numpy(), wp) and np.array_equal(gwind.cpu().numpy(), ww)
    with pytest.raises(pkg.DcError):
        pkg.forecast_error_gathered(cfg, n, 6, 0, 0, truth)
    for ens in [whole] + parts:
        ens.close()


def test_snapshot_bytes_match_reference_writer(oracle, ref, tmp_path):
    pkg, cfg, p = setup()
    e, u, v = spread_states(oracle, p, 2, 4)
    ens = pkg.Ensemble(cfg, 2)
    ens.upload(e, u, v, 1234.5)
    ens.save_snapshot(1, tmp_path / "gpu.dcst")
    ref.save_snapshot(p, State(e[1], u[1], v[1], 1234.5), tmp_path / "ref.dcst")
    assert (tmp_path / "gpu.dcst").read_bytes() == (tmp_path / "ref.dcst").read_bytes()
    # the reference reads ours and we read the reference's
    s = ref.load_snapshot(p, tmp_path / "gpu.dcst")
    assert np.array_equal(s.eta, e[1]) and np.array_equal(s.hv, v[1]) and s.t == 1234.5
    ens.load_snapshot(0, tmp_path / "ref.dcst")
    ge, gu, gv, gt = ens.download()
    assert np.array_equal(ge[0], e[1]) and np.array_equal(gu[0], u[1]) and gt[0] == 1234.5


def test_snapshot_errors(tmp_path):
    pkg, cfg, p = setup()
    ens = pkg.Ensemble(cfg, 1)
    ens.init_double_jet()
    ens.save_snapshot(0, tmp_path / "a.dcst")
    raw = (tmp_path / "a.dcst").read_bytes()
    cases = {"bad magic": b"DCSX" + raw[4:], "unsupported version": raw[:4] + b"\x02" + raw[5:],
             "truncated field data": raw[:-7], "implausible extents": raw[:8] + b"\0\0\0\0" + raw[12:]}
    for msg, blob in cases.items():
        (tmp_path / "b.dcst").write_bytes(blob)
        with pytest.raises(pkg.DcError) as ex:
            ens.load_snapshot(0, tmp_path / "b.dcst")
        assert msg in str(ex.value) and ex.value.status == 8
    other = pkg.Ensemble(pkg.Config(nx=50, ny=60), 1)
    with pytest.raises(pkg.DcError) as ex:
        other.load_snapshot(0, tmp_path / "a.dcst")
    assert ex.value.status == 1


def test_checkpoint_resume_is_bitwise(oracle, tmp_path):
    """checkpoint/restore mid-assimilation reproduces the uninterrupted run."""
    pkg, cfg, p = setup()
    n = 4
    e, u, v = spread_states(oracle, p, n, 5)
    rng = np.random.default_rng(6)
    obs = [np.hstack([rng.uniform(0, 1, (6, 2)) * [p.nx * p.dx, p.ny * p.dy],
                      rng.normal(0, 20.0, (6, 2))]) for _ in range(4)]
    _, S = pkg.precompute_S(cfg)
    _, usig = pkg.precompute_local_svd(cfg, S)
    pos = np.random.default_rng(7).uniform(0, 1, size=(n, 5, 2)) * [p.nx * p.dx, p.ny * p.dy]
    a = pkg.Ensemble(cfg, n)
    a.upload(e, u, v, 0.0)
    a.drifters_set(pos)  # drifter copies are advected by every cycle: they must resume too
    for c in range(2):
        a.da_cycle(5, obs[c], S, usig, c)
    a.checkpoint_save(tmp_path / "ck", filter_cycle=2)
    for c in range(2, 4):
        a.da_cycle(5, obs[c], S, usig, c)
    want = a.download()
    want_d = a.drifters_get()
    b = pkg.Ensemble(cfg, n)
    cyc = b.checkpoint_load(tmp_path / "ck")
    assert cyc == 2 and b.draw_counter == a.draw_counter - 8
    for c in range(cyc, 4):
        b.da_cycle(5, obs[c], S, usig, c)
    got = b.download()
    for x, y in zip(want, got):
        assert np.array_equal(x, y)
    got_d = b.drifters_get()
    assert np.array_equal(want_d[0], got_d[0]) and np.array_equal(want_d[1], got_d[1])
    names = sorted(os.listdir(tmp_path / "ck" / "ensemble"))
    assert names == sorted([f"particle_{i}.dcst" for i in range(n)] +
                           [f"particle_{i}.drifters" for i in range(n)])


def test_trajectory_file(tmp_path):
    pkg, cfg, p = setup()
    ens = pkg.Ensemble(cfg, 3, member_base=10)
    ens.init_double_jet()
    pos = np.random.default_rng(1).uniform(0, 1, (3, 4, 2)) * [p.nx * p.dx, p.ny * p.dy]
    ens.drifters_set(pos)
    ens.trajectory_write(tmp_path / "traj.txt", 0.0, append=False)
    ens.advect_drifters(60.0)
    ens.trajectory_write(tmp_path / "traj.txt", 60.0)
    lines = open(tmp_path / "traj.txt").read().splitlines()
    assert len(lines) == 2 * 3 * 4
    gp, gw = ens.drifters_get()
    t, particle, drifter, x, y, wx, wy = lines[-1].split(",")
    assert float(t) == 60.0 and int(particle) == 12 and int(drifter) == 3
    assert float(x) == gp[2, 3, 0] and float(y) == gp[2, 3, 1] and int(wx) == gw[2, 3, 0]


def test_generate_truth_matches_oracle(oracle, tmp_path):
    """generate_truth: the GPU truth run, its drifter/mooring records and
    its snapshots equal the oracle's replay of the same definition bit for bit; same seed
    twice gives byte-identical observation files."""
    pkg, cfg, p = setup()
    kw = dict(duration=1800.0, insert_time=600.0, obs_interval=300.0, snapshot_interval=900.0,
              drifters=(4, 3), moorings=(3, 2), r=(1.0, 2.0))
    n = pkg.generate_truth(cfg, tmp_path / "a", **kw)
    assert n == (12 + 6) * 4  # platforms x observation times (900, 1200, 1500, 1800)
    pkg.generate_truth(cfg, tmp_path / "b", **kw)
    fa = (tmp_path / "a" / "observations.txt").read_bytes()
    assert fa == (tmp_path / "b" / "observations.txt").read_bytes()
    recs = pkg.read_obs_file(tmp_path / "a" / "observations.txt")
    # oracle replay: init, then per 60 s step: drifters, model step, truth model error
    s = oracle.init_double_jet(p)
    lx, ly = p.nx * p.dx, p.ny * p.dy
    lat = lambda a, b: np.array([[(i + 0.5) / a * lx, (j + 0.5) / b * ly]  # noqa: E731
                                 for j in range(b) for i in range(a)])
    moor = lat(3, 2)
    want, pos, prev, k = [], None, None, 0
    for step in range(31):
        if step == 10:
            pos = lat(4, 3)
            prev = pos.copy()
        if step > 10 and (step - 10) % 5 == 0:
            t = step * 60.0
            eps = oracle.obs_noise(p, 0, np.arange(12), k, 1.0, 2.0)
            y = oracle.observe_drifters(p, prev, pos, 300.0, eps)
            want += [(t, 0, i, pos[i, 0], pos[i, 1], y[i, 0], y[i, 1]) for i in range(12)]
            prev = pos.copy()
            eps = oracle.obs_noise(p, 1, np.arange(6), k, 1.0, 2.0)
            for i in range(6):
                ym = oracle.observe_mooring(p, s, moor[i, 0], moor[i, 1])
                want.append((t, 1, i, moor[i, 0], moor[i, 1], ym[0] + eps[i, 0],
                             ym[1] + eps[i, 1]))
            k += 1
        if step in (15, 30):
            g = pkg.Ensemble(cfg, 1)
            g.load_snapshot(0, tmp_path / "a" / f"truth_{step * 60}.dcst")
            ge, gu, gv, gt = g.download()
            assert np.array_equal(ge[0], s.eta) and np.array_equal(gv[0], s.hv)
            assert gt[0] == step * 60.0
        if step == 30:
            break
        if pos is not None:
            oracle.advect_drifters(p, s, pos, 60.0)
        oracle.model_step(p, s, 1)
        oracle.perturb_philox_tag(p, s, 3, 0, step)
    assert len(recs) == len(want)
    for a, b in zip(recs, want):
        assert a[:3] == b[:3] and all(np.float64(x) == np.float64(y) for x, y in zip(a[3:], b[3:]))


def test_resample_across_two_contexts_equals_one(oracle):
    """Cross-rank resampling (resample.py): two contexts on one GPU stand in for two
    ranks; members that change context travel as dc_member_export / dc_member_import
    buffers routed by exchange_plan. Fields, times and drifter copies equal one context
    resampling with the same global index, bit for bit."""
    import torch
    pkg, cfg, p = setup()
    from paper_1910_01031_b200.resample import exchange_plan
    n, per = 6, 3
    e, u, v = spread_states(oracle, p, n, 9)
    rng = np.random.default_rng(12)
    pos = rng.uniform(0, 1, (n, 4, 2)) * [p.nx * p.dx, p.ny * p.dy]
    whole = pkg.Ensemble(cfg, n)
    parts = [pkg.Ensemble(cfg, per), pkg.Ensemble(cfg, per, member_base=per)]
    whole.upload(e, u, v, 0.0)
    whole.drifters_set(pos)
    for r, ens in enumerate(parts):
        ens.upload(e[r * per:(r + 1) * per], u[r * per:(r + 1) * per], v[r * per:(r + 1) * per], 0.0)
        ens.drifters_set(pos[r * per:(r + 1) * per])
    for ens in [whole] + parts:
        for _ in range(2):
            ens.advect_drifters(3000.0)
            ens.model_step(1)
    idx = np.array([0, 4, 4, 1, 5, 2], np.int32)  # sorted is not required by the routing
    whole.resample_members(idx)
    nb = parts[0].member_bytes()
    assert nb == whole.member_bytes()
    plans = [exchange_plan(idx, per, r) for r in range(2)]
    wire = {}
    for r, ens in enumerate(parts):  # exports first (the local gather overwrites members)
        for dest, src in plans[r][1]:
            b = torch.empty(nb, dtype=torch.uint8, device="cuda")
            ens.member_export(src, b.data_ptr())
            wire[(r, src, dest)] = b
    for r, ens in enumerate(parts):
        ens.sync()
    for r, ens in enumerate(parts):
        ens.resample_members(plans[r][0])
        for sr, sl, slots in plans[r][2]:
            for i in slots:
                ens.member_import(i, wire[(sr, sl, r)].data_ptr())
        ens.sync()
    we, wu, wv, wt = whole.download()
    wp, ww = whole.drifters_get()
    for r, ens in enumerate(parts):
        ge, gu, gv, gt = ens.download()
        gp, gw = ens.drifters_get()
        sl = slice(r * per, (r + 1) * per)
        assert np.array_equal(ge, we[sl]) and np.array_equal(gu, wu[sl]) and np.array_equal(gv, wv[sl])
        assert np.array_equal(gt, wt[sl]) and np.array_equal(gp, wp[sl]) and np.array_equal(gw, ww[sl])
    # the imported states step on like the whole ensemble (CFL statistics rescanned)
    whole.model_step(1)
    for ens in parts:
        ens.model_step(1)
    we = whole.download()[0]
    assert np.array_equal(np.concatenate([ens.download()[0] for ens in parts]), we)
