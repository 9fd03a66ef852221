"""§8(f) rows on the CPU: the oracle's restatement against SPEC.md's known answers, and
the library's host-side functions (PF weight normalisation, residual resampling, the
observation file) against the oracle, bit for bit. No GPU needed."""
import math
import os

import numpy as np
import pytest

from checkers import Oracle, make_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def lib():
    from paper_1910_01031_b200 import _lib
    try:
        return _lib.load()
    except ImportError as e:
        pytest.skip(str(e))


# ---- observe_drifter ----
def test_observe_drifter_known_answers(orc):
    p = make_params(nx=100, ny=60, dx=2220.0, dy=2220.0)
    # stationary drifter, eps = 0 -> y = [0, 0]
    y = orc.observe_drifters(p, [[1000.0, 2000.0]], [[1000.0, 2000.0]], 300.0)
    assert y.tolist() == [[0.0, 0.0]]
    # dx = 30 m, dt_obs = 300 s, H = 230 -> y_hu = 23.0 before noise
    y = orc.observe_drifters(p, [[1000.0, 2000.0]], [[1030.0, 2000.0]], 300.0)
    assert y[0, 0] == 23.0 and y[0, 1] == 0.0
    # wrapped drifter: minimal image, |dx| <= nx*dx/2
    lx = p.nx * p.dx
    y = orc.observe_drifters(p, [[lx - 10.0, 5.0]], [[20.0, 5.0]], 300.0)
    assert y[0, 0] == pytest.approx(30.0 / 300.0 * 230.0, rel=1e-12)
    y = orc.observe_drifters(p, [[20.0, 5.0]], [[lx - 10.0, 5.0]], 300.0)
    assert y[0, 0] == pytest.approx(-30.0 / 300.0 * 230.0, rel=1e-12)
    # noise is added
    y = orc.observe_drifters(p, [[1000.0, 2000.0]], [[1030.0, 2000.0]], 300.0,
                             eps=[[0.5, -0.25]])
    assert y.tolist() == [[23.5, -0.25]]


def test_obs_noise_statistics_and_determinism(orc):
    p = make_params(nx=100, ny=60)
    ids = np.arange(4000)
    e1 = orc.obs_noise(p, 0, ids, 7, r_hu=1.0, r_hv=4.0)
    e2 = orc.obs_noise(p, 0, ids, 7, r_hu=1.0, r_hv=4.0)
    assert np.array_equal(e1, e2)
    assert abs(e1[:, 0].mean()) < 0.06 and abs(e1[:, 0].var() - 1.0) < 0.08
    assert abs(e1[:, 1].var() - 4.0) < 0.3
    # streams differ by platform kind and by observation index
    assert not np.array_equal(e1, orc.obs_noise(p, 1, ids, 7, r_hu=1.0, r_hv=4.0))
    assert not np.array_equal(e1, orc.obs_noise(p, 0, ids, 8, r_hu=1.0, r_hv=4.0))


# ---- standard PF weights / residual resampling ----
def test_pf_weights_known_answers(orc):
    w, mx, ok = orc.pf_weights(np.zeros(5))
    assert ok and np.allclose(w, 0.2) and mx == 0.0
    ll = np.array([-3.0, -1.0, -2.0, -7.5])
    w1, _, _ = orc.pf_weights(ll)
    w2, _, _ = orc.pf_weights(ll + 123.25)
    assert np.allclose(w1, w2, rtol=1e-14, atol=0)  # invariant under a constant shift
    assert math.isclose(w1.sum(), 1.0, rel_tol=1e-15)
    w, _, _ = orc.pf_weights(np.array([-1e4, 0.0, -2e4]))
    assert w[1] == 1.0
    _, mx, ok = orc.pf_weights(np.array([-800.0, -801.0]))
    assert not ok and mx == -800.0  # every exp(loglik) underflows: ensemble collapse


def test_residual_resample_known_answers(orc):
    assert orc.residual_resample(np.full(7, 1 / 7), 1, 0).tolist() == list(range(7))
    assert orc.residual_resample(np.full(49, 1 / 49), 1, 0).tolist() == list(range(49))
    assert orc.residual_resample([0.5, 0.5, 0, 0], 1, 0).tolist() == [0, 0, 1, 1]
    rng = np.random.default_rng(3)
    for trial in range(20):
        w = rng.random(50) ** 4
        w /= w.sum()
        idx = orc.residual_resample(w, 5, trial)
        assert len(idx) == 50 and np.all(np.diff(idx) >= 0)
        counts = np.bincount(idx, minlength=50)
        assert np.all(counts >= np.floor(50 * w + 1e-12))  # the floor guarantee
        assert np.all(counts[w >= 1 / 50] >= 1)


def test_library_pf_weights_and_resample_match_oracle(orc):
    import paper_1910_01031_b200 as dc
    rng = np.random.default_rng(11)
    for trial in range(10):
        ll = -rng.random(64) * 50.0 - 10.0
        w_o, mx_o, _ = orc.pf_weights(ll)
        w_l, mx_l = dc.pf_weights(ll)
        assert np.array_equal(w_o, w_l) and mx_o == mx_l
        assert np.array_equal(orc.residual_resample(w_o, 1, trial),
                              dc.residual_resample(w_l, 1, trial))
    with pytest.raises(dc.DcError):
        dc.pf_weights([-900.0, -950.0])
    w, mx = dc.pf_weights([-900.0, -950.0], strict=False)
    assert mx == -900.0 and w[0] == 1.0


# ---- forecast_error ----
def test_forecast_error_known_answers(orc):
    p = make_params(nx=100, ny=60)
    truth = np.array([[5000.0, 7000.0], [1000.0, 100.0]])
    pos = np.repeat(truth[None], 3, 0)
    wind = np.zeros(pos.shape, np.int32)
    E, R, ed, rd = orc.forecast_error(p, pos, wind, truth)
    assert E == 0.0 and R == 0.0
    # one drifter, two particles at +-a in x: E = a, spread about the mean = a
    a = 250.0
    pos = np.array([[[5000.0 + a, 7000.0]], [[5000.0 - a, 7000.0]]])
    E, R, ed, rd = orc.forecast_error(p, pos, np.zeros(pos.shape, np.int32), truth[:1])
    assert E == a and R == a
    # periodic: particles either side of x = 0 are close to a truth at x = 0
    lx = p.nx * p.dx
    pos = np.array([[[lx - 10.0, 50.0]], [[10.0, 50.0]]])
    wind = np.array([[[-1, 0]], [[0, 0]]], np.int32)  # the first wrapped left
    E, R, ed, rd = orc.forecast_error(p, pos, wind, np.array([[0.0, 50.0]]))
    assert E == pytest.approx(10.0, rel=1e-12) and R == pytest.approx(10.0, rel=1e-9)


# ---- observation file ----
def test_obs_file_round_trip(tmp_path, lib):
    import paper_1910_01031_b200 as dc
    rng = np.random.default_rng(5)
    recs = []
    for i in range(200):
        recs.append((300.0 * (i // 20), i % 2, i, rng.random() * 1.1e6, rng.random() * 6.6e5,
                     rng.normal() * 30.0, rng.normal() * 1e-7))
    recs.append((0.1 + 0.2, 0, 7, -0.0, 5e-324, 1.7976931348623157e308, math.pi))
    path = tmp_path / "obs.txt"
    dc.write_obs_file(path, recs[:100])
    dc.write_obs_file(path, recs[100:], append=True)
    back = dc.read_obs_file(path)
    assert len(back) == len(recs)
    for a, b in zip(recs, back):
        assert a[1:3] == b[1:3]
        for u, v in zip(a[:1] + a[3:], b[:1] + b[3:]):
            assert np.float64(u).tobytes() == np.float64(v).tobytes()
    line = open(path).read().splitlines()[1]
    assert line.split(",")[1] == "mooring" and len(line.split(",")) == 7


def test_obs_file_rejects_malformed(tmp_path, lib):
    import paper_1910_01031_b200 as dc
    p = tmp_path / "bad.txt"
    p.write_text("0,drifter,1,2,3,4\n")
    with pytest.raises(dc.DcError):
        dc.read_obs_file(p)
    p.write_text("0,buoy,1,2,3,4,5\n")
    with pytest.raises(dc.DcError):
        dc.read_obs_file(p)
    with pytest.raises(dc.DcError):
        dc.read_obs_file(tmp_path / "missing.txt")
