"""Pin the CPU restatement (oracle/liboracle.so) against golden vectors produced by the
REFERENCE's own compiled operators (tests/golden/make_golden.py, oracle/ref_shim.cpp).
Bitwise for every array: the restatement must reproduce the reference exactly before it
is trusted as the checker of the CUDA path. Runs on any host (no /root/reference needed).
"""
import os

import numpy as np
import pytest

from checkers import State, make_params

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_ops.npz"))


def test_golden_jet(oracle):
    p = make_params(nx=40, ny=30)
    s = oracle.init_double_jet(p)
    assert np.array_equal(s.eta, G["jet_eta"]) and np.array_equal(s.hu, G["jet_hu"])
    assert np.array_equal(s.hv, G["jet_hv"])


def test_golden_flux_rhs_and_cfl(oracle):
    p = make_params(nx=40, ny=30)
    s = State(G["s0_eta"].copy(), G["s0_hu"].copy(), G["s0_hv"].copy())
    r = oracle.flux_rhs(p, s)
    for a, k in zip(r, ("rhs_eta", "rhs_hu", "rhs_hv")):
        assert np.array_equal(a, G[k]), k
    assert oracle.cfl_dt(p, s) == float(G["cfl_dt"])


def test_golden_model_step(oracle):
    """Three Stepper::model_step calls: state and the full substep dt sequence."""
    p = make_params(nx=40, ny=30)
    s = State(G["s0_eta"].copy(), G["s0_hu"].copy(), G["s0_hv"].copy(), 0.0)
    dts = [oracle.model_step(p, s, 1) for _ in range(3)]
    assert [len(d) for d in dts] == list(G["step3_nsub"])
    assert np.array_equal(np.concatenate(dts), G["step3_dts"])
    assert np.array_equal(s.eta, G["step3_eta"]) and np.array_equal(s.hu, G["step3_hu"])
    assert np.array_equal(s.hv, G["step3_hv"]) and s.t == float(G["step3_t"])


def test_golden_perturb_with_reference_noise(oracle):
    """perturb_state x3 with NoiseStream(123, model_error, 4): the restatement fed the
    reference's offsets + xi reproduces the reference state bitwise."""
    q = make_params(nx=60, ny=60)
    s = State(G["pe_in_eta"].copy(), G["pe_in_hu"].copy(), G["pe_in_hv"].copy())
    for d in range(3):
        oj, ok = G["pe_offsets"][d]
        oracle.perturb_injected(q, s, int(oj), int(ok), G["pe_xi"][d])
    assert np.array_equal(s.eta, G["pe_out_eta"])
    assert np.array_equal(s.hu, G["pe_out_hu"]) and np.array_equal(s.hv, G["pe_out_hv"])


def test_golden_covariance_operators(oracle):
    q = make_params(nx=60, ny=60)
    assert np.array_equal(oracle.apply_soar(q, G["soar_in"]), G["soar_out"])
    assert np.array_equal(oracle.interpolate_bicubic(q, 2, 3, G["soar_in"]), G["interp_out_2_3"])
    u, v = oracle.geostrophic_balance(q, G["gb_in"])
    assert np.array_equal(u, G["gb_hu"]) and np.array_equal(v, G["gb_hv"])
    qt, offs = oracle.apply_q_half_T(q, 0.7, -1.3, 13, 22)
    assert np.array_equal(qt, G["qT_out"]) and tuple(offs) == tuple(G["qT_offsets"])


def test_golden_grid_and_stream_identity(oracle):
    q = make_params(nx=60, ny=60)
    cells = np.array([oracle.locate_cell(q, x, y) for x, y in G["locate_pts"]])
    assert np.array_equal(cells, G["locate_cells"])
    seeds = [oracle.stream_seed(m, t, i) for m, t, i in
             [(1, 1, 0), (1, 2, 5), (99, 1, 3), (2**63, 7, 2**40)]]
    assert seeds == [int(x) for x in G["stream_seed"]]


def test_philox_known_answers(oracle):
    """Philox4x32-10 known-answer vectors (Salmon et al. SC'11 / Random123 kat_vectors)."""
    assert oracle.philox([0, 0, 0, 0], 0) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    assert oracle.philox([0xffffffff] * 4, 0xffffffffffffffff) == \
        [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert oracle.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                         0x299f31d0a4093822) == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_deterministic_elementary_functions(oracle):
    """The libm-free log/exp/sincos used by the counter-based normals and the alpha solve
    are accurate to a few ulp (their determinism, not accuracy, is the parity contract)."""
    L = oracle.lib
    xs = np.concatenate([np.geomspace(1e-16, 1.0, 2000), np.linspace(0.5, 2.0, 777)])
    for x in xs:
        assert abs(L.orc_det_log(x) - np.log(x)) <= 4e-16 * max(1.0, abs(np.log(x)))
    for x in np.linspace(-40, 5, 3001):
        assert abs(L.orc_det_exp(x) - np.exp(x)) <= 4e-16 * np.exp(x)
    import ctypes as C
    s, c = C.c_double(), C.c_double()
    for u in np.linspace(0, 1, 4001, endpoint=False):
        L.orc_det_sincos2pi(u, C.byref(s), C.byref(c))
        assert abs(s.value - np.sin(2 * np.pi * u)) < 2e-15
        assert abs(c.value - np.cos(2 * np.pi * u)) < 2e-15


def test_philox_normals_moments(oracle):
    """test_stochastic.cpp:59-76 / test_grid.cpp:161-175 on the counter-based stream:
    mean within 4 sigma of 0, variance in [0.99, 1.01] over 1e6 draws."""
    p = make_params(nx=1000, ny=1000, c_omega=1)
    _, _, xi = oracle.philox_draw(p, 1, 0, 0, 0)
    n = xi.size
    assert abs(xi.mean()) <= 4.0 / np.sqrt(n)
    assert 0.99 <= xi.var() <= 1.01
    _, _, xi2 = oracle.philox_draw(p, 1, 0, 0, 0)
    assert np.array_equal(xi, xi2)
    _, _, xi3 = oracle.philox_draw(p, 1, 1, 0, 0)
    assert not np.array_equal(xi, xi3)


def test_philox_offsets_uniform(oracle):
    import ctypes as C
    p = make_params(nx=60, ny=60)
    counts = np.zeros((5, 5), int)
    for d in range(5000):
        a, b = C.c_int32(), C.c_int32()
        oracle.lib.orc_philox_draw(C.byref(p), 1, 3, 0, d, C.byref(a), C.byref(b), None)
        counts[a.value, b.value] += 1
    assert counts.min() > 140 and counts.max() < 260  # 200 expected per cell
