"""Generate tests/golden/*.npz from the REFERENCE's own compiled operators.

Run here (where /root/reference exists and oracle/_ref/libdcref.so is built):
    python tests/golden/make_golden.py
The fixtures are small (40x30 / 60x60 grids) and committed, so the CPU restatement
(oracle/liboracle.so) can be pinned against reference outputs on any host, including the
GPU box where /root/reference is absent. Every array is produced by a reference
operator call (oracle/ref_shim.cpp -> proj/include/driftcast/*.hpp).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from checkers import Ref, State, make_params  # noqa: E402


def perturbed(ref, p, seed):
    s = ref.init_double_jet(p)
    y, x = np.mgrid[0:p.ny, 0:p.nx]
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0, 2 * np.pi, 3)
    b = np.sin(2 * np.pi * x / p.nx + ph[0]) * np.cos(4 * np.pi * y / p.ny + ph[1])
    s.eta += (0.03 * b).astype(np.float32)
    s.hv += (3.0 * b).astype(np.float32)
    s.hu += (2.0 * np.cos(2 * np.pi * y / p.ny + ph[2])).astype(np.float32)
    return s


def main():
    ref = Ref()
    out = {}
    # --- model operator (swe.hpp) on a 40x30 grid ---
    p = make_params(nx=40, ny=30)
    jet = ref.init_double_jet(p)
    out["jet_eta"], out["jet_hu"], out["jet_hv"] = jet.eta, jet.hu, jet.hv
    s = perturbed(ref, p, 1)
    out["s0_eta"], out["s0_hu"], out["s0_hv"] = s.eta.copy(), s.hu.copy(), s.hv.copy()
    rhs = ref.flux_rhs(p, s)
    out["rhs_eta"], out["rhs_hu"], out["rhs_hv"] = rhs
    out["cfl_dt"] = np.array(ref.cfl_dt(p, s))
    dts = []
    for _ in range(3):
        dts.append(ref.model_step_dts(p, s))
    out["step3_eta"], out["step3_hu"], out["step3_hv"] = s.eta, s.hu, s.hv
    out["step3_t"] = np.array(s.t)
    out["step3_dts"] = np.concatenate(dts)
    out["step3_nsub"] = np.array([len(d) for d in dts])
    # --- model error (stochastic.hpp) on a 60x60 grid, c_omega = 5 ---
    q = make_params(nx=60, ny=60)
    s2 = perturbed(ref, q, 2)
    out["pe_in_eta"], out["pe_in_hu"], out["pe_in_hv"] = s2.eta.copy(), s2.hu.copy(), s2.hv.copy()
    offs, xi = ref.perturb(q, s2, seed=123, tag=1, index=4, n_draws=3)
    out["pe_offsets"], out["pe_xi"] = offs, xi
    out["pe_out_eta"], out["pe_out_hu"], out["pe_out_hv"] = s2.eta, s2.hu, s2.hv
    nr = (q.nx // 5) * (q.ny // 5)
    rng = np.random.default_rng(3)
    cf = rng.standard_normal(nr)
    out["soar_in"] = cf
    out["soar_out"] = ref.apply_soar(q, 0, 0, cf)
    out["interp_out_2_3"] = ref.interpolate_bicubic(q, 2, 3, cf)
    deta = rng.standard_normal((q.ny, q.nx))
    out["gb_in"] = deta
    out["gb_hu"], out["gb_hv"] = ref.geostrophic_balance(q, deta)
    qt, offq = ref.apply_q_half_T(q, 0.7, -1.3, 13, 22)
    out["qT_out"], out["qT_offsets"] = qt, np.array(offq)
    out["soar_kernel"] = np.array([ref.soar_kernel(q, d) for d in (0.0, 8325.0, 20000.0)])
    # --- grid / rng ---
    lx, ly = q.nx * q.dx, q.ny * q.dy
    pts = np.array([[0.5 * q.dx, 0.5 * q.dy], [(q.nx + 0.5) * q.dx, 3.0], [3331.0, 10.0],
                    [-1.0, -1.0], [lx, ly], [lx * 7.25, -ly * 3.5], [1e-12, ly - 1e-9]])
    out["locate_pts"] = pts
    out["locate_cells"] = np.array([ref.locate_cell(q, x, y) for x, y in pts])
    out["stream_seed"] = np.array([ref.stream_seed(m, t, i) for m, t, i in
                                   [(1, 1, 0), (1, 2, 5), (99, 1, 3), (2**63, 7, 2**40)]],
                                  dtype=np.uint64)
    out["normals_77_1_0"] = ref.normals(77, 1, 0, 16)
    np.savez_compressed(os.path.join(HERE, "reference_ops.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_ops.npz"),
          sum(v.nbytes for v in out.values()) / 1e3, "kB raw")


if __name__ == "__main__":
    main()
