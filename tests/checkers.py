"""ctypes bindings of the CPU checkers under oracle/ (TEST INFRASTRUCTURE ONLY).

- ``Oracle``: this repo's CPU restatement, oracle/liboracle.so (oracle/dc_oracle.cpp).
- ``Ref``: the reference's own operators compiled from /root/reference headers,
  oracle/_ref/libdcref.so (oracle/ref_shim.cpp). Present only where it was built; it
  travels to the GPU box as a built artefact, but tests must skip cleanly without it.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdcref.so")

TAG_MODEL_ERROR, TAG_FILTER, TAG_TRUTH, TAG_OBS_NOISE = 1, 2, 3, 4


class Params(C.Structure):
    """Mirror of orc_params / dc_config (oracle/oracle_api.h, include/driftcast_gpu.h)."""

    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
        ("g", C.c_double), ("f", C.c_double), ("h_eq", C.c_double),
        ("courant", C.c_double), ("limiter_theta", C.c_double), ("model_dt", C.c_double),
        ("q0", C.c_double), ("l0", C.c_double), ("c_omega", C.c_int32), ("c_soar", C.c_int32),
        ("seed", C.c_uint64), ("exact_fp", C.c_int32), ("reserved", C.c_int32),
    ]


def make_params(nx=500, ny=300, dx=2220.0, dy=2220.0, g=9.806, f=1.405e-4, h_eq=230.0,
                courant=0.8, theta=1.3, model_dt=60.0, q0=2.5e-4, c_omega=5, l0=None,
                seed=1, exact_fp=1) -> Params:
    """Paper defaults: L0 = 3/4 coarse spacing."""
    if l0 is None:
        l0 = 0.75 * c_omega * dx
    return Params(nx, ny, dx, dy, g, f, h_eq, courant, theta, model_dt, q0, l0, c_omega, 2,
                  seed, exact_fp, 0)


def fptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def iptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


@dataclass
class State:
    eta: np.ndarray
    hu: np.ndarray
    hv: np.ndarray
    t: float = 0.0

    def copy(self):
        return State(self.eta.copy(), self.hu.copy(), self.hv.copy(), self.t)

    @staticmethod
    def zeros(ny, nx):
        z = lambda: np.zeros((ny, nx), np.float32)  # noqa: E731
        return State(z(), z(), z(), 0.0)


class Oracle:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or build())")
        self.lib = L = C.CDLL(path)
        P = C.POINTER(Params)
        fp, dp, ip = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int32)
        L.orc_last_error.restype = C.c_char_p
        sig = {
            "orc_init_double_jet": [P, fp, fp, fp],
            "orc_model_step": [P, fp, fp, fp, dp, C.c_int, dp, C.c_int, C.POINTER(C.c_int)],
            "orc_flux_rhs": [P, fp, fp, fp, fp, fp, fp],
            "orc_cfl_dt": [P, fp, fp, fp, dp],
            "orc_cfl_internal": [P, fp, fp, fp, dp],
            "orc_apply_soar": [P, dp, dp],
            "orc_interpolate_bicubic": [P, C.c_int, C.c_int, dp, dp],
            "orc_geostrophic_balance": [P, dp, dp, dp],
            "orc_add_q_half": [P, C.c_int, C.c_int, dp, C.c_double, fp, fp, fp],
            "orc_perturb_injected": [P, C.c_int, C.c_int, dp, fp, fp, fp],
            "orc_philox_draw": [P, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, ip, ip, dp],
            "orc_perturb_philox": [P, C.c_uint64, C.c_uint64, fp, fp, fp],
            "orc_perturb_philox_tag": [P, C.c_uint64, C.c_uint64, C.c_uint64, fp, fp, fp],
            "orc_apply_q_half_T": [P, C.c_double, C.c_double, C.c_int, C.c_int, dp, ip, ip],
            "orc_locate_cell": [P, C.c_double, C.c_double, ip, ip],
            "orc_observe_state": [P, fp, fp, fp, C.c_double, C.c_double, dp],
            "orc_observe_mooring": [P, fp, fp, fp, C.c_double, C.c_double, dp],
            "orc_innovations": [P, fp, fp, fp, C.c_int, dp, dp],
            "orc_advect_drifters": [P, fp, fp, fp, C.c_int, C.c_double, dp, ip],
            "orc_precompute_S": [P, C.c_int, C.c_int, C.c_double, C.c_double, dp, dp],
            "orc_local_block": [P, dp, dp],
            "orc_iewpf_assimilate": [P, C.c_int, C.c_uint64, C.c_int, fp, fp, fp, C.c_int, dp,
                                     dp, dp, C.c_uint64, dp, dp, dp, dp],
            "orc_perp_pair": [P, C.c_uint64, C.c_uint64, dp, dp, dp, dp, ip, ip],
            "orc_solve_alpha": [C.c_double, C.c_double, C.c_double, dp, C.POINTER(C.c_int)],
            "orc_lambert_w0": [C.c_double, dp, C.POINTER(C.c_int)],
            "orc_sync_target_beta": [C.c_int, dp, dp, dp, dp],
            "orc_obs_noise": [P, C.c_int, ip, C.c_int, C.c_uint64, C.c_double, C.c_double, dp],
            "orc_observe_drifters": [P, dp, dp, C.c_int, C.c_double, dp, dp],
            "orc_pf_loglik": [P, fp, fp, fp, C.c_int, dp, C.c_double, C.c_double, dp],
            "orc_pf_weights": [dp, C.c_int, dp, dp],
            "orc_residual_resample": [dp, C.c_int, C.c_uint64, C.c_uint64, ip],
            "orc_forecast_error": [P, C.c_int, C.c_int, dp, ip, dp, dp, dp, dp, dp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.orc_stream_seed.argtypes = [C.c_uint64] * 3
        L.orc_stream_seed.restype = C.c_uint64
        L.orc_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_uint32)]
        L.orc_philox4x32_10.restype = None
        for nm in ("orc_det_log", "orc_det_exp"):
            getattr(L, nm).argtypes = [C.c_double]
            getattr(L, nm).restype = C.c_double
        L.orc_det_sincos2pi.argtypes = [C.c_double, dp, dp]
        L.orc_det_sincos2pi.restype = None
        L.orc_nearest_coarse.argtypes = [C.c_int] * 4
        L.orc_nearest_coarse.restype = C.c_int
        L.orc_iewpf_set_mode.argtypes = [C.c_int]
        L.orc_iewpf_set_mode.restype = None
        L.orc_dot_tree.argtypes = [dp, dp, C.c_int]
        L.orc_dot_tree.restype = C.c_double

    def _ck(self, rc):
        if rc:
            raise CheckerError(rc, self.lib.orc_last_error().decode())

    # ---- forecast ----
    def init_double_jet(self, p):
        s = State.zeros(p.ny, p.nx)
        self._ck(self.lib.orc_init_double_jet(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv)))
        return s

    def model_step(self, p, s: State, n_steps=1):
        t = C.c_double(s.t)
        dts = np.zeros(4096, np.float64)
        nsub = C.c_int(0)
        self._ck(self.lib.orc_model_step(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                         C.byref(t), n_steps, dptr(dts), 4096, C.byref(nsub)))
        s.t = t.value
        return dts[: nsub.value].copy()

    def flux_rhs(self, p, s: State):
        out = [np.zeros_like(s.eta) for _ in range(3)]
        self._ck(self.lib.orc_flux_rhs(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                       *[fptr(o) for o in out]))
        return out

    def cfl_dt(self, p, s):
        o = C.c_double()
        self._ck(self.lib.orc_cfl_dt(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv), C.byref(o)))
        return o.value

    def cfl_internal(self, p, s):
        o = C.c_double()
        self._ck(self.lib.orc_cfl_internal(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                           C.byref(o)))
        return o.value

    # ---- model error ----
    def nr(self, p):
        return (p.nx // p.c_omega) * (p.ny // p.c_omega)

    def apply_soar(self, p, x):
        x = np.ascontiguousarray(x, np.float64)
        o = np.zeros_like(x)
        self._ck(self.lib.orc_apply_soar(C.byref(p), dptr(x), dptr(o)))
        return o

    def interpolate_bicubic(self, p, oj, ok, cf):
        cf = np.ascontiguousarray(cf, np.float64)
        o = np.zeros((p.ny, p.nx), np.float64)
        self._ck(self.lib.orc_interpolate_bicubic(C.byref(p), oj, ok, dptr(cf), dptr(o)))
        return o

    def geostrophic_balance(self, p, deta):
        deta = np.ascontiguousarray(deta, np.float64)
        u, v = np.zeros_like(deta), np.zeros_like(deta)
        self._ck(self.lib.orc_geostrophic_balance(C.byref(p), dptr(deta), dptr(u), dptr(v)))
        return u, v

    def add_q_half(self, p, s, oj, ok, coarse, scale=1.0):
        coarse = np.ascontiguousarray(coarse, np.float64)
        self._ck(self.lib.orc_add_q_half(C.byref(p), oj, ok, dptr(coarse), scale, fptr(s.eta),
                                         fptr(s.hu), fptr(s.hv)))

    def perturb_injected(self, p, s, oj, ok, xi):
        xi = np.ascontiguousarray(xi, np.float64)
        self._ck(self.lib.orc_perturb_injected(C.byref(p), oj, ok, dptr(xi), fptr(s.eta),
                                               fptr(s.hu), fptr(s.hv)))

    def philox_draw(self, p, tag, member, substream, draw):
        oj, ok = C.c_int32(), C.c_int32()
        xi = np.zeros(self.nr(p), np.float64)
        self._ck(self.lib.orc_philox_draw(C.byref(p), tag, member, substream, draw,
                                          C.byref(oj), C.byref(ok), dptr(xi)))
        return oj.value, ok.value, xi

    def perturb_philox(self, p, s, member, draw):
        self._ck(self.lib.orc_perturb_philox(C.byref(p), member, draw, fptr(s.eta), fptr(s.hu),
                                             fptr(s.hv)))

    def perturb_philox_tag(self, p, s, tag, member, draw):
        self._ck(self.lib.orc_perturb_philox_tag(C.byref(p), tag, member, draw, fptr(s.eta),
                                                 fptr(s.hu), fptr(s.hv)))

    def apply_q_half_T(self, p, y_hu, y_hv, j, k):
        o = np.zeros(self.nr(p), np.float64)
        oj, ok = C.c_int32(), C.c_int32()
        self._ck(self.lib.orc_apply_q_half_T(C.byref(p), y_hu, y_hv, j, k, dptr(o), C.byref(oj),
                                             C.byref(ok)))
        return o, (oj.value, ok.value)

    def stream_seed(self, master, tag, index):
        return self.lib.orc_stream_seed(master, tag, index)

    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        o = (C.c_uint32 * 4)()
        self.lib.orc_philox4x32_10(c, key, o)
        return list(o)

    # ---- observation ----
    def locate_cell(self, p, x, y):
        j, k = C.c_int32(), C.c_int32()
        self._ck(self.lib.orc_locate_cell(C.byref(p), x, y, C.byref(j), C.byref(k)))
        return j.value, k.value

    def innovations(self, p, s, obs):
        obs = np.ascontiguousarray(obs, np.float64).reshape(-1, 4)
        d = np.zeros((obs.shape[0], 2), np.float64)
        self._ck(self.lib.orc_innovations(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                          obs.shape[0], dptr(obs), dptr(d)))
        return d

    def observe_mooring(self, p, s, x, y):
        o = np.zeros(2, np.float64)
        self._ck(self.lib.orc_observe_mooring(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                              x, y, dptr(o)))
        return o

    def advect_drifters(self, p, s, pos, dt, wind=None):
        n = pos.shape[0]
        self._ck(self.lib.orc_advect_drifters(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                              n, dt, dptr(pos),
                                              iptr(wind) if wind is not None else None))

    # ---- IEWPF ----
    def precompute_S(self, p, j=0, k=0, r_hu=1.0, r_hv=1.0):
        h = np.zeros(4, np.float64)
        S = np.zeros(4, np.float64)
        self._ck(self.lib.orc_precompute_S(C.byref(p), j, k, r_hu, r_hv, dptr(h), dptr(S)))
        return h.reshape(2, 2), S.reshape(2, 2)

    def local_block(self, p, S):
        S = np.ascontiguousarray(S, np.float64).reshape(4)
        b = np.zeros((49, 49), np.float64)
        self._ck(self.lib.orc_local_block(C.byref(p), dptr(S), dptr(b)))
        return b

    def iewpf_assimilate(self, p, eta, hu, hv, obs, S, usig, cycle, member_base=0,
                         n_total=None, c_all=None, zeta_all=None):
        n_local = eta.shape[0]
        n_total = n_local if n_total is None else n_total
        obs = np.ascontiguousarray(obs, np.float64).reshape(-1, 4)
        S = np.ascontiguousarray(S, np.float64).reshape(4)
        usig = np.ascontiguousarray(usig, np.float64).reshape(49 * 49)
        diag = np.zeros((n_local, 5), np.float64)
        dg = np.zeros(2, np.float64)
        self._ck(self.lib.orc_iewpf_assimilate(
            C.byref(p), n_local, member_base, n_total, fptr(eta), fptr(hu), fptr(hv),
            obs.shape[0], dptr(obs), dptr(S), dptr(usig), cycle,
            dptr(c_all) if c_all is not None else None,
            dptr(zeta_all) if zeta_all is not None else None, dptr(diag), dptr(dg)))
        return diag, dg

    def perp_pair(self, p, member, cycle):
        nr = self.nr(p)
        xi, nu = np.zeros(nr), np.zeros(nr)
        g, z = C.c_double(), C.c_double()
        oj, ok = C.c_int32(), C.c_int32()
        self._ck(self.lib.orc_perp_pair(C.byref(p), member, cycle, dptr(xi), dptr(nu),
                                        C.byref(g), C.byref(z), C.byref(oj), C.byref(ok)))
        return xi, nu, g.value, z.value, (oj.value, ok.value)

    def solve_alpha(self, c_star, gamma, n_psi):
        a, cl = C.c_double(), C.c_int()
        self._ck(self.lib.orc_solve_alpha(c_star, gamma, n_psi, C.byref(a), C.byref(cl)))
        return a.value, cl.value

    def lambert_w0(self, x):
        w, cl = C.c_double(), C.c_int()
        self._ck(self.lib.orc_lambert_w0(x, C.byref(w), C.byref(cl)))
        return w.value, cl.value

    def sync_target_beta(self, c, zeta):
        c = np.ascontiguousarray(c, np.float64)
        zeta = np.ascontiguousarray(zeta, np.float64)
        w, b = C.c_double(), C.c_double()
        self._ck(self.lib.orc_sync_target_beta(len(c), dptr(c), dptr(zeta), C.byref(w),
                                               C.byref(b)))
        return w.value, b.value


    # ---- §8(f): twin experiment ----
    def obs_noise(self, p, kind, ids, obs_index, r_hu=1.0, r_hv=1.0):
        ids = np.ascontiguousarray(ids, np.int32).reshape(-1)
        out = np.empty((ids.size, 2), np.float64)
        self._ck(self.lib.orc_obs_noise(C.byref(p), kind, iptr(ids), ids.size, obs_index, r_hu,
                                        r_hv, dptr(out)))
        return out

    def observe_drifters(self, p, prev, cur, dt_obs, eps=None):
        prev = np.ascontiguousarray(prev, np.float64).reshape(-1, 2)
        cur = np.ascontiguousarray(cur, np.float64).reshape(-1, 2)
        e = None if eps is None else np.ascontiguousarray(eps, np.float64).reshape(-1, 2)
        out = np.empty_like(prev)
        self._ck(self.lib.orc_observe_drifters(C.byref(p), dptr(prev), dptr(cur), prev.shape[0],
                                               dt_obs, None if e is None else dptr(e),
                                               dptr(out)))
        return out

    def pf_loglik(self, p, s, obs, r_hu=1.0, r_hv=1.0):
        obs = np.ascontiguousarray(obs, np.float64).reshape(-1, 4)
        out = C.c_double()
        self._ck(self.lib.orc_pf_loglik(C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                                        obs.shape[0], dptr(obs), r_hu, r_hv, C.byref(out)))
        return out.value

    def pf_weights(self, loglik):
        ll = np.ascontiguousarray(loglik, np.float64)
        w = np.empty_like(ll)
        mx = C.c_double()
        rc = self.lib.orc_pf_weights(dptr(ll), ll.size, dptr(w), C.byref(mx))
        return w, mx.value, rc == 0

    def residual_resample(self, w, seed, cycle):
        w = np.ascontiguousarray(w, np.float64)
        out = np.empty(w.size, np.int32)
        self._ck(self.lib.orc_residual_resample(dptr(w), w.size, seed, cycle, iptr(out)))
        return out

    def forecast_error(self, p, pos, wind, truth):
        pos = np.ascontiguousarray(pos, np.float64)
        wind = np.ascontiguousarray(wind, np.int32)
        truth = np.ascontiguousarray(truth, np.float64).reshape(-1, 2)
        n_m, n_d = pos.shape[0], pos.shape[1]
        E, R = C.c_double(), C.c_double()
        ed, rd = np.empty(n_d), np.empty(n_d)
        self._ck(self.lib.orc_forecast_error(C.byref(p), n_m, n_d, dptr(pos), iptr(wind),
                                             dptr(truth), C.byref(E), C.byref(R), dptr(ed),
                                             dptr(rd)))
        return E.value, R.value, ed, rd


class Ref:
    """The reference's own operators (oracle/_ref/libdcref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = L = C.CDLL(path)
        P = C.POINTER(Params)
        fp, dp, ip = C.POINTER(C.c_float), C.POINTER(C.c_double), C.POINTER(C.c_int32)
        E = [C.c_char_p, C.c_int]
        sig = {
            "ref_init_double_jet": [P, fp, fp, fp] + E,
            "ref_model_step": [P, fp, fp, fp, dp, C.c_int] + E,
            "ref_model_step_dts": [P, fp, fp, fp, dp, dp, C.c_int, C.POINTER(C.c_int)] + E,
            "ref_flux_rhs": [P, fp, fp, fp, fp, fp, fp] + E,
            "ref_cfl_dt": [P, fp, fp, fp, dp] + E,
            "ref_perturb": [P, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, fp, fp, fp, ip, dp] + E,
            "ref_add_q_half": [P, C.c_int, C.c_int, dp, C.c_double, fp, fp, fp] + E,
            "ref_apply_soar": [P, C.c_int, C.c_int, dp, dp] + E,
            "ref_interpolate_bicubic": [P, C.c_int, C.c_int, dp, dp] + E,
            "ref_geostrophic_balance": [P, dp, dp, dp] + E,
            "ref_apply_q_half_T": [P, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_int, dp, ip] + E,
            "ref_adjoint_geo_balance": [P, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                        C.c_int, dp] + E,
            "ref_locate_cell": [P, C.c_double, C.c_double, ip, ip] + E,
            "ref_align_coarse_offset": [P, C.c_int, C.c_int, ip, ip] + E,
            "ref_forecast_threads": [P, C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_uint8),
                                     C.c_int, fp, fp, fp, dp] + E,
            "ref_save_snapshot": [P, fp, fp, fp, C.c_double, C.c_char_p] + E,
            "ref_load_snapshot": [P, C.c_char_p, fp, fp, fp, dp] + E,
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = C.c_int
        L.ref_soar_kernel.argtypes = [P, C.c_double]
        L.ref_soar_kernel.restype = C.c_double
        L.ref_stream_seed.argtypes = [C.c_uint64] * 3
        L.ref_stream_seed.restype = C.c_uint64
        L.ref_noise_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, dp]
        L.ref_noise_normals.restype = None
        L.ref_noise_uniform_below.argtypes = [C.c_uint64] * 4 + [C.c_int, C.POINTER(C.c_uint64)]
        L.ref_noise_uniform_below.restype = None

    def _call(self, fn, *args):
        buf = C.create_string_buffer(512)
        rc = fn(*args, buf, 512)
        if rc:
            raise CheckerError(rc, buf.value.decode())

    def save_snapshot(self, p, s, path):
        self._call(self.lib.ref_save_snapshot, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                   s.t, str(path).encode())

    def load_snapshot(self, p, path):
        s = State.zeros(p.ny, p.nx)
        t = C.c_double()
        self._call(self.lib.ref_load_snapshot, C.byref(p), str(path).encode(), fptr(s.eta),
                   fptr(s.hu), fptr(s.hv), C.byref(t))
        s.t = t.value
        return s

    def init_double_jet(self, p):
        s = State.zeros(p.ny, p.nx)
        self._call(self.lib.ref_init_double_jet, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv))
        return s

    def model_step(self, p, s, n_steps=1):
        t = C.c_double(s.t)
        self._call(self.lib.ref_model_step, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                   C.byref(t), n_steps)
        s.t = t.value

    def model_step_dts(self, p, s):
        t = C.c_double(s.t)
        dts = np.zeros(4096)
        n = C.c_int()
        self._call(self.lib.ref_model_step_dts, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                   C.byref(t), dptr(dts), 4096, C.byref(n))
        s.t = t.value
        return dts[: n.value].copy()

    def flux_rhs(self, p, s):
        out = [np.zeros_like(s.eta) for _ in range(3)]
        self._call(self.lib.ref_flux_rhs, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                   *[fptr(o) for o in out])
        return out

    def cfl_dt(self, p, s):
        o = C.c_double()
        self._call(self.lib.ref_cfl_dt, C.byref(p), fptr(s.eta), fptr(s.hu), fptr(s.hv),
                   C.byref(o))
        return o.value

    def perturb(self, p, s, seed, tag, index, n_draws=1):
        nr = (p.nx // p.c_omega) * (p.ny // p.c_omega)
        offs = np.zeros((n_draws, 2), np.int32)
        xi = np.zeros((n_draws, nr), np.float64)
        self._call(self.lib.ref_perturb, C.byref(p), seed, tag, index, n_draws, fptr(s.eta),
                   fptr(s.hu), fptr(s.hv), iptr(offs), dptr(xi))
        return offs, xi

    def add_q_half(self, p, s, oj, ok, coarse, scale=1.0):
        coarse = np.ascontiguousarray(coarse, np.float64)
        self._call(self.lib.ref_add_q_half, C.byref(p), oj, ok, dptr(coarse), scale,
                   fptr(s.eta), fptr(s.hu), fptr(s.hv))

    def apply_soar(self, p, oj, ok, x):
        x = np.ascontiguousarray(x, np.float64)
        o = np.zeros_like(x)
        self._call(self.lib.ref_apply_soar, C.byref(p), oj, ok, dptr(x), dptr(o))
        return o

    def interpolate_bicubic(self, p, oj, ok, cf):
        cf = np.ascontiguousarray(cf, np.float64)
        o = np.zeros((p.ny, p.nx))
        self._call(self.lib.ref_interpolate_bicubic, C.byref(p), oj, ok, dptr(cf), dptr(o))
        return o

    def geostrophic_balance(self, p, deta):
        deta = np.ascontiguousarray(deta, np.float64)
        u, v = np.zeros_like(deta), np.zeros_like(deta)
        self._call(self.lib.ref_geostrophic_balance, C.byref(p), dptr(deta), dptr(u), dptr(v))
        return u, v

    def apply_q_half_T(self, p, y_hu, y_hv, j, k, align=True, oj=0, ok=0):
        nr = (p.nx // p.c_omega) * (p.ny // p.c_omega)
        o = np.zeros(nr)
        offs = np.zeros(2, np.int32)
        self._call(self.lib.ref_apply_q_half_T, C.byref(p), y_hu, y_hv, j, k, int(align), oj, ok,
                   dptr(o), iptr(offs))
        return o, (int(offs[0]), int(offs[1]))

    def locate_cell(self, p, x, y):
        j, k = C.c_int32(), C.c_int32()
        self._call(self.lib.ref_locate_cell, C.byref(p), x, y, C.byref(j), C.byref(k))
        return j.value, k.value

    def align_coarse_offset(self, p, j, k):
        a, b = C.c_int32(), C.c_int32()
        self._call(self.lib.ref_align_coarse_offset, C.byref(p), j, k, C.byref(a), C.byref(b))
        return a.value, b.value

    def soar_kernel(self, p, d):
        return self.lib.ref_soar_kernel(C.byref(p), d)

    def stream_seed(self, m, t, i):
        return self.lib.ref_stream_seed(m, t, i)

    def normals(self, seed, tag, index, n):
        o = np.zeros(n)
        self.lib.ref_noise_normals(seed, tag, index, n, dptr(o))
        return o

    def forecast_threads(self, p, eta, hu, hv, n_steps, perturb_after, n_threads, member_base=0):
        pa = np.ascontiguousarray(perturb_after, np.uint8)
        el = C.c_double()
        self._call(self.lib.ref_forecast_threads, C.byref(p), eta.shape[0], member_base, n_steps,
                   pa.ctypes.data_as(C.POINTER(C.c_uint8)), n_threads, fptr(eta), fptr(hu),
                   fptr(hv), C.byref(el))
        return el.value


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Float equality per element (treats +0 == -0; NaN never equal)."""
    return a.shape == b.shape and bool(np.all(a == b))
