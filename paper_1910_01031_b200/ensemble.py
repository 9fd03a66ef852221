"""Python handle on one GPU ensemble context (the C ABI of include/driftcast_gpu.h).

Method names follow the reference operator surface they replace
(/root/reference/proj/include/driftcast/*.hpp and SPEC.md): ``model_step`` is
Stepper::model_step over every member, ``perturb_state`` is perturb_state, etc.
Host arrays use the reference layout (row-major, j fastest; member-major).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import DcConfig, DcError, DcObs, DcObsRecord, DcParticleDiag


@dataclass
class Config:
    """ModelGrid + PhysParams + SchemeParams + ErrorParams (+ seed): paper defaults
    (§5): 500x300 double jet, dx=dy=2220 m, c_Omega=5,
    L0 = 3/4 coarse spacing, q0 = 2.5e-4."""

    nx: int = 500
    ny: int = 300
    dx: float = 2220.0
    dy: float = 2220.0
    g: float = 9.806
    f: float = 1.405e-4
    h_eq: float = 230.0
    courant: float = 0.8
    limiter_theta: float = 1.3
    model_dt: float = 60.0
    q0: float = 2.5e-4
    l0: float | None = None
    c_omega: int = 5
    seed: int = 1
    exact_fp: bool = True

    def to_c(self) -> DcConfig:
        l0 = self.l0 if self.l0 is not None else 0.75 * self.c_omega * self.dx
        return DcConfig(self.nx, self.ny, self.dx, self.dy, self.g, self.f, self.h_eq,
                        self.courant, self.limiter_theta, self.model_dt, self.q0, l0,
                        self.c_omega, 2, self.seed, 1 if self.exact_fp else 0, 0)

    @property
    def nr(self) -> int:
        return (self.nx // self.c_omega) * (self.ny // self.c_omega)


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def obs_array(obs) -> C.Array:
    """(n,4) array of (x, y, y_hu, y_hv) -> dc_obs[n]."""
    obs = np.ascontiguousarray(obs, np.float64).reshape(-1, 4)
    arr = (DcObs * max(1, obs.shape[0]))()
    C.memmove(arr, obs.ctypes.data, obs.nbytes)
    return arr


class Ensemble:
    """N_e particles of the double-jet shallow-water model resident on one GPU."""

    def __init__(self, cfg: Config, n_members: int, member_base: int = 0, device: int = 0,
                 stream: int | None = None):
        self.L = _lib.load()
        self.cfg = cfg
        self.n = n_members
        self.base = member_base
        self._c = cfg.to_c()
        h = C.c_void_p()
        rc = self.L.dc_create(C.byref(self._c), n_members, member_base, device,
                              C.c_void_p(stream) if stream else None, C.byref(h))
        if rc:
            raise DcError(rc, "dc_create failed (see stderr)")
        self.h = h

    # ---- plumbing ----
    def _ck(self, rc):
        if rc:
            m, j, k, s = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            msg = self.L.dc_last_error(self.h, C.byref(m), C.byref(j), C.byref(k), C.byref(s))
            raise DcError(rc, msg.decode(), m.value, j.value, k.value, s.value)

    def close(self):
        if getattr(self, "h", None):
            self.L.dc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self._ck(self.L.dc_sync(self.h))

    @property
    def stream(self) -> int:
        return self.L.dc_stream(self.h) or 0

    def kernel_launches(self) -> int:
        return int(self.L.dc_kernel_launches(self.h))

    def counters(self):
        """(kernels launched, member-substeps, substep-loop iterations) since creation."""
        out = (C.c_uint64 * 3)()
        self._ck(self.L.dc_counters(self.h, out))
        return int(out[0]), int(out[1]), int(out[2])

    def time_stages(self, n_substeps=7):
        """Mean CUDA-event duration (ms) of the stage-1 / stage-2 SWE kernels."""
        out = np.zeros(2, np.float64)
        self._ck(self.L.dc_time_stages(self.h, n_substeps, _d(out)))
        return float(out[0]), float(out[1])

    # ---- multi-GPU (dc_comm_*: NCCL inside the library) ----
    def comm_attach(self, nccl_id: bytes, rank: int, world: int, n_total: int):
        """Join the ranks' NCCL communicator (collective). nccl_id: the 128 bytes of
        comm_unique_id() made on rank 0 and broadcast by the host driver."""
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
        self._ck(self.L.dc_comm_attach(self.h, buf, rank, world, n_total))

    def comm_detach(self):
        self._ck(self.L.dc_comm_detach(self.h))

    def comm_info(self):
        r, w, n = C.c_int32(), C.c_int32(), C.c_int64()
        self._ck(self.L.dc_comm_info(self.h, C.byref(r), C.byref(w), C.byref(n)))
        return r.value, w.value, n.value

    def profile_begin(self):
        """Open a per-kernel profile window (dc_profile_begin): every kernel launched by
        this thread until profile_end is timed with CUDA events on its stream."""
        self._ck(self.L.dc_profile_begin(self.h))

    def profile_end(self):
        """Close the window: [(kernel, launches, total ms, total algorithmic bytes)] in
        first-launch order."""
        cap = 64
        out = (_lib.DcKernelTime * cap)()
        n = C.c_int32()
        self._ck(self.L.dc_profile_end(self.h, out, cap, C.byref(n)))
        return [(out[i].name.decode(), int(out[i].launches), float(out[i].ms), float(out[i].bytes))
                for i in range(min(n.value, cap))]

    # ---- state I/O ----
    def upload(self, eta, hu, hv, t=None):
        eta, hu, hv = (np.ascontiguousarray(a, np.float32) for a in (eta, hu, hv))
        tt = None if t is None else np.ascontiguousarray(np.broadcast_to(t, (self.n,)), np.float64)
        self._ck(self.L.dc_upload_all(self.h, _f(eta), _f(hu), _f(hv),
                                      _d(tt) if tt is not None else None))
        self.sync()

    def upload_member(self, m, eta, hu, hv, t=0.0):
        eta, hu, hv = (np.ascontiguousarray(a, np.float32) for a in (eta, hu, hv))
        self._ck(self.L.dc_upload_member(self.h, m, _f(eta), _f(hu), _f(hv), t))

    def download(self, strict=True):
        """All members' fields and times. A member that failed (dry cell, non-finite
        state, runaway substeps) raises DcError unless strict=False, which returns every
        member's fields as they are -- the failed ones stopped where they failed."""
        shp = (self.n, self.cfg.ny, self.cfg.nx)
        e, u, v = (np.empty(shp, np.float32) for _ in range(3))
        t = np.empty(self.n, np.float64)
        rc = self.L.dc_download_all(self.h, _f(e), _f(u), _f(v), _d(t))
        if rc and (strict or rc not in (_lib.DC_EDRY, _lib.DC_ENONFINITE, _lib.DC_ERUNAWAY)):
            self._ck(rc)
        return e, u, v, t

    def download_member(self, m):
        shp = (self.cfg.ny, self.cfg.nx)
        e, u, v = (np.empty(shp, np.float32) for _ in range(3))
        t = C.c_double()
        self._ck(self.L.dc_download_member(self.h, m, _f(e), _f(u), _f(v), C.byref(t)))
        return e, u, v, t.value

    # ---- model operator ----
    def init_double_jet(self):
        self._ck(self.L.dc_init_double_jet(self.h))

    def model_step(self, n_steps: int = 1):
        self._ck(self.L.dc_step(self.h, n_steps))

    def flux_rhs(self, m=0):
        shp = (self.cfg.ny, self.cfg.nx)
        out = [np.empty(shp, np.float32) for _ in range(3)]
        self._ck(self.L.dc_flux_rhs(self.h, m, *[_f(o) for o in out]))
        return out

    def cfl_dt(self):
        out = np.empty(self.n, np.float64)
        self._ck(self.L.dc_cfl_dt(self.h, _d(out)))
        return out

    def substeps(self):
        out = np.empty(self.n, np.int32)
        self._ck(self.L.dc_substeps(self.h, _i(out)))
        return out

    # ---- model error ----
    def perturb_state(self, offsets=None, xi=None):
        """perturb_state on every member: Philox draw, or injected (offsets, xi)."""
        if offsets is None:
            self._ck(self.L.dc_perturb(self.h, _lib.DC_NOISE_PHILOX, None, None))
        else:
            offsets = np.ascontiguousarray(offsets, np.int32).reshape(self.n, 2)
            xi = np.ascontiguousarray(xi, np.float64).reshape(self.n, self.cfg.nr)
            self._ck(self.L.dc_perturb(self.h, _lib.DC_NOISE_INJECTED, _i(offsets), _d(xi)))

    def add_q_half(self, offsets, coarse, scale=1.0):
        offsets = np.ascontiguousarray(offsets, np.int32).reshape(self.n, 2)
        coarse = np.ascontiguousarray(coarse, np.float64).reshape(self.n, self.cfg.nr)
        self._ck(self.L.dc_add_q_half(self.h, _i(offsets), _d(coarse), scale))

    @property
    def draw_counter(self) -> int:
        v = C.c_uint64()
        self._ck(self.L.dc_get_draw_counter(self.h, C.byref(v)))
        return v.value

    @draw_counter.setter
    def draw_counter(self, v: int):
        self._ck(self.L.dc_set_draw_counter(self.h, v))

    def set_model_error_tag(self, tag: int):
        """1: model_error (ensemble), 3: truth_model_error (twin-experiment truth)."""
        self._ck(self.L.dc_set_model_error_tag(self.h, tag))

    # ---- observation system ----
    def innovations(self, obs):
        arr = obs_array(obs)
        n = len(np.asarray(obs).reshape(-1, 4))
        out = np.empty((self.n, n, 2), np.float64)
        self._ck(self.L.dc_innovations(self.h, arr, n, _d(out)))
        return out

    def observe_mooring(self, m, xy):
        xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
        out = np.empty((xy.shape[0], 2), np.float64)
        self._ck(self.L.dc_observe_mooring(self.h, m, _d(xy), xy.shape[0], _d(out)))
        return out

    def drifters_set(self, pos):
        pos = np.ascontiguousarray(pos, np.float64)
        if pos.ndim == 2:
            pos = np.ascontiguousarray(np.broadcast_to(pos, (self.n,) + pos.shape))
        self._ck(self.L.dc_drifters_set(self.h, _d(pos), pos.shape[1]))

    @property
    def n_drifters(self) -> int:
        """drifter copies per member (set by drifters_set or a checkpoint load)."""
        n = C.c_int32()
        rc = self.L.dc_drifters_count(self.h, C.byref(n))
        return n.value if rc == 0 else 0

    def advect_drifters(self, dt):
        self._ck(self.L.dc_drifters_advect(self.h, dt))

    def drifters_get(self):
        pos = np.empty((self.n, self.n_drifters, 2), np.float64)
        wind = np.empty((self.n, self.n_drifters, 2), np.int32)
        self._ck(self.L.dc_drifters_get(self.h, _d(pos), _i(wind)))
        return pos, wind

    # ---- snapshots / checkpoints (state.hpp:43-116) ----
    def save_snapshot(self, m, path):
        self._ck(self.L.dc_save_snapshot(self.h, m, str(path).encode()))

    def load_snapshot(self, m, path):
        self._ck(self.L.dc_load_snapshot(self.h, m, str(path).encode()))

    def checkpoint_save(self, directory, filter_cycle=0):
        self._ck(self.L.dc_checkpoint_save(self.h, str(directory).encode(), filter_cycle))

    def checkpoint_load(self, directory) -> int:
        c = C.c_uint64(0)
        self._ck(self.L.dc_checkpoint_load(self.h, str(directory).encode(), C.byref(c)))
        return int(c.value)

    # ---- twin experiment ----
    def obs_noise(self, kind, ids, obs_index, r_hu=1.0, r_hv=1.0):
        """eps ~ N(0, diag(r_hu, r_hv)) for platforms (kind, ids) at observation index."""
        ids = np.ascontiguousarray(ids, np.int32).reshape(-1)
        out = np.empty((ids.size, 2), np.float64)
        self._ck(self.L.dc_obs_noise(self.h, kind, _i(ids), ids.size, obs_index, r_hu, r_hv,
                                     _d(out)))
        return out

    def observe_drifters(self, prev_xy, cur_xy, dt_obs, eps=None):
        p = np.ascontiguousarray(prev_xy, np.float64).reshape(-1, 2)
        c = np.ascontiguousarray(cur_xy, np.float64).reshape(-1, 2)
        e = None if eps is None else np.ascontiguousarray(eps, np.float64).reshape(-1, 2)
        out = np.empty_like(p)
        self._ck(self.L.dc_observe_drifters(self.h, _d(p), _d(c), p.shape[0], dt_obs,
                                            None if e is None else _d(e), _d(out)))
        return out

    def pf_loglik(self, obs, r_hu=1.0, r_hv=1.0):
        arr = obs_array(obs)
        n = len(np.asarray(obs).reshape(-1, 4))
        out = np.empty(self.n, np.float64)
        self._ck(self.L.dc_pf_loglik(self.h, arr, n, r_hu, r_hv, _d(out)))
        return out

    def resample_members(self, idx):
        idx = np.ascontiguousarray(idx, np.int32).reshape(self.n)
        self._ck(self.L.dc_resample_members(self.h, _i(idx)))

    def forecast_error(self, truth_xy):
        t = np.ascontiguousarray(truth_xy, np.float64).reshape(-1, 2)
        E, R = C.c_double(0), C.c_double(0)
        ed = np.empty(t.shape[0], np.float64)
        rd = np.empty(t.shape[0], np.float64)
        self._ck(self.L.dc_forecast_error(self.h, _d(t), C.byref(E), C.byref(R), _d(ed), _d(rd)))
        return E.value, R.value, ed, rd

    # ---- member state export / import (resampling across ranks) ----
    def member_bytes(self) -> int:
        v = C.c_uint64(0)
        self._ck(self.L.dc_member_bytes(self.h, C.byref(v)))
        return int(v.value)

    def member_export(self, m, dev_ptr):
        """Stream-ordered copy of member m's state into a device buffer of member_bytes()."""
        self._ck(self.L.dc_member_export(self.h, m, C.c_void_p(dev_ptr)))

    def member_import(self, m, dev_ptr):
        self._ck(self.L.dc_member_import(self.h, m, C.c_void_p(dev_ptr)))

    def drifters_to_device(self, pos_ptr, wind_ptr):
        """Stream-ordered copy of the drifter ensemble into device buffers
        ([n][n_d][2] fp64 / int32), e.g. torch tensors feeding an NCCL gather."""
        self._ck(self.L.dc_drifters_get_device(self.h, C.c_void_p(pos_ptr), C.c_void_p(wind_ptr)))

    def trajectory_write(self, path, time, append=True):
        self._ck(self.L.dc_trajectory_write(self.h, str(path).encode(), time, int(append)))

    # ---- IEWPF ----
    def iewpf_set_mode(self, one_stage: bool):
        """one-stage IEWPF (target max c_i) instead of the two-stage default."""
        self._ck(self.L.dc_iewpf_set_mode(self.h, 1 if one_stage else 0))

    def iewpf_assimilate(self, obs, S, usig, cycle):
        arr = obs_array(obs)
        n = len(np.asarray(obs).reshape(-1, 4))
        S = np.ascontiguousarray(S, np.float64).reshape(4)
        usig = np.ascontiguousarray(usig, np.float64).reshape(49 * 49)
        self._ck(self.L.dc_iewpf_assimilate(self.h, arr, n, _d(S), _d(usig), cycle))

    def iewpf_begin(self, obs, S, usig, cycle, n_total, cz_out=None, cz_ptr=None):
        """Stages 1-3; writes this slice's (c, zeta) to a host array or a device pointer."""
        arr = obs_array(obs)
        n = len(np.asarray(obs).reshape(-1, 4))
        S = np.ascontiguousarray(S, np.float64).reshape(4)
        usig = np.ascontiguousarray(usig, np.float64).reshape(49 * 49)
        if cz_ptr is not None:
            self._ck(self.L.dc_iewpf_begin(self.h, arr, n, _d(S), _d(usig), cycle, n_total,
                                           C.c_void_p(cz_ptr), 1))
            return None
        out = np.empty((self.n, 2), np.float64) if cz_out is None else cz_out
        self._ck(self.L.dc_iewpf_begin(self.h, arr, n, _d(S), _d(usig), cycle, n_total,
                                       out.ctypes.data_as(C.c_void_p), 0))
        return out

    def iewpf_finish(self, cz_all=None, cz_ptr=None):
        if cz_ptr is not None:
            self._ck(self.L.dc_iewpf_finish(self.h, C.c_void_p(cz_ptr), 1))
        else:
            cz = np.ascontiguousarray(cz_all, np.float64)
            self._ck(self.L.dc_iewpf_finish(self.h, cz.ctypes.data_as(C.c_void_p), 0))

    def iewpf_diagnostics(self):
        d = (DcParticleDiag * self.n)()
        wb = np.empty(2, np.float64)
        self._ck(self.L.dc_iewpf_diagnostics(self.h, d, _d(wb)))
        arr = np.array([[x.c, x.phi, x.gamma, x.zeta, x.alpha] for x in d], np.float64)
        return arr, wb

    # ---- pipelined per-cycle readback (dc_readback_enqueue / dc_readback_wait) ----
    def readback_enqueue(self, slot, diag=True, drifters=True, truth_xy=None):
        """Queue copies of the outputs of the work queued so far into pinned slot 0 or 1
        (particle diagnostics, drifter ensemble, forecast_error vs truth_xy); returns at
        once. Read them with readback_wait(slot), e.g. after queueing the next cycle."""
        what = (1 if diag else 0) | (2 if drifters else 0) | (4 if truth_xy is not None else 0)
        t = None if truth_xy is None else np.ascontiguousarray(truth_xy, np.float64).reshape(-1, 2)
        self._ck(self.L.dc_readback_enqueue(self.h, slot, what, None if t is None else _d(t)))
        if not hasattr(self, "_rb_what"):
            self._rb_what = {}
        self._rb_what[slot] = what

    def readback_wait(self, slot):
        """Block until slot's copies landed; returns dict(diag [n,5] (c, phi, gamma, zeta,
        alpha), w_beta, pos, wind, E, RMSE) with None for what was not queued."""
        what = getattr(self, "_rb_what", {}).pop(slot, 0)
        diag = np.empty((self.n, 5), np.float64) if what & 1 else None
        wb = np.empty(2, np.float64) if what & 1 else None
        pos = wind = None
        if what & 2:
            pos = np.empty((self.n, self.n_drifters, 2), np.float64)
            wind = np.empty((self.n, self.n_drifters, 2), np.int32)
        E, R = C.c_double(0), C.c_double(0)
        self._ck(self.L.dc_readback_wait(
            self.h, slot, None if diag is None else diag.ctypes.data_as(C.POINTER(DcParticleDiag)),
            None if wb is None else _d(wb), None if pos is None else _d(pos),
            None if wind is None else _i(wind), C.byref(E), C.byref(R)))
        fe = bool(what & 4)
        return {"diag": diag, "w_beta": wb, "pos": pos, "wind": wind,
                "E": E.value if fe else None, "RMSE": R.value if fe else None}

    def iewpf_diagnostics_write(self, path, cycle, append=True):
        self._ck(self.L.dc_iewpf_diagnostics_write(self.h, str(path).encode(), cycle,
                                                   int(append)))

    def da_cycle(self, n_steps, obs, S, usig, cycle):
        arr = obs_array(obs)
        n = len(np.asarray(obs).reshape(-1, 4))
        S = np.ascontiguousarray(S, np.float64).reshape(4)
        usig = np.ascontiguousarray(usig, np.float64).reshape(49 * 49)
        self._ck(self.L.dc_da_cycle(self.h, n_steps, arr, n, _d(S), _d(usig), cycle))


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for dc_comm_attach; made on rank 0."""
    L = _lib.load()
    buf = (C.c_uint8 * 128)()
    rc = L.dc_comm_unique_id(buf)
    if rc:
        raise DcError(rc, "dc_comm_unique_id failed (NCCL not loadable?)")
    return bytes(buf)


def forecast_error_gathered(cfg: Config, n_members, n_drifters, pos_ptr, wind_ptr, truth_xy,
                            device=0, stream=None):
    """forecast_error over drifter ensembles gathered (member-id order) into device memory
    from several ranks: returns (E, RMSE, E_d, RMSE_d) like Ensemble.forecast_error."""
    L = _lib.load()
    c = cfg.to_c()
    t = np.ascontiguousarray(truth_xy, np.float64).reshape(-1, 2)
    if t.shape[0] != n_drifters:
        raise ValueError("truth_xy must hold one position per drifter")
    E, R = C.c_double(0), C.c_double(0)
    ed = np.empty(n_drifters, np.float64)
    rd = np.empty(n_drifters, np.float64)
    rc = L.dc_forecast_error_gathered(C.byref(c), device, C.c_void_p(stream) if stream else None,
                                      n_members, n_drifters, C.c_void_p(pos_ptr),
                                      C.c_void_p(wind_ptr), _d(t), C.byref(E), C.byref(R),
                                      _d(ed), _d(rd))
    if rc:
        raise DcError(rc, "dc_forecast_error_gathered failed")
    return E.value, R.value, ed, rd


def precompute_S(cfg: Config, r_hu=1.0, r_hv=1.0):
    """precompute_S: returns (HQH^T, S) as 2x2 arrays."""
    L = _lib.load()
    c = cfg.to_c()
    h = np.empty(4, np.float64)
    s = np.empty(4, np.float64)
    rc = L.dc_precompute_S(C.byref(c), r_hu, r_hv, _d(h), _d(s))
    if rc:
        raise DcError(rc, "dc_precompute_S failed")
    return h.reshape(2, 2), s.reshape(2, 2)


def precompute_local_svd(cfg: Config, S):
    """precompute_local_svd: returns (block, U Sigma^{1/2}) 49x49."""
    L = _lib.load()
    c = cfg.to_c()
    S = np.ascontiguousarray(S, np.float64).reshape(4)
    b = np.empty((49, 49), np.float64)
    u = np.empty((49, 49), np.float64)
    rc = L.dc_precompute_local_svd(C.byref(c), _d(S), _d(b), _d(u))
    if rc:
        raise DcError(rc, "dc_precompute_local_svd failed")
    return b, u


def pf_weights(loglik, strict=True):
    """standard_pf_weights normalisation: returns (w, max_loglik).
    Every exp(loglik) underflowing is the spec's "ensemble collapse": raised as
    DcError(DC_ECOLLAPSE) when strict, else the max-shifted weights are returned anyway
    (what the collapse experiment counts)."""
    L = _lib.load()
    ll = np.ascontiguousarray(loglik, np.float64).reshape(-1)
    w = np.empty_like(ll)
    mx = C.c_double(0)
    rc = L.dc_pf_weights(_d(ll), ll.size, _d(w), C.byref(mx))
    if rc and (strict or rc != _lib.DC_ECOLLAPSE):
        raise DcError(rc, f"ensemble collapse (max log-weight {mx.value:.6g})")
    return w, mx.value


def residual_resample(w, seed, cycle):
    """residual_resample: ascending index multiset of len(w)."""
    L = _lib.load()
    w = np.ascontiguousarray(w, np.float64).reshape(-1)
    out = np.empty(w.size, np.int32)
    rc = L.dc_residual_resample(_d(w), w.size, seed, cycle, _i(out))
    if rc:
        raise DcError(rc, "residual_resample: invalid weights")
    return out


def write_obs_file(path, records, append=False):
    """records: iterable of (time, kind, id, x, y, y_hu, y_hv); kind 0 drifter, 1 mooring."""
    L = _lib.load()
    recs = list(records)
    arr = (DcObsRecord * max(1, len(recs)))()
    for i, r in enumerate(recs):
        arr[i] = DcObsRecord(float(r[0]), int(r[1]), int(r[2]), *[float(v) for v in r[3:7]])
    rc = L.dc_obs_file_write(str(path).encode(), arr, len(recs), int(append))
    if rc:
        raise DcError(rc, f"cannot write {path}")


def read_obs_file(path):
    """-> list of (time, kind, id, x, y, y_hu, y_hv)."""
    L = _lib.load()
    n = C.c_int32(0)
    rc = L.dc_obs_file_read(str(path).encode(), None, 0, C.byref(n))
    if rc:
        raise DcError(rc, f"cannot read {path}")
    arr = (DcObsRecord * max(1, n.value))()
    rc = L.dc_obs_file_read(str(path).encode(), arr, n.value, C.byref(n))
    if rc:
        raise DcError(rc, f"cannot read {path}")
    return [(r.time, r.kind, r.id, r.x, r.y, r.y_hu, r.y_hv) for r in arr[:n.value]]


def generate_truth(cfg: Config, out_dir, duration, insert_time=0.0, obs_interval=300.0,
                   snapshot_interval=0.0, drifters=(8, 8), moorings=(0, 0), r=(1.0, 1.0),
                   device=0):
    """generate_truth on the GPU: writes out_dir/observations.txt and
    out_dir/truth_<t>.dcst; returns the number of observation records."""
    import os
    from ._lib import DcTruthPlan
    L = _lib.load()
    os.makedirs(out_dir, exist_ok=True)
    plan = DcTruthPlan(duration, insert_time, obs_interval, snapshot_interval, drifters[0],
                       drifters[1], moorings[0], moorings[1], r[0], r[1])
    n = C.c_int64(0)
    c = cfg.to_c()
    rc = L.dc_generate_truth(C.byref(c), C.byref(plan), str(out_dir).encode(), device,
                             C.byref(n))
    if rc:
        raise DcError(rc, "generate_truth failed")
    return int(n.value)
