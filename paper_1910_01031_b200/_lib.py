"""ctypes binding of the C ABI in include/driftcast_gpu.h (libdriftcast_gpu.so).

This is the Python face of the drop-in boundary used by the tests and bench.py; the
library itself is C++/CUDA. There is no CPU fallback: if the shared library is missing
or no GPU is present, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DC_LIB_PATH selects an alternative build of the same library (A/B timing of variants).
LIB_PATH = os.environ.get("DC_LIB_PATH") or os.path.join(HERE, "libdriftcast_gpu.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "driftcast_gpu.h")

(DC_OK, DC_EINVAL, DC_EDRY, DC_ENONFINITE, DC_ERUNAWAY, DC_EALIGN, DC_ECUDA, DC_ESTATE, DC_EIO,
 DC_ECOLLAPSE, DC_ENCCL) = range(11)
DC_NOISE_PHILOX, DC_NOISE_INJECTED = 0, 1

STATUS_NAMES = {
    DC_OK: "DC_OK", DC_EINVAL: "DC_EINVAL", DC_EDRY: "DC_EDRY", DC_ENONFINITE: "DC_ENONFINITE",
    DC_ERUNAWAY: "DC_ERUNAWAY", DC_EALIGN: "DC_EALIGN", DC_ECUDA: "DC_ECUDA",
    DC_ESTATE: "DC_ESTATE", DC_EIO: "DC_EIO", DC_ECOLLAPSE: "DC_ECOLLAPSE", DC_ENCCL: "DC_ENCCL",
}


class DcConfig(C.Structure):
    """dc_config (include/driftcast_gpu.h)."""

    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
        ("g", C.c_double), ("f", C.c_double), ("h_eq", C.c_double),
        ("courant", C.c_double), ("limiter_theta", C.c_double), ("model_dt", C.c_double),
        ("q0", C.c_double), ("l0", C.c_double), ("c_omega", C.c_int32), ("c_soar", C.c_int32),
        ("seed", C.c_uint64), ("exact_fp", C.c_int32), ("reserved", C.c_int32),
    ]


class DcObs(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("y_hu", C.c_double), ("y_hv", C.c_double)]


class DcObsRecord(C.Structure):
    """dc_obs_record: one line of the observation file."""

    _fields_ = [("time", C.c_double), ("kind", C.c_int32), ("id", C.c_int32),
                ("x", C.c_double), ("y", C.c_double), ("y_hu", C.c_double), ("y_hv", C.c_double)]


class DcTruthPlan(C.Structure):
    """dc_truth_plan (generate_truth)."""

    _fields_ = [("duration", C.c_double), ("insert_time", C.c_double),
                ("obs_interval", C.c_double), ("snapshot_interval", C.c_double),
                ("drifters_x", C.c_int32), ("drifters_y", C.c_int32),
                ("moorings_x", C.c_int32), ("moorings_y", C.c_int32),
                ("r_hu", C.c_double), ("r_hv", C.c_double)]


class DcKernelTime(C.Structure):
    """dc_kernel_time: one kernel of a dc_profile_begin / dc_profile_end window."""

    _fields_ = [("name", C.c_char * 40), ("launches", C.c_int64), ("ms", C.c_double),
                ("bytes", C.c_double)]


class DcParticleDiag(C.Structure):
    _fields_ = [("c", C.c_double), ("phi", C.c_double), ("gamma", C.c_double),
                ("zeta", C.c_double), ("alpha", C.c_double)]


# Every symbol the header declares (checked by tests/test_cabi.py without a GPU).
EXPORTS = [
    "dc_create", "dc_destroy", "dc_sync", "dc_last_error", "dc_version",
    "dc_upload_member", "dc_download_member", "dc_upload_all", "dc_download_all",
    "dc_init_double_jet", "dc_step", "dc_flux_rhs", "dc_cfl_dt", "dc_substeps",
    "dc_perturb", "dc_add_q_half", "dc_get_draw_counter", "dc_set_draw_counter",
    "dc_innovations", "dc_observe_mooring", "dc_drifters_set", "dc_drifters_advect",
    "dc_drifters_get", "dc_precompute_S", "dc_precompute_local_svd", "dc_iewpf_begin",
    "dc_iewpf_finish", "dc_iewpf_assimilate", "dc_iewpf_diagnostics", "dc_da_cycle",
    "dc_kernel_launches", "dc_stream", "dc_selftest_math", "dc_counters", "dc_time_stages",
    "dc_drifters_count", "dc_get_config", "dc_save_snapshot", "dc_load_snapshot",
    "dc_checkpoint_save", "dc_checkpoint_load", "dc_obs_noise", "dc_observe_drifters",
    "dc_pf_loglik", "dc_pf_weights", "dc_residual_resample", "dc_resample_members",
    "dc_forecast_error", "dc_obs_file_write", "dc_obs_file_read", "dc_trajectory_write",
    "dc_set_model_error_tag", "dc_generate_truth", "dc_iewpf_set_mode",
    "dc_iewpf_diagnostics_write", "dc_drifters_get_device", "dc_forecast_error_gathered",
    "dc_readback_enqueue", "dc_readback_wait", "dc_member_bytes", "dc_member_export",
    "dc_member_import", "dc_profile_begin", "dc_profile_end", "dc_comm_unique_id",
    "dc_comm_attach", "dc_comm_detach", "dc_comm_info", "dc_drifters_restore",
    "dc_get_model_error_tag", "dc_iewpf_get_mode", "dc_check_guards",
]


class DcError(RuntimeError):
    def __init__(self, status: int, message: str, member=-1, j=-1, k=-1, substep=-1):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message
        self.member, self.j, self.k, self.substep = member, j, k, substep


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libdriftcast_gpu.so and declare every signature. Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA library is required; there is no CPU fallback)")
    L = C.CDLL(path)
    vp, dp, fp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_float), C.POINTER(C.c_int32)
    cfgp = C.POINTER(DcConfig)
    obsp = C.POINTER(DcObs)
    st = C.c_int
    sigs = {
        "dc_create": (st, [cfgp, C.c_int32, C.c_int64, C.c_int32, vp, C.POINTER(vp)]),
        "dc_destroy": (st, [vp]),
        "dc_sync": (st, [vp]),
        "dc_last_error": (C.c_char_p, [vp, ip, ip, ip, ip]),
        "dc_version": (C.c_char_p, []),
        "dc_upload_member": (st, [vp, C.c_int32, fp, fp, fp, C.c_double]),
        "dc_download_member": (st, [vp, C.c_int32, fp, fp, fp, dp]),
        "dc_upload_all": (st, [vp, fp, fp, fp, dp]),
        "dc_download_all": (st, [vp, fp, fp, fp, dp]),
        "dc_init_double_jet": (st, [vp]),
        "dc_step": (st, [vp, C.c_int32]),
        "dc_flux_rhs": (st, [vp, C.c_int32, fp, fp, fp]),
        "dc_cfl_dt": (st, [vp, dp]),
        "dc_substeps": (st, [vp, ip]),
        "dc_perturb": (st, [vp, C.c_int32, ip, dp]),
        "dc_add_q_half": (st, [vp, ip, dp, C.c_double]),
        "dc_get_draw_counter": (st, [vp, C.POINTER(C.c_uint64)]),
        "dc_set_draw_counter": (st, [vp, C.c_uint64]),
        "dc_innovations": (st, [vp, obsp, C.c_int32, dp]),
        "dc_observe_mooring": (st, [vp, C.c_int32, dp, C.c_int32, dp]),
        "dc_drifters_set": (st, [vp, dp, C.c_int32]),
        "dc_drifters_advect": (st, [vp, C.c_double]),
        "dc_drifters_get": (st, [vp, dp, ip]),
        "dc_precompute_S": (st, [cfgp, C.c_double, C.c_double, dp, dp]),
        "dc_precompute_local_svd": (st, [cfgp, dp, dp, dp]),
        "dc_iewpf_begin": (st, [vp, obsp, C.c_int32, dp, dp, C.c_uint64, C.c_int32, vp, C.c_int32]),
        "dc_iewpf_finish": (st, [vp, vp, C.c_int32]),
        "dc_iewpf_assimilate": (st, [vp, obsp, C.c_int32, dp, dp, C.c_uint64]),
        "dc_iewpf_diagnostics": (st, [vp, C.POINTER(DcParticleDiag), dp]),
        "dc_da_cycle": (st, [vp, C.c_int32, obsp, C.c_int32, dp, dp, C.c_uint64]),
        "dc_kernel_launches": (C.c_int64, [vp]),
        "dc_stream": (vp, [vp]),
        "dc_selftest_math": (st, [C.c_int32, C.POINTER(C.c_uint64)]),
        "dc_counters": (st, [vp, C.POINTER(C.c_uint64)]),
        "dc_time_stages": (st, [vp, C.c_int32, dp]),
        "dc_profile_begin": (st, [vp]),
        "dc_comm_unique_id": (st, [C.POINTER(C.c_uint8)]),
        "dc_comm_attach": (st, [vp, C.POINTER(C.c_uint8), C.c_int32, C.c_int32, C.c_int64]),
        "dc_comm_detach": (st, [vp]),
        "dc_drifters_restore": (st, [vp, dp, ip, C.c_int32]),
        "dc_get_model_error_tag": (st, [vp, C.POINTER(C.c_uint64)]),
        "dc_iewpf_get_mode": (st, [vp, ip]),
        "dc_check_guards": (st, [C.c_char_p, C.c_int32, ip]),
        "dc_comm_info": (st, [vp, ip, ip, C.POINTER(C.c_int64)]),
        "dc_profile_end": (st, [vp, C.POINTER(DcKernelTime), C.c_int32, ip]),
        "dc_drifters_count": (st, [vp, ip]),
        "dc_get_config": (st, [vp, cfgp, ip, C.POINTER(C.c_int64)]),
        "dc_save_snapshot": (st, [vp, C.c_int32, C.c_char_p]),
        "dc_load_snapshot": (st, [vp, C.c_int32, C.c_char_p]),
        "dc_checkpoint_save": (st, [vp, C.c_char_p, C.c_uint64]),
        "dc_checkpoint_load": (st, [vp, C.c_char_p, C.POINTER(C.c_uint64)]),
        "dc_obs_noise": (st, [vp, C.c_int32, ip, C.c_int32, C.c_uint64, C.c_double, C.c_double,
                              dp]),
        "dc_observe_drifters": (st, [vp, dp, dp, C.c_int32, C.c_double, dp, dp]),
        "dc_pf_loglik": (st, [vp, obsp, C.c_int32, C.c_double, C.c_double, dp]),
        "dc_pf_weights": (st, [dp, C.c_int32, dp, dp]),
        "dc_residual_resample": (st, [dp, C.c_int32, C.c_uint64, C.c_uint64, ip]),
        "dc_resample_members": (st, [vp, ip]),
        "dc_forecast_error": (st, [vp, dp, dp, dp, dp, dp]),
        "dc_readback_enqueue": (st, [vp, C.c_int32, C.c_int32, dp]),
        "dc_member_bytes": (st, [vp, C.POINTER(C.c_uint64)]),
        "dc_member_export": (st, [vp, C.c_int32, vp]),
        "dc_member_import": (st, [vp, C.c_int32, vp]),
        "dc_readback_wait": (st, [vp, C.c_int32, C.POINTER(DcParticleDiag), dp, dp, ip, dp, dp]),
        "dc_drifters_get_device": (st, [vp, vp, vp]),
        "dc_forecast_error_gathered": (st, [cfgp, C.c_int32, vp, C.c_int32, C.c_int32, vp, vp,
                                            dp, dp, dp, dp, dp]),
        "dc_obs_file_write": (st, [C.c_char_p, C.POINTER(DcObsRecord), C.c_int32, C.c_int32]),
        "dc_obs_file_read": (st, [C.c_char_p, C.POINTER(DcObsRecord), C.c_int32, ip]),
        "dc_trajectory_write": (st, [vp, C.c_char_p, C.c_double, C.c_int32]),
        "dc_set_model_error_tag": (st, [vp, C.c_uint64]),
        "dc_iewpf_set_mode": (st, [vp, C.c_int32]),
        "dc_iewpf_diagnostics_write": (st, [vp, C.c_char_p, C.c_uint64, C.c_int32]),
        "dc_generate_truth": (st, [cfgp, C.POINTER(DcTruthPlan), C.c_char_p, C.c_int32,
                                   C.POINTER(C.c_int64)]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L
