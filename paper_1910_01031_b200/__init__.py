"""B200-native IEWPF hot path (arXiv 1910.01031): ensemble shallow-water forecast,
model-error perturbation, two-stage IEWPF analysis and drifter advection as sm_100a
CUDA kernels behind the C ABI in include/driftcast_gpu.h.

The compute lives in libdriftcast_gpu.so (C++/CUDA). This package only binds it.
"""
from ._lib import DcError, load  # noqa: F401
from .resample import exchange_plan, resample_across_ranks  # noqa: F401
from .ensemble import (Config, Ensemble, comm_unique_id, forecast_error_gathered,  # noqa: F401
                       generate_truth,
                       obs_array, pf_weights, precompute_S, precompute_local_svd, read_obs_file, residual_resample,
                       write_obs_file)

__all__ = ["Config", "Ensemble", "DcError", "load", "obs_array", "precompute_S",
           "precompute_local_svd", "pf_weights", "residual_resample", "write_obs_file",
           "read_obs_file", "generate_truth", "forecast_error_gathered", "comm_unique_id"]
