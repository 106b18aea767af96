"""B200-native all-mode CP gradient and fast CP_ALS (arXiv 1204.1586).

The product is libcpdgpu.so (hand-written sm_100a CUDA behind a C-ABI,
include/cpdgpu.h); this package is its host-side mirror of the reference API.
"""
from .errors import (ArgumentError, CpdError, DeviceError, DomainError, IndexError,  # noqa: A004
                     NumericError, ParseError, ShapeError)
from .api import (DIST_NORMAL, DIST_UNIFORM_PM1, F32, F64, Context, CostCounter, DenseTensor,
                  FastStats, RunTrace, SolveOptions, SolveResult, als_sweep_fast, als_update_mode,
                  cp_gradient_all, cp_gradient_all_device, default_context, fast_count_realized,
                  fast_update_order, pinv_psd, run, select_pivot, sort_modes, mttkrp_direct,
                  mttkrp_direct_device, als_sweep_direct, mu_sweep, gd_step, uniform01, random_init,
                  generate_problem, cost, relative_error, cp_gradient_set, Communicator,
                  comm_unique_id, slab_bounds, cp_gradient_all_sharded, cp_gradient_all_sharded_device,
                  als_sweep_sharded, als_run_sharded)

__all__ = [
    "ArgumentError", "CpdError", "DeviceError", "DomainError", "IndexError", "NumericError", "ParseError",
    "ShapeError", "DIST_NORMAL", "DIST_UNIFORM_PM1", "F32", "F64", "Context", "CostCounter",
    "DenseTensor", "FastStats", "RunTrace", "SolveOptions", "SolveResult", "als_sweep_fast",
    "als_update_mode", "cp_gradient_all", "cp_gradient_all_device", "default_context",
    "fast_count_realized", "fast_update_order", "pinv_psd", "run", "select_pivot", "sort_modes",
    "mttkrp_direct", "mttkrp_direct_device", "als_sweep_direct", "mu_sweep", "gd_step", "uniform01",
    "random_init", "generate_problem", "cost", "relative_error", "cp_gradient_set", "Communicator",
    "comm_unique_id", "slab_bounds", "cp_gradient_all_sharded", "cp_gradient_all_sharded_device",
    "als_sweep_sharded", "als_run_sharded",
]
