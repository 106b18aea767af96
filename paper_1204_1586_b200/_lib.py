"""ctypes binding of the C-ABI (include/cpdgpu.h).

The shared library is the product: if it is missing or cannot be loaded this
module raises — there is no CPU fallback behind it.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("CPDGPU_LIB", _PKG / "lib" / "libcpdgpu.so"))

c_i64 = C.c_int64
c_u64 = C.c_uint64
c_dbl_p = C.POINTER(C.c_double)
c_dbl_pp = C.POINTER(c_dbl_p)

HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, c_dbl_p, c_i64, c_i64, c_u64)
# cpdgpu_allreduce_fn: sum `count` doubles of buf across the ranks, in place
ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, c_dbl_p, c_i64)
COMM_ID_BYTES = 128

# name -> (restype, argtypes); mirrors include/cpdgpu.h one to one
SIGNATURES = {
    "cpdgpu_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "cpdgpu_destroy": (C.c_int, [C.c_void_p]),
    "cpdgpu_last_error": (C.c_char_p, [C.c_void_p]),
    "cpdgpu_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cpdgpu_synchronize": (C.c_int, [C.c_void_p]),
    "cpdgpu_set_graphs": (C.c_int, [C.c_void_p, C.c_int]),
    "cpdgpu_set_deterministic": (C.c_int, [C.c_void_p, C.c_int]),
    "cpdgpu_launch_count": (c_u64, [C.c_void_p]),
    "cpdgpu_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "cpdgpu_last_seed_ms": (C.c_int, [C.c_void_p, c_dbl_p]),
    "cpdgpu_last_seed_path": (C.c_int, [C.c_void_p]),
    "cpdgpu_tensor_update": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpdgpu_tensor_upload": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(c_i64), C.POINTER(C.c_void_p)]),
    "cpdgpu_tensor_wrap_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(c_i64), C.POINTER(C.c_void_p)]),
    "cpdgpu_tensor_generate": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(c_i64), C.c_int, c_u64, c_i64, C.POINTER(C.c_void_p)]),
    "cpdgpu_tensor_axpby_kruskal": (C.c_int, [C.c_void_p, C.c_void_p, C.c_double, C.c_double, c_dbl_pp, c_i64]),
    "cpdgpu_tensor_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "cpdgpu_tensor_norm2": (C.c_int, [C.c_void_p, C.c_void_p, c_dbl_p]),
    "cpdgpu_tensor_device_ptr": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "cpdgpu_tensor_free": (C.c_int, [C.c_void_p]),
    "cpdgpu_select_pivot": (C.c_int, [C.c_int, C.POINTER(c_i64), C.POINTER(C.c_int)]),
    "cpdgpu_sort_modes": (C.c_int, [C.c_int, C.POINTER(c_i64), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "cpdgpu_fast_update_order": (C.c_int, [C.c_int, C.POINTER(c_i64), C.POINTER(C.c_int)]),
    "cpdgpu_fast_count_realized": (c_u64, [C.c_int, C.POINTER(c_i64), c_i64, C.c_int]),
    "cpdgpu_predicted_mult_count": (C.c_int, [C.c_int, C.POINTER(c_i64), c_i64, C.c_int, C.c_int, C.POINTER(c_u64)]),
    "cpdgpu_reference_workspace": (C.c_int, [C.c_int, C.POINTER(c_i64), c_i64, C.POINTER(c_i64)]),
    "cpdgpu_device_workspace": (C.c_int, [C.c_void_p, C.POINTER(c_i64), C.POINTER(c_i64)]),
    "cpdgpu_cp_gradient_all": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, c_dbl_pp, C.POINTER(c_u64), C.POINTER(c_i64)]),
    "cpdgpu_cp_gradient_all_hook": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, c_dbl_pp, HOOK, C.c_void_p, C.POINTER(c_i64)]),
    "cpdgpu_cp_gradient_all_device": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, C.c_void_p, C.c_void_p, C.c_int]),
    "cpdgpu_pinv_psd": (C.c_int, [C.c_void_p, c_i64, c_dbl_p, C.c_double, c_dbl_p]),
    "cpdgpu_als_update_mode": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(c_i64), c_i64, c_dbl_p, c_dbl_pp, C.c_int, C.c_double, c_dbl_p]),
    "cpdgpu_uniform01_fill": (C.c_int, [c_u64, c_i64, c_dbl_p]),
    "cpdgpu_cost": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, c_dbl_p]),
    "cpdgpu_tensor_load_tdnb": (C.c_int, [C.c_void_p, C.c_char_p, c_i64, c_i64, C.POINTER(C.c_void_p)]),
    "cpdgpu_tensor_save_tdnb": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p]),
    "cpdgpu_comm_unique_id": (C.c_int, [C.c_void_p]),
    "cpdgpu_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
    "cpdgpu_comm_init_host": (C.c_int, [C.c_void_p, C.c_int, C.c_int, ALLREDUCE, C.c_void_p]),
    "cpdgpu_comm_destroy": (C.c_int, [C.c_void_p]),
    "cpdgpu_slab_bounds": (C.c_int, [c_i64, C.c_int, C.c_int, C.POINTER(c_i64), C.POINTER(c_i64)]),
    "cpdgpu_cp_gradient_all_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(c_i64), c_i64, c_dbl_pp,
                                                 c_dbl_pp, C.POINTER(c_u64)]),
    "cpdgpu_cp_gradient_all_sharded_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(c_i64), c_i64,
                                                        C.c_void_p, C.c_void_p]),
    "cpdgpu_als_sweep_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(c_i64), c_i64, c_dbl_pp,
                                           C.c_double, c_dbl_p, C.POINTER(c_u64)]),
    "cpdgpu_als_run_sharded": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(c_i64), c_i64, c_dbl_pp, C.c_int,
                                         C.c_double, C.c_double, c_dbl_p, c_dbl_p, c_dbl_p, C.POINTER(c_u64),
                                         C.POINTER(C.c_int)]),
    "cpdgpu_mttkrp_direct": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_int, c_dbl_p, C.POINTER(c_u64)]),
    "cpdgpu_mttkrp_direct_device": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, C.c_void_p, C.c_int, C.c_void_p]),
    "cpdgpu_als_sweep_direct": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.POINTER(C.c_int), C.c_int,
                                          C.c_double, C.POINTER(c_u64)]),
    "cpdgpu_mu_sweep": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_double, C.POINTER(c_u64)]),
    "cpdgpu_gd_step": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_double, C.POINTER(c_u64)]),
    "cpdgpu_run_algo": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_int, C.c_int, C.c_int, C.c_double,
                                  C.c_double, C.c_double, C.c_double, c_dbl_p, c_dbl_p, c_dbl_p, C.POINTER(c_u64),
                                  C.POINTER(C.c_int)]),
    "cpdgpu_als_sweep": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_double, c_dbl_p, C.POINTER(c_u64)]),
    "cpdgpu_als_run": (C.c_int, [C.c_void_p, C.c_void_p, c_i64, c_dbl_pp, C.c_int, C.c_double, C.c_double, c_dbl_p, c_dbl_p, c_dbl_p, C.POINTER(c_u64), C.POINTER(C.c_int)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libcpdgpu.so (raises errors.DeviceError when it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise errors.DeviceError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1204_1586_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    # A/B timing of older builds only (tools/ab.sh): tolerate entry points they lack
    partial = os.environ.get("CPDGPU_ABI_PARTIAL") == "1"
    for name, (res, args) in SIGNATURES.items():
        if partial and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, ctx=None) -> None:
    if status == 0:
        return
    msg = ""
    if ctx is not None:
        raw = load().cpdgpu_last_error(ctx)
        msg = raw.decode() if raw else ""
    raise errors.from_status(status, msg)
