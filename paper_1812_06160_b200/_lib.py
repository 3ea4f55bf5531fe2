"""ctypes binding of libjv.so, the C-ABI declared in include/jv.h.

The shared library is built in-tree by __graft_entry__.build() (nvcc, sm_100a).
There is no fallback: if the library or a CUDA device is missing, every
hot-path call raises BackendUnavailable.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint32, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JV_LIB") or os.path.join(_HERE, "libjv.so")  # JV_LIB: diagnostic builds


class BackendUnavailable(RuntimeError):
    """libjv.so or the CUDA device it needs is missing."""


_P = c_void_p  # device pointer
_I32P = POINTER(c_int32)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "jv_last_error": [],
    "jv_version": [],
    "jv_host_register": [_P, c_int64],
    "jv_host_unregister": [_P],
    "jv_memcpy_async": [_P, _P, c_int64, c_int, _P],
    "jv_device_info": [c_int, _I32P, _I32P],
    "jv_reset_row": [_P, _P],
    "jv_status": [_I32P],
    "jv_set_spin_limit": [ctypes.c_uint],
    "jv_set_backoff": [ctypes.c_uint],
    "jv_set_gate": [ctypes.c_uint],
    "jv_set_poll": [ctypes.c_uint],
    "jv_set_sfp_group": [ctypes.c_uint],
    "jv_set_solve_staged": [ctypes.c_uint],
    "jv_set_trace": [_P, ctypes.c_longlong],
    "jv_test_ddiv": [c_int32, _P, _P, _P, _P],
    "jv_spmv_tile": [],
    "jv_set_spmv_impl": [c_int],
    "jv_spmv_impl_for": [c_int32, _P],
    "jv_spmv_plan": [c_int32, c_int32, _P, _P, _P],
    "jv_spmv": [c_int32, c_int32, _P, _P, _P, _P, _P, _P, _P],
    "jv_spmv_rows": [c_int32, c_int32, _P, _P, _P, _P, _P, _P, _P, _P],
    "jv_gather": [c_int32, _P, _P, _P, _P],
    "jv_levels": [c_int, c_int32, _P, _P, _P, _P, c_uint32, _I32P, _P],
    "jv_level_sort": [c_int32, c_int32, _P, _P, _P, _P],
    "jv_partition": [c_int32, c_int32, _P, _P, _P, c_int32, c_double, c_int, _I32P, _I32P, _P],
    "jv_transpose_pattern": [c_int32, _P, _P, _P, _P, _P, _P],
    "jv_sym_lower": [c_int32, _P, _P, _P, _P, c_int, _P, _P, POINTER(c_int64), _P],
    "jv_permute_symmetric": [c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "jv_check_diagonal": [c_int32, _P, _P, _P, _P],
    "jv_iluk1_pattern": [c_int32, _P, _P, _P, _P, _P, POINTER(c_int64), _P],
    "jv_iluk_round": [c_int32, _P, _P, _P, c_int32, _P, _P, _P, POINTER(c_int64), _P],
    "jv_assemble": [c_int32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "jv_row_norms": [c_int32, _P, _P, c_double, _P, _P],
    "jv_rcm_host": [c_int32, _P, _P, _P],
    "jv_rcm_device": [c_int32, _P, _P, _P, c_int32, _I32P, _P],
    "jv_iluk_host": [c_int32, _P, _P, c_int32, POINTER(_I32P), POINTER(_I32P), POINTER(_I32P)],
    "jv_free_host": [c_void_p],
    "jv_factor": [c_int32, _P, _P, _P, _P, _P, c_double, c_int, _P, _P, c_int32, c_int32, _P,
                  c_uint32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "jv_elim_lists": [c_int32, _P, _P, _P, c_int, c_int64, _P, _P, _P, _P, POINTER(c_int64), _P],
    "jv_solve": [c_int, c_int32, _P, _P, _P, _P, _P, _P, c_int32, _P, _P, _P, c_uint32, _P, _P],
    "jv_check_zero_diag": [c_int32, _P, _P, _P, _P],
    "jv_solve_level": [c_int, _P, _P, _P, _P, _P, c_int32, c_int32, _P, _P, _P],
    "jv_build_batches": [c_int32, _P, _P, _I32P, _P],
    "jv_build_schedule": [c_int32, _P, _P, c_int32, _P, _P, _I32P, _P],
    "jv_hub_plan_host": [c_int32, c_int32, _P, _P, _P, _P, _P, POINTER(c_int64), _P,
                         POINTER(c_int64)],
    "jv_dot_workspace": [],
    "jv_dot": [c_int64, _P, _P, _P, _P, c_int, _P],
    "jv_axpy": [c_int64, c_double, _P, c_double, _P, _P, _P],
    "jv_xpby": [c_int64, _P, c_double, _P, _P],
    "jv_scale": [c_int64, c_double, _P, _P, _P],
    "jv_pcg_update": [c_int64, c_double, _P, _P, _P, _P, _P, _P, _P],
    "jv_build_schedule_n": [c_int32, _P, _P, c_int32, c_int32, _P, _P, _P, _I32P, _P],
    "jv_classify_factor": [c_int32, _P, _P, _P, c_int, _P, _P],
    "jv_classify_solve": [c_int, c_int32, _P, _P, _P, _P],
    "jv_region_partition_host": [c_int32, _P, _P, _P, c_int32, c_int32, c_int32, _P],
    "jv_rstream_build": [c_int32, c_int32, _P, _P, _P, _P, c_int32, c_int32, c_int64, c_int32, _P],
    "jv_rstream_export": [c_int64, _P, _P, _P, _P, _P],
    "jv_pack_values": [c_int64, _P, _P, _P, _P],
    "jv_pack_values2": [c_int64, _P, _P, _P, c_int64, _P, _P, _P, _P, _P],
    "jv_region_smem_fixed": [c_int32, c_int32],
    "jv_region_run": [c_int32, c_int32, c_int32, _P, _P, _P, c_int32, c_int32, c_int32, c_int32, c_int32,
                      c_int32, _P, _P, _P, _P, _P, c_double, _P, c_uint32, _P, _P],
    "jv_region_threads": [],
    "jv_set_region_flags": [ctypes.c_uint],
    "jv_tail_plan_build": [c_int32, c_int32, _P, _P, _P, c_int, _P],
    "jv_tail_plan_info": [c_int64, POINTER(c_int64)],
    "jv_tail_upper": [c_int64, _P, _P, _P, _P, c_double, _P],
    "jv_tail_corner": [c_int64, _P, _P, _P, _P, _P],
    "jv_tail_plan_free": [c_int64],
    "jv_scatter": [c_int64, _P, _P, _P, _P],
    "jv_hop_latency": [c_int32, POINTER(c_double)],
    "jv_solve_small_bytes": [c_int, c_int32, c_int32, c_int64],
    "jv_solve_small_max": [],
    "jv_solve_small": [c_int, c_int32, _P, _P, _P, _P, _P, _P, c_int32, _P, c_int64, c_int32, _P, _P, _P],
    "jv_cta_max_rows": [],
    "jv_cta_plan_build": [c_int32, _P, _P, _P, c_int, _P],
    "jv_cta_plan_export": [c_int64, _P, _P, _P, _P, _P, POINTER(c_int64)],
    "jv_cta_plan_free": [c_int64],
    "jv_cta_program_host": [c_int, c_int32, _P, _P, _P, _P, _P, c_int32, _P, _P, _P, _P, _P,
                            c_int, _P, _P, POINTER(c_int64)],
    "jv_cta_smem": [c_int, c_int32, c_int64, c_int32, c_int64, c_int64, c_int, c_int],
    "jv_cta_run": [c_int, c_int32, c_int64, c_int32, _P, _P, c_int64, c_int64, c_int, c_int, c_int32,
                   _P, _P,
                   c_double, c_int, _P, _P, _P, _P],
}
_RESTYPES = {
    "jv_last_error": ctypes.c_char_p,
    "jv_iluk_host": c_int64,
    "jv_free_host": None,
    "jv_region_partition_host": c_int32,
    "jv_rstream_build": c_int64,
    "jv_region_smem_fixed": c_int64,
    "jv_tail_plan_build": c_int64,
    "jv_cta_plan_build": c_int64,
    "jv_cta_smem": c_int64,
    "jv_solve_small_bytes": c_int64,
    "jv_solve_small_max": c_int64,
}

_lib = None


def load():
    """Load libjv.so once; raise BackendUnavailable if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise BackendUnavailable(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (nvcc sm_100a)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, argtypes in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


def exported_symbols():
    return list(_SIGS)


# hot-path entry points that launch exactly one kernel of ours per call;
# launch_counts tallies them (bench.py reports the count it observes)
_ONE_LAUNCH = {"jv_factor", "jv_solve", "jv_region_run", "jv_pack_values", "jv_pack_values2", "jv_row_norms",
               "jv_reset_row", "jv_spmv", "jv_spmv_rows", "jv_gather", "jv_check_zero_diag",
               "jv_solve_level", "jv_tail_upper", "jv_scatter", "jv_cta_run", "jv_solve_small"}
launch_counts = {}


def call(name, *args):
    """Invoke a status-returning entry point; raise on a nonzero status."""
    lib = load()
    if name in _ONE_LAUNCH:
        launch_counts[name] = launch_counts.get(name, 0) + 1
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.jv_last_error().decode(errors="replace")
        raise RuntimeError(f"{name} failed ({rc}): {msg}")
    return rc
