"""ctypes binding of the C ABI in include/b200lu.h (libb200lu.so, built in-tree by __graft_entry__.build()).

There is no fallback: if the CUDA library is missing, importing the solver raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libb200lu.so")

(OK, ZERO_PIVOT, PATTERN_MISMATCH, DIMENSION, INVALID_FACTORS, CUDA_ERROR, INVALID_ARGUMENT, NO_DEVICE, ZERO_DIAGONAL,
 STRUCTURALLY_SINGULAR) = range(10)

i64, u64, dbl, i32, vp = C.c_int64, C.c_uint64, C.c_double, C.c_int, C.c_void_p


class SymbolicView(C.Structure):
    _fields_ = [("n", i64), ("nnz_factors", i64), ("nnz_source", i64),
                ("row_offsets", vp), ("col_indices", vp), ("diag_pos", vp),
                ("scatter_map", vp), ("scatter_scale", vp), ("amd_forward", vp),
                ("col_perm_forward", vp), ("row_scale", vp), ("col_scale", vp),
                ("source_row_offsets", vp), ("source_col_indices", vp)]


class Options(C.Structure):
    _fields_ = [("pivot_floor", dbl), ("device", i32), ("stream", vp), ("refine_capacity", i32),
                ("flags", i32), ("concurrency", i32)]


class RefineConfig(C.Structure):
    _fields_ = [("max_iterations", i32), ("tolerance", dbl)]


class RefineOutcome(C.Structure):
    _fields_ = [("iterations", i32), ("converged", i32), ("history_len", i32),
                ("residual_history", dbl * 66)]


class Stats(C.Structure):
    _fields_ = [(k, i64) for k in ("n", "nnz_factors", "nnz_source", "nnz_lower", "update_pairs",
                                   "lower_levels", "upper_levels", "max_row_len", "big_rows",
                                   "device_bytes", "alloc_events", "lower_tail_rows",
                                   "lower_tail_levels", "upper_tail_rows", "upper_tail_levels")]


class BatchInfo(C.Structure):
    _fields_ = [(k, i64) for k in ("batch", "padded_batch", "unit_scenarios", "blocks", "factor_rows",
                                   "blocked_rows", "blocked_pairs", "factor_grid", "tri_grid", "n", "nnz_factors",
                                   "nnz_source", "update_pairs", "lower_levels", "upper_levels", "device_bytes",
                                   "alloc_events", "launches", "tiled", "tile_rows", "tile_smem_bytes", "tile_grid",
                                   "tile_fetched_entries")]


class TilePlanStats(C.Structure):
    _fields_ = [(k, i64) for k in ("tiles", "rows", "items", "pairs", "fetched_entries", "consumed_entries",
                                   "largest_tile_entries")]


EXPORTS = {
    # name: (restype, argtypes)
    "b200lu_default_options": (None, [C.POINTER(Options)]),
    "b200lu_status_string": (C.c_char_p, [i32]),
    "b200lu_last_error": (C.c_char_p, [vp]),
    "b200lu_device_count": (i32, []),
    "b200lu_create": (i32, [C.POINTER(SymbolicView), C.POINTER(Options), C.POINTER(vp)]),
    "b200lu_destroy": (None, [vp]),
    "b200lu_check_pattern": (i32, [vp, i64, vp, vp]),
    "b200lu_reset_values": (i32, [vp, vp, i32]),
    "b200lu_factorize_scattered": (i32, [vp, C.POINTER(i64)]),
    "b200lu_refactorize": (i32, [vp, vp, i32, C.POINTER(i64)]),
    "b200lu_valid": (i32, [vp]),
    "b200lu_generation": (u64, [vp]),
    "b200lu_get_values": (i32, [vp, vp]),
    "b200lu_set_values": (i32, [vp, vp, i32]),
    "b200lu_values_device": (vp, [vp]),
    "b200lu_lower_solve": (i32, [vp, i64, vp, vp, i32]),
    "b200lu_upper_solve": (i32, [vp, i64, vp, vp, i32, C.POINTER(i64)]),
    "b200lu_solve": (i32, [vp, i64, vp, vp, i32, C.POINTER(i64)]),
    "b200lu_spmv": (i32, [vp, vp, vp, i32]),
    "b200lu_relative_residual": (i32, [vp, vp, vp, i32, C.POINTER(dbl)]),
    "b200lu_refine_fgmres": (i32, [vp, vp, vp, vp, i32, i32, C.POINTER(RefineConfig),
                                   C.POINTER(RefineOutcome)]),
    "b200lu_refine_classic": (i32, [vp, vp, vp, vp, i32, i32, C.POINTER(RefineConfig),
                                    C.POINTER(RefineOutcome)]),
    "b200lu_cgs2_orthonormalize": (i32, [vp, i64, vp, vp, i32, vp, vp, C.POINTER(dbl), C.POINTER(i32)]),
    "b200lu_get_stats": (i32, [vp, C.POINTER(Stats)]),
    "b200lu_schedule_probe": (i32, [C.POINTER(SymbolicView), C.POINTER(Stats), vp, vp, vp, C.c_char_p, i32]),
    "b200lu_set_timing": (i32, [vp, i32]),
    "b200lu_get_phase_times": (i32, [vp, C.POINTER(dbl), C.POINTER(i64), i32]),
    "b200lu_launch_count": (u64, [vp]),
    "b200lu_synchronize": (i32, [vp]),
    "b200lu_kkt_bind": (i32, [vp, i64, vp, vp]),
    "b200lu_kkt_update": (i32, [vp, vp, i32, dbl, dbl]),
    "b200lu_batch_kkt_bind": (i32, [vp, i64, vp, vp]),
    "b200lu_batch_kkt_update": (i32, [vp, vp, i32, dbl, dbl]),
    # scenario batches
    "b200lu_batch_create": (i32, [C.POINTER(SymbolicView), C.POINTER(Options), i64, C.POINTER(vp)]),
    "b200lu_batch_destroy": (None, [vp]),
    "b200lu_batch_last_error": (C.c_char_p, [vp]),
    "b200lu_batch_check_pattern": (i32, [vp, i64, vp, vp]),
    "b200lu_batch_reset_values": (i32, [vp, vp, i32]),
    "b200lu_batch_factorize_scattered": (i32, [vp, vp]),
    "b200lu_batch_refactorize": (i32, [vp, vp, i32, vp]),
    "b200lu_batch_valid": (i32, [vp, i64]),
    "b200lu_batch_get_values": (i32, [vp, i64, vp]),
    "b200lu_batch_lower_solve": (i32, [vp, vp, vp, i32]),
    "b200lu_batch_upper_solve": (i32, [vp, vp, vp, i32, vp]),
    "b200lu_batch_solve": (i32, [vp, vp, vp, i32, vp]),
    "b200lu_batch_relative_residual": (i32, [vp, vp, vp, i32, vp]),
    "b200lu_batch_refine_fgmres": (i32, [vp, vp, vp, vp, i32, i32, C.POINTER(RefineConfig), vp]),
    "b200lu_batch_refine_classic": (i32, [vp, vp, vp, vp, i32, i32, C.POINTER(RefineConfig), vp]),
    "b200lu_batch_stage_inputs": (i32, [vp, vp, vp]),
    "b200lu_batch_refactorize_staged": (i32, [vp, vp]),
    "b200lu_batch_solve_refine_staged": (i32, [vp, i32, C.POINTER(RefineConfig), vp, vp, vp]),
    "b200lu_batch_staged_wait": (i32, [vp]),
    "b200lu_batch_get_info": (i32, [vp, C.POINTER(BatchInfo)]),
    "b200lu_tile_plan_emulate": (i32, [C.POINTER(SymbolicView), i32, i64, i64, dbl, vp, C.POINTER(i64),
                                       C.POINTER(TilePlanStats), C.c_char_p, i32]),
    "b200lu_batch_tile_profile": (i32, [vp, vp, i32]),
    "b200lu_batch_set_timing": (i32, [vp, i32]),
    "b200lu_batch_get_phase_times": (i32, [vp, C.POINTER(dbl), C.POINTER(i64), i32]),
    "b200lu_batch_synchronize": (i32, [vp]),
    # host-side symbolic analysis
    "b200lu_analyze": (i32, [i64, vp, vp, vp, i32, i32, C.POINTER(vp)]),
    "b200lu_analysis_status": (i32, [vp, C.POINTER(i64), C.POINTER(vp), C.POINTER(i64)]),
    "b200lu_analysis_message": (C.c_char_p, [vp]),
    "b200lu_analysis_view": (i32, [vp, C.POINTER(SymbolicView), C.POINTER(i64)]),
    "b200lu_analysis_times": (i32, [vp, C.POINTER(dbl), C.POINTER(dbl)]),
    "b200lu_analysis_destroy": (None, [vp]),
}

FLAG_STRICT_ORDER = 1
PHASES = ("scatter", "factor", "lower", "upper", "permute", "spmv", "vector", "tail")

_lib = None


def lib():
    """Loads libb200lu.so; raises (no fallback) when it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: the CUDA library is the only implementation of this "
                "path. Build it with `python -c 'import __graft_entry__ as g; g.build()'`.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
