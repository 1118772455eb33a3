"""b200lu — B200-native (sm_100a, FP64 CUDA) refactorize + solve path for fixed-pattern KKT sequences.

Drop-in for the reference library's numeric / triangular-solve / refinement entry points; the
reference's host-side symbolic analysis is consumed as-is — from the reference itself or from `analysis.py`,
which reproduces it bit for bit. See include/b200lu.h for the C ABI and DESIGN.md for the kernels.
"""
from .analysis import AnalyzeOptions, StructurallySingularError, ZeroDiagonalError, symbolic_analyze
from .solver import (Cgs2Result, CsrMatrix, DeviceError, DimensionError, Error, FactorOptions, NumericFactors,
                     PatternMismatchError, RefineConfig, RefineOutcome, SymbolicFactors,
                     ZeroPivotError, cgs2_orthonormalize, classic_refine, factorize, factorize_scattered, fgmres_refine,
                     kkt_bind, kkt_update, lower_solve, refactorize, relative_residual, reset_values, scatter_values,
                     solve_system, spmv, upper_solve)

__all__ = [
    "AnalyzeOptions", "StructurallySingularError", "ZeroDiagonalError", "symbolic_analyze",
    "Cgs2Result", "CsrMatrix", "DeviceError", "DimensionError", "Error", "FactorOptions", "NumericFactors",
    "PatternMismatchError", "RefineConfig", "RefineOutcome", "SymbolicFactors", "ZeroPivotError",
    "cgs2_orthonormalize", "classic_refine", "factorize", "factorize_scattered", "fgmres_refine", "kkt_bind", "kkt_update", "lower_solve",
    "refactorize", "relative_residual", "reset_values", "scatter_values", "solve_system", "spmv",
    "upper_solve",
]
