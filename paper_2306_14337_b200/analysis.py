"""Host-side symbolic analysis: rlu::symbolic_analyze (include/rlu/symbolic.hpp:67-75, src/symbolic.cpp:156-203)
with the reference's AnalyzeOptions, reproduced bit for bit by the host code in csrc/analyze.cpp.

Runs without a GPU; the product is the same SymbolicFactors image the numeric path consumes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from .solver import CsrMatrix, DimensionError, Error, SymbolicFactors


class ZeroDiagonalError(Error):
    """rlu::ZeroDiagonalError (include/rlu/errors.hpp:37-42): no stored diagonal entry in `row` of the permuted matrix."""

    def __init__(self, msg: str, row: int):
        super().__init__(msg)
        self.row = row


class StructurallySingularError(Error):
    """rlu::StructurallySingularError (include/rlu/errors.hpp:27-34)."""

    def __init__(self, msg: str, deficient_rows):
        super().__init__(msg)
        self.deficient_rows = list(deficient_rows)


@dataclass
class AnalyzeOptions:
    """rlu::AnalyzeOptions (include/rlu/symbolic.hpp:67-70)."""
    use_scaling: bool = True
    use_amd: bool = True


@dataclass
class AnalysisTimes:
    matching_ms: float
    ordering_ms: float
    permutation_ms: float
    fill_ms: float
    scatter_map_ms: float
    total_ms: float


def _copy(ptr, count, dtype):
    if not ptr or count == 0:
        return np.zeros(0, dtype=dtype)
    ctype = C.c_int64 if dtype == np.int64 else C.c_double
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,)).copy()


def symbolic_analyze(A: CsrMatrix, options: AnalyzeOptions | None = None, with_times: bool = False):
    """symbolic_analyze(A, options): MC64 scaling/matching (optional), AMD (optional), fill pattern, diag_pos,
    scatter map and scale. Returns SymbolicFactors (and AnalysisTimes with `with_times`)."""
    opt = options or AnalyzeOptions()
    if A.nrows != A.ncols:
        raise DimensionError("symbolic_analyze: matrix must be square")
    ro = np.ascontiguousarray(A.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_indices, dtype=np.int64)
    if ro.size != A.nrows + 1:
        raise Error("row_offsets length must be nrows + 1")
    if ci.size != (int(ro[-1]) if ro.size else 0):
        raise Error("col_indices length disagrees with row_offsets")
    vals = None
    if opt.use_scaling:
        if A.values is None or np.size(A.values) != ci.size:
            raise Error("mc64_scale: matrix has no values")
        vals = np.ascontiguousarray(A.values, dtype=np.float64)
    L = _capi.lib()
    h = C.c_void_p()
    st = L.b200lu_analyze(A.nrows, ro.ctypes.data, ci.ctypes.data, vals.ctypes.data if vals is not None else None,
                          int(opt.use_scaling), int(opt.use_amd), C.byref(h))
    if not h:
        raise Error("symbolic_analyze: " + L.b200lu_status_string(st).decode())
    try:
        if st != _capi.OK:
            row, rows, cnt = C.c_int64(-1), C.c_void_p(), C.c_int64(0)
            L.b200lu_analysis_status(h, C.byref(row), C.byref(rows), C.byref(cnt))
            msg = L.b200lu_analysis_message(h).decode()
            if st == _capi.ZERO_DIAGONAL:
                raise ZeroDiagonalError(msg, int(row.value))
            if st == _capi.STRUCTURALLY_SINGULAR:
                raise StructurallySingularError(msg, _copy(rows.value, cnt.value, np.int64).tolist())
            raise Error(msg or L.b200lu_status_string(st).decode())
        v = _capi.SymbolicView()
        fill = C.c_int64(0)
        L.b200lu_analysis_view(h, C.byref(v), C.byref(fill))
        n, nf, ns = int(v.n), int(v.nnz_factors), int(v.nnz_source)
        sym = SymbolicFactors(
            n, _copy(v.row_offsets, n + 1, np.int64), _copy(v.col_indices, nf, np.int64), _copy(v.diag_pos, n, np.int64),
            _copy(v.scatter_map, ns, np.int64), _copy(v.scatter_scale, ns, np.float64), _copy(v.amd_forward, n, np.int64),
            _copy(v.source_row_offsets, n + 1, np.int64), _copy(v.source_col_indices, ns, np.int64),
            _copy(v.col_perm_forward, n, np.int64) if v.col_perm_forward else None,
            _copy(v.row_scale, n, np.float64) if v.row_scale else None,
            _copy(v.col_scale, n, np.float64) if v.col_scale else None,
            int(fill.value))
        if with_times:
            ms = (C.c_double * 6)()
            L.b200lu_analysis_times(h, ms, None)
            return sym, AnalysisTimes(*[float(x) for x in ms])
        return sym
    finally:
        L.b200lu_analysis_destroy(h)
