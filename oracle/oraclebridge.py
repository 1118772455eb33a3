"""TEST INFRASTRUCTURE — ctypes bridge to this repo's plain-C oracle (`oracle/rlu_oracle.c`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import this.
Array conventions are the reference's: int64 indices, float64 values.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "librlu_oracle.so")

OK, ZERO_PIVOT = 0, 1


class _Pattern(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p),
                ("diag_pos", C.c_void_p)]


class _Transform(C.Structure):
    _fields_ = [("amd_forward", C.c_void_p), ("col_perm_forward", C.c_void_p),
                ("row_scale", C.c_void_p), ("col_scale", C.c_void_p)]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_offsets", C.c_void_p), ("col_indices", C.c_void_p),
                ("values", C.c_void_p)]


class _Precond(C.Structure):
    _fields_ = [("F", C.POINTER(_Pattern)), ("values", C.c_void_p), ("T", C.POINTER(_Transform))]


_lib = None


def build():
    subprocess.run(["make", "-C", _HERE, "oracle"], check=True, capture_output=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.rlo_dot.restype = C.c_double
        L.rlo_norm2.restype = C.c_double
        L.rlo_relative_residual.restype = C.c_double
        _lib = L
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class Factors:
    """Pattern + transform of one analysis (fields of rlu::SymbolicFactors), oracle-side."""

    def __init__(self, sym):
        """`sym` is any object with the SymbolicArrays fields (see oracle/refbridge.py)."""
        self.n = int(sym.n)
        self.ro, self.ci, self.dp = _i64(sym.row_offsets), _i64(sym.col_indices), _i64(sym.diag_pos)
        self.smap, self.sscale = _i64(sym.scatter_map), _f64(sym.scatter_scale)
        self.amd = _i64(sym.amd_forward)
        self.q = None if sym.col_perm_forward is None else _i64(sym.col_perm_forward)
        self.dr = None if sym.row_scale is None else _f64(sym.row_scale)
        self.dc = None if sym.col_scale is None else _f64(sym.col_scale)
        self.pat = _Pattern(self.n, _p(self.ro), _p(self.ci), _p(self.dp))
        self.tr = _Transform(_p(self.amd), _p(self.q), _p(self.dr), _p(self.dc))
        self.nnz_factors = int(self.ro[-1])

    def scatter_values(self, a_values) -> np.ndarray:
        a = _f64(a_values)
        out = np.empty(self.nnz_factors, dtype=np.float64)
        lib().rlo_scatter_values(C.c_int64(self.nnz_factors), C.c_int64(a.size), _p(self.smap),
                                 _p(self.sscale), _p(a), _p(out))
        return out

    def eliminate(self, values, pivot_floor=1e-30):
        """Returns (values, failed_row); failed_row == -1 on success."""
        v = _f64(values).copy()
        colpos = np.zeros(max(self.n, 1), dtype=np.int64)
        failed = C.c_int64(-1)
        lib().rlo_eliminate(C.byref(self.pat), _p(v), C.c_double(pivot_floor), _p(colpos),
                            C.byref(failed))
        return v, int(failed.value)

    def factorize(self, a_values, pivot_floor=1e-30):
        return self.eliminate(self.scatter_values(a_values), pivot_floor)

    def lower_solve(self, values, y) -> np.ndarray:
        v, y = _f64(values), _f64(y)
        x = np.empty(self.n, dtype=np.float64)
        lib().rlo_lower_solve(C.byref(self.pat), _p(v), _p(y), _p(x))
        return x

    def upper_solve(self, values, y):
        v, y = _f64(values), _f64(y)
        x = np.empty(self.n, dtype=np.float64)
        failed = C.c_int64(-1)
        st = lib().rlo_upper_solve(C.byref(self.pat), _p(v), _p(y), _p(x), C.byref(failed))
        return x, (int(failed.value) if st == ZERO_PIVOT else -1)

    def solve_system(self, values, b):
        v, b = _f64(values), _f64(b)
        x = np.empty(self.n, dtype=np.float64)
        w1, w2 = np.empty(self.n), np.empty(self.n)
        failed = C.c_int64(-1)
        st = lib().rlo_solve_system(C.byref(self.pat), _p(v), C.byref(self.tr), _p(b), _p(x),
                                    _p(w1), _p(w2), C.byref(failed))
        return x, (int(failed.value) if st == ZERO_PIVOT else -1)


class Csr:
    def __init__(self, n, row_offsets, col_indices, values):
        self.n = int(n)
        self.ro, self.ci, self.v = _i64(row_offsets), _i64(col_indices), _f64(values)
        self.c = _Csr(self.n, _p(self.ro), _p(self.ci), _p(self.v))

    def spmv(self, x):
        x = _f64(x)
        y = np.empty(self.n, dtype=np.float64)
        lib().rlo_spmv(C.byref(self.c), _p(x), _p(y))
        return y

    def relative_residual(self, x, b) -> float:
        x, b = _f64(x), _f64(b)
        return float(lib().rlo_relative_residual(C.byref(self.c), _p(x), _p(b)))


def dot(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return float(lib().rlo_dot(C.c_int64(a.size), _p(a), _p(b)))


def norm2(a) -> float:
    a = _f64(a)
    return float(lib().rlo_norm2(C.c_int64(a.size), _p(a)))


def cgs2(basis, v):
    v = _f64(v).copy()
    n = v.size
    basis = _f64(basis).reshape(-1, n) if np.size(basis) else np.zeros((0, n))
    k = basis.shape[0]
    coef = np.zeros(max(k, 1), dtype=np.float64)
    norm, bd = C.c_double(), C.c_int()
    lib().rlo_cgs2(C.c_int64(n), C.c_int64(k), _p(basis), _p(v), _p(coef), C.byref(norm),
                   C.byref(bd))
    return coef[:k], v, norm.value, bool(bd.value)


def refine(A: Csr, b, x0, factors: Factors | None = None, values=None, method="fgmres",
           max_iterations=20, tolerance=1e-14):
    """Returns (x, iterations, converged, residual_history)."""
    b, x0 = _f64(b), _f64(x0)
    x = np.empty(A.n, dtype=np.float64)
    hist = np.zeros(max(1, max_iterations) + 2, dtype=np.float64)
    it, conv, hl = C.c_int(), C.c_int(), C.c_int()
    if factors is not None:
        vals = _f64(values)
        M = _Precond(C.pointer(factors.pat), _p(vals), C.pointer(factors.tr))
        Mp = C.byref(M)
    else:
        Mp = None
    fn = lib().rlo_fgmres if method == "fgmres" else lib().rlo_classic_refine
    fn(C.byref(A.c), _p(b), _p(x0), Mp, C.c_int(max_iterations), C.c_double(tolerance), _p(x),
       C.byref(it), C.byref(conv), _p(hist), C.byref(hl))
    return x, it.value, bool(conv.value), hist[:hl.value].copy()
