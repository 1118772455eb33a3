"""Host-side mirror of the reference's numeric/solve/refine interface over the b200lu C ABI.

Names, argument meaning and error behaviour follow the reference (paths relative to the
reference's proj/):
  factorize / refactorize / reset_values / factorize_scattered   include/rlu/numeric.hpp:42-53
  lower_solve / upper_solve / solve_system                        include/rlu/trisolve.hpp:23-39
  fgmres_refine / classic_refine                                  include/rlu/refine.hpp:43-52
  Error / DimensionError / ZeroPivotError / PatternMismatchError  include/rlu/errors.hpp:11-54

Vectors may be numpy arrays (host path: copied over the handle's stream) or CUDA torch
tensors (device path: pointers are used in place, nothing is copied).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi


class Error(RuntimeError):
    """rlu::Error (include/rlu/errors.hpp:11-14)."""


class DimensionError(Error):
    """rlu::DimensionError (include/rlu/errors.hpp:21-24)."""


class ZeroPivotError(Error):
    """rlu::ZeroPivotError (include/rlu/errors.hpp:42-47); `row` is the permuted row index."""

    def __init__(self, msg: str, row: int):
        super().__init__(msg)
        self.row = row


class PatternMismatchError(Error):
    """rlu::PatternMismatchError (include/rlu/errors.hpp:51-54)."""


class DeviceError(Error):
    """CUDA failure or missing device — there is no CPU fallback."""


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _is_device_tensor(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


@dataclass
class CsrMatrix:
    """rlu::CsrMatrix (include/rlu/sparse.hpp:31-47). `values` may be None (pattern only) or a
    CUDA torch tensor (device-resident values)."""
    nrows: int
    ncols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: object = None

    def has_values(self) -> bool:
        if self.values is None:
            return False
        return int(self.values.numel() if _is_device_tensor(self.values) else np.size(self.values)) \
            == int(np.size(self.col_indices))


@dataclass
class SymbolicFactors:
    """Plain-array image of rlu::SymbolicFactors (include/rlu/symbolic.hpp:48-59), produced by
    the reference's host-side symbolic_analyze and consumed bit-exact."""
    n: int
    row_offsets: np.ndarray       # combined_pattern.row_offsets
    col_indices: np.ndarray       # combined_pattern.col_indices
    diag_pos: np.ndarray
    scatter_map: np.ndarray
    scatter_scale: np.ndarray
    amd_forward: np.ndarray
    src_row_offsets: np.ndarray   # source_pattern.row_offsets
    src_col_indices: np.ndarray   # source_pattern.col_indices
    col_perm_forward: np.ndarray | None = None
    row_scale: np.ndarray | None = None
    col_scale: np.ndarray | None = None
    fill_count: int = 0

    @classmethod
    def from_arrays(cls, s) -> "SymbolicFactors":
        """Accepts any object carrying the same field names (e.g. the test bridge's arrays)."""
        return cls(int(s.n), _i64(s.row_offsets), _i64(s.col_indices), _i64(s.diag_pos),
                   _i64(s.scatter_map), _f64(s.scatter_scale), _i64(s.amd_forward),
                   _i64(s.src_row_offsets), _i64(s.src_col_indices),
                   None if s.col_perm_forward is None else _i64(s.col_perm_forward),
                   None if s.row_scale is None else _f64(s.row_scale),
                   None if s.col_scale is None else _f64(s.col_scale),
                   int(getattr(s, "fill_count", 0)))


@dataclass
class FactorOptions:
    """rlu::FactorOptions (include/rlu/numeric.hpp:12-15) plus device placement. The CPU
    ExecPolicy has no device counterpart."""
    pivot_floor: float = 1e-30
    device: int = 0
    stream: int | None = None      # raw cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)
    refine_capacity: int = 20
    strict_order: bool = False     # sweeps in the reference's summation order (bit-identical x)
    concurrency: int = 1           # handles sharing the device at the same time (scenario batches)


@dataclass
class RefineConfig:
    """rlu::RefineConfig (include/rlu/refine.hpp:13-17)."""
    max_iterations: int = 20
    tolerance: float = 1e-14
    enabled: bool = True


@dataclass
class RefineOutcome:
    """rlu::RefineOutcome (include/rlu/refine.hpp:19-24)."""
    x: object = None
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    converged: bool = False


class NumericFactors:
    """rlu::NumericFactors (include/rlu/numeric.hpp:22-31) with its SolveWorkspace
    (include/rlu/trisolve.hpp:12-19) folded in: one handle == one stream == one operation at a
    time; distinct instances are independent and may share one SymbolicFactors."""

    def __init__(self, sym: SymbolicFactors, options: FactorOptions | None = None):
        self.symbolic = sym
        self.options = options or FactorOptions()
        self._h = C.c_void_p()
        L = _capi.lib()
        v = _capi.SymbolicView()
        v.n, v.nnz_factors, v.nnz_source = sym.n, int(sym.row_offsets[-1]) if sym.n >= 0 and len(sym.row_offsets) else 0, len(sym.scatter_map)
        keep = [sym.row_offsets, sym.col_indices, sym.diag_pos, sym.scatter_map, sym.scatter_scale,
                sym.amd_forward, sym.src_row_offsets, sym.src_col_indices]
        v.row_offsets, v.col_indices, v.diag_pos = (a.ctypes.data for a in keep[:3])
        v.scatter_map, v.scatter_scale, v.amd_forward = (a.ctypes.data for a in keep[3:6])
        v.source_row_offsets, v.source_col_indices = keep[6].ctypes.data, keep[7].ctypes.data
        if sym.col_perm_forward is not None:
            v.col_perm_forward = sym.col_perm_forward.ctypes.data
            v.row_scale = sym.row_scale.ctypes.data
            v.col_scale = sym.col_scale.ctypes.data
        o = _capi.Options()
        L.b200lu_default_options(C.byref(o))
        o.pivot_floor = self.options.pivot_floor
        o.device = self.options.device
        o.stream = self.options.stream
        o.refine_capacity = self.options.refine_capacity
        o.flags = _capi.FLAG_STRICT_ORDER if self.options.strict_order else 0
        o.concurrency = self.options.concurrency
        st = L.b200lu_create(C.byref(v), C.byref(o), C.byref(self._h))
        if st != _capi.OK:
            msg = L.b200lu_last_error(self._h).decode() if self._h else ""
            if self._h:
                L.b200lu_destroy(self._h)
                self._h = C.c_void_p()
            if st == _capi.NO_DEVICE:
                raise DeviceError("no CUDA device: the b200lu path has no CPU fallback")
            raise (DeviceError if st == _capi.CUDA_ERROR else Error)(
                f"b200lu_create: {L.b200lu_status_string(st).decode()}: {msg}")

    def close(self):
        if getattr(self, "_h", None):
            _capi.lib().b200lu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state -------------------------------------------------------------
    @property
    def valid(self) -> bool:
        return bool(_capi.lib().b200lu_valid(self._h))

    @property
    def generation(self) -> int:
        return int(_capi.lib().b200lu_generation(self._h))

    @property
    def values(self) -> np.ndarray:
        out = np.empty(int(self.symbolic.row_offsets[-1]) if self.symbolic.n else 0, dtype=np.float64)
        self._check(_capi.lib().b200lu_get_values(self._h, out.ctypes.data))
        return out

    def set_values(self, values, valid=True):
        v = _f64(values)
        self._check(_capi.lib().b200lu_set_values(self._h, v.ctypes.data, 1 if valid else 0))

    @property
    def values_device_ptr(self) -> int:
        return int(_capi.lib().b200lu_values_device(self._h) or 0)

    @property
    def stats(self) -> dict:
        s = _capi.Stats()
        self._check(_capi.lib().b200lu_get_stats(self._h, C.byref(s)))
        return {k: int(getattr(s, k)) for k, _ in _capi.Stats._fields_}

    @property
    def launch_count(self) -> int:
        return int(_capi.lib().b200lu_launch_count(self._h))

    def set_timing(self, enabled: bool = True):
        """Per-phase device timing (CUDA events around each kernel), cf. src/cli.cpp:105-132."""
        self._check(_capi.lib().b200lu_set_timing(self._h, 1 if enabled else 0))

    def phase_times(self, reset: bool = True) -> dict:
        """{phase: (kernel milliseconds, launches)} accumulated since the last reset."""
        n = len(_capi.PHASES)
        ms, cnt = (C.c_double * n)(), (C.c_int64 * n)()
        self._check(_capi.lib().b200lu_get_phase_times(self._h, ms, cnt, 1 if reset else 0))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(_capi.PHASES)}

    def synchronize(self):
        self._check(_capi.lib().b200lu_synchronize(self._h))

    # -- error mapping -----------------------------------------------------
    def _check(self, st: int, failed_row: int = -1):
        if st == _capi.OK:
            return
        L = _capi.lib()
        msg = L.b200lu_last_error(self._h).decode() or L.b200lu_status_string(st).decode()
        if st == _capi.ZERO_PIVOT:
            raise ZeroPivotError(msg, failed_row)
        if st == _capi.PATTERN_MISMATCH:
            raise PatternMismatchError("matrix pattern differs from the analyzed pattern")
        if st == _capi.DIMENSION:
            raise DimensionError(msg)
        if st in (_capi.CUDA_ERROR, _capi.NO_DEVICE):
            raise DeviceError(msg)
        raise Error(msg)

    # -- vector plumbing -----------------------------------------------------
    def _vec_in(self, x):
        """Returns (pointer, on_device, length, keepalive)."""
        if _is_device_tensor(x):
            import torch
            assert x.dtype == torch.float64 and x.is_contiguous()
            return x.data_ptr(), 1, x.numel(), x
        a = _f64(x)
        return a.ctypes.data, 0, a.size, a

    def _vec_out(self, like, n):
        if _is_device_tensor(like):
            import torch
            out = torch.empty(n, dtype=torch.float64, device=like.device)
            return out.data_ptr(), out
        out = np.empty(n, dtype=np.float64)
        return out.ctypes.data, out


def _values_ptr(A: CsrMatrix):
    if _is_device_tensor(A.values):
        return A.values.data_ptr(), 1, A.values
    v = _f64(A.values)
    return v.ctypes.data, 0, v


def _guard_pattern(f: NumericFactors, A: CsrMatrix):
    """scatter_values' guards, src/numeric.cpp:15-18: pattern_equal runs on EVERY scatter, as in
    the reference — an 8*(n+1+nnz)-byte memcmp, small next to a factorization — so neither a
    recycled handle nor an in-place edit of the pattern arrays can slip through. The value count is
    checked too: reset_values copies nnz_source doubles from the caller's buffer."""
    ro, ci = _i64(A.row_offsets), _i64(A.col_indices)
    st = _capi.PATTERN_MISMATCH
    if A.nrows == A.ncols and ro.size == A.nrows + 1 and ci.size == len(f.symbolic.src_col_indices):
        st = _capi.lib().b200lu_check_pattern(f._h, A.nrows, ro.ctypes.data, ci.ctypes.data)
    if st != _capi.OK:
        raise PatternMismatchError("matrix pattern differs from the analyzed pattern")
    if A.values is None:
        raise Error("scatter_values: matrix has no values")
    nvals = A.values.numel() if _is_device_tensor(A.values) else np.asarray(A.values).size
    if nvals != ci.size:
        raise PatternMismatchError("matrix has %d values for %d pattern entries" % (nvals, ci.size))


def reset_values(f: NumericFactors, A: CsrMatrix):
    """reset_values, src/numeric.cpp:75-77."""
    _guard_pattern(f, A)
    p, dev, keep = _values_ptr(A)
    f._check(_capi.lib().b200lu_reset_values(f._h, p, dev))


def factorize_scattered(f: NumericFactors):
    """factorize_scattered, src/numeric.cpp:79."""
    row = C.c_int64(-1)
    st = _capi.lib().b200lu_factorize_scattered(f._h, C.byref(row))
    f._check(st, int(row.value))


def refactorize(f: NumericFactors, A: CsrMatrix):
    """refactorize, src/numeric.cpp:70-73."""
    _guard_pattern(f, A)
    p, dev, keep = _values_ptr(A)
    row = C.c_int64(-1)
    st = _capi.lib().b200lu_refactorize(f._h, p, dev, C.byref(row))
    f._check(st, int(row.value))


def factorize(sym: SymbolicFactors, A: CsrMatrix, options: FactorOptions | None = None) -> NumericFactors:
    """factorize, src/numeric.cpp:62-68."""
    f = NumericFactors(sym, options)
    try:
        refactorize(f, A)
    except Exception:
        f.close()
        raise
    return f


def scatter_values(sym_or_factors, A: CsrMatrix) -> np.ndarray:
    """scatter_values, src/numeric.cpp:14-23: the scattered (not yet eliminated) values."""
    f = sym_or_factors if isinstance(sym_or_factors, NumericFactors) else NumericFactors(sym_or_factors)
    reset_values(f, A)
    out = f.values
    if f is not sym_or_factors:
        f.close()
    return out


def lower_solve(f: NumericFactors, y):
    """lower_solve, src/trisolve.cpp:72-79."""
    p, dev, n, keep = f._vec_in(y)
    if not f.valid:
        raise Error("lower_solve: factors are not valid")
    if n != f.symbolic.n:
        raise DimensionError(f"lower_solve: vector length {n}, expected {f.symbolic.n}")
    po, out = f._vec_out(y, n)
    f._check(_capi.lib().b200lu_lower_solve(f._h, n, p, po, dev))
    return out


def upper_solve(f: NumericFactors, y):
    """upper_solve, src/trisolve.cpp:81-88."""
    p, dev, n, keep = f._vec_in(y)
    if not f.valid:
        raise Error("upper_solve: factors are not valid")
    if n != f.symbolic.n:
        raise DimensionError(f"upper_solve: vector length {n}, expected {f.symbolic.n}")
    po, out = f._vec_out(y, n)
    row = C.c_int64(-1)
    st = _capi.lib().b200lu_upper_solve(f._h, n, p, po, dev, C.byref(row))
    f._check(st, int(row.value))
    return out


def solve_system(f: NumericFactors, b, out=None):
    """solve_system, src/trisolve.cpp:90-119."""
    p, dev, n, keep = f._vec_in(b)
    if not f.valid:
        raise Error("solve_system: factors are not valid")
    if n != f.symbolic.n:
        raise DimensionError(f"solve_system: vector length {n}, expected {f.symbolic.n}")
    if out is None:
        po, out = f._vec_out(b, n)
    else:
        po = out.data_ptr() if _is_device_tensor(out) else out.ctypes.data
    row = C.c_int64(-1)
    st = _capi.lib().b200lu_solve(f._h, n, p, po, dev, C.byref(row))
    f._check(st, int(row.value))
    return out


def spmv(f: NumericFactors, x):
    """spmv, src/sparse.cpp:128-143, with A = the matrix last handed to reset_values/refactorize."""
    p, dev, n, keep = f._vec_in(x)
    if n != f.symbolic.n:
        raise DimensionError(f"spmv: x has length {n}, expected {f.symbolic.n}")
    po, out = f._vec_out(x, n)
    f._check(_capi.lib().b200lu_spmv(f._h, p, po, dev))
    return out


def relative_residual(f: NumericFactors, x, b) -> float:
    """relative_residual, src/sparse.cpp:283-288."""
    px, dev, n, k1 = f._vec_in(x)
    pb, dev2, n2, k2 = f._vec_in(b)
    assert dev == dev2 and n == n2 == f.symbolic.n
    out = C.c_double()
    f._check(_capi.lib().b200lu_relative_residual(f._h, px, pb, dev, C.byref(out)))
    return float(out.value)


def _refine(fn_name, f, b, x0, config, preconditioned):
    config = config or RefineConfig()
    pb, dev, n, k1 = f._vec_in(b)
    px, dev2, n2, k2 = f._vec_in(x0)
    if dev != dev2:
        raise Error("refine: b and x0 must both be host arrays or both device tensors")
    if n != f.symbolic.n or n2 != f.symbolic.n:
        raise DimensionError(f"refine: vector length {n}/{n2}, expected {f.symbolic.n}")
    po, out = f._vec_out(b, n)
    cfg = _capi.RefineConfig(config.max_iterations, config.tolerance)
    oc = _capi.RefineOutcome()
    st = getattr(_capi.lib(), fn_name)(f._h, pb, px, po, dev, 1 if preconditioned else 0,
                                       C.byref(cfg), C.byref(oc))
    f._check(st)
    return RefineOutcome(out, int(oc.iterations), list(oc.residual_history[:oc.history_len]),
                         bool(oc.converged))


def fgmres_refine(f: NumericFactors, b, x0, config: RefineConfig | None = None,
                  preconditioned: bool = True) -> RefineOutcome:
    """fgmres_refine, src/refine.cpp:39-142, with A = the handle's matrix and the preconditioner
    solve_system(f, .) (src/cli.cpp:121-135); preconditioned=False is the identity operator."""
    return _refine("b200lu_refine_fgmres", f, b, x0, config, preconditioned)


def classic_refine(f: NumericFactors, b, x0, config: RefineConfig | None = None,
                   preconditioned: bool = True) -> RefineOutcome:
    """classic_refine, src/refine.cpp:150-188."""
    return _refine("b200lu_refine_classic", f, b, x0, config, preconditioned)


@dataclass
class Cgs2Result:
    """include/rlu/refine.hpp:25-30."""
    coefficients: np.ndarray
    vector: np.ndarray
    norm: float
    breakdown: bool


def cgs2_orthonormalize(f: NumericFactors, basis, v) -> Cgs2Result:
    """cgs2_orthonormalize, src/refine.cpp:8-26, on the device of handle `f` (vectors of length f.symbolic.n):
    two full Gram-Schmidt passes of v against the orthonormal rows of `basis` ([k, n]), then normalisation."""
    n = f.symbolic.n
    B = np.ascontiguousarray(basis, dtype=np.float64).reshape(-1, n) if np.size(basis) else np.zeros((0, n))
    vv = _f64(v)
    if vv.size != n:
        raise DimensionError(f"cgs2_orthonormalize: vector length {vv.size}, expected {n}")
    k = B.shape[0]
    coef = np.zeros(max(k, 1), dtype=np.float64)
    out = np.empty(n, dtype=np.float64)
    norm, bd = C.c_double(), C.c_int()
    f._check(_capi.lib().b200lu_cgs2_orthonormalize(f._h, k, B.ctypes.data, vv.ctypes.data, 0, coef.ctypes.data,
                                                    out.ctypes.data, C.byref(norm), C.byref(bd)))
    return Cgs2Result(coef[:k], out, float(norm.value), bool(bd.value))


def kkt_bind(f: NumericFactors, n_primal: int, h_diag, diag_source_pos):
    """Prepares the device-resident KKT value path (include/b200lu.h, b200lu_kkt_bind): H's own
    diagonal and the position of every K_ii in source-CSR order."""
    hd, pos = _f64(h_diag), _i64(diag_source_pos)
    if hd.size != n_primal or pos.size != f.symbolic.n:
        raise DimensionError("kkt_bind: h_diag needs n_primal entries, diag_source_pos needs n")
    f._check(_capi.lib().b200lu_kkt_bind(f._h, n_primal, hd.ctypes.data, pos.ctypes.data))
    f._kkt_n_primal = n_primal


def kkt_update(f: NumericFactors, d_y, delta_p: float, delta_d: float):
    """assemble_kkt's value path on the device (src/kkt.cpp:53-77): rewrites K's diagonal from D_y and
    the regularization shifts and scatters — replaces reset_values for a system that differs from the
    last one only in its barrier diagonal / regularization. Follow with factorize_scattered."""
    p, dev, n, keep = f._vec_in(d_y)
    if n != getattr(f, "_kkt_n_primal", -1):
        raise DimensionError(f"kkt_update: D_y has length {n}, expected {getattr(f, '_kkt_n_primal', -1)}")
    f._check(_capi.lib().b200lu_kkt_update(f._h, p, dev, float(delta_p), float(delta_d)))
