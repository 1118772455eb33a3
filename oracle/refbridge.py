"""TEST INFRASTRUCTURE — ctypes bridge to the UNMODIFIED reference (`oracle/_ref/librlu_ref.so`).

Built by `oracle/Makefile` from the reference sources where they lie under
`/root/reference/proj` plus `oracle/ref_shim.cpp`. Only `tests/`,
`__graft_entry__.smoke()` and `bench.py` (input fixtures, CPU-baseline arm) may
import this module; the shipped CUDA path never does.

The classes mirror the reference's own objects:
  RefCsr       rlu::CsrMatrix        (proj/include/rlu/sparse.hpp:31-47)
  RefSequence  rlu::KktSequence      (proj/include/rlu/kkt.hpp:34-42) from gen_sequence
  RefSymbolic  rlu::SymbolicFactors  (proj/include/rlu/symbolic.hpp:48-59)
  RefNumeric   rlu::NumericFactors + SolveWorkspace (numeric.hpp:22-31, trisolve.hpp:12-19)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librlu_ref.so")

OK, ZERO_PIVOT, PATTERN_MISMATCH, DIMENSION, ERROR, STRUCT_SINGULAR, ZERO_DIAGONAL = range(7)


class RefError(RuntimeError):
    def __init__(self, status: int, message: str, row: int = -1):
        super().__init__(f"[reference status {status}] {message}")
        self.status = status
        self.row = row


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not available():
        raise FileNotFoundError(
            f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
    L = C.CDLL(LIB_PATH)
    vp, i64, u64, dbl, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
    P = C.POINTER

    def sig(name, res, *args):
        f = getattr(L, name)
        f.restype = res
        f.argtypes = list(args)

    sig("rluref_last_error", C.c_char_p)
    sig("rluref_last_row", i64)
    sig("rluref_max_threads", i32)
    sig("rluref_rng_create", vp, u64)
    sig("rluref_rng_destroy", None, vp)
    sig("rluref_rng_uniform_int", i64, vp, i64, i64)
    sig("rluref_rng_uniform_real", dbl, vp, dbl, dbl)
    sig("rluref_random_sparse", vp, vp, i64, i64, dbl, dbl, i32)
    sig("rluref_random_vector", None, vp, i64, dbl, dbl, vp)
    sig("rluref_csr_create", vp, i64, vp, vp, vp)
    sig("rluref_csr_destroy", None, vp)
    sig("rluref_csr_n", i64, vp)
    sig("rluref_csr_nnz", i64, vp)
    sig("rluref_csr_get", None, vp, vp, vp, vp)
    sig("rluref_csr_set_values", None, vp, vp)
    sig("rluref_gen_sequence", vp, i64, i64, u64, u64, i64, dbl, dbl, dbl, dbl, dbl)
    sig("rluref_gen_sequence_blocks", vp, i64, i64, u64, u64, i64, dbl, dbl, dbl, dbl, dbl)
    sig("rluref_seq_has_blocks", C.c_int, vp)
    sig("rluref_seq_n_primal", i64, vp)
    sig("rluref_seq_h_diag", None, vp, i64, vp)
    sig("rluref_seq_dy", None, vp, i64, vp)
    sig("rluref_seq_deltas", None, vp, i64, C.POINTER(dbl), C.POINTER(dbl))
    sig("rluref_seq_double_regularization", C.c_int, vp, i64)
    sig("rluref_seq_destroy", None, vp)
    sig("rluref_seq_num_systems", i64, vp)
    sig("rluref_seq_n", i64, vp)
    sig("rluref_seq_nnz", i64, vp)
    sig("rluref_seq_mu", dbl, vp, i64)
    sig("rluref_seq_pattern", None, vp, vp, vp)
    sig("rluref_seq_values", None, vp, i64, vp)
    sig("rluref_seq_rhs", None, vp, i64, vp)
    sig("rluref_seq_matrix", vp, vp, i64)
    sig("rluref_analyze", vp, vp, i32, i32, P(dbl))
    sig("rluref_sym_destroy", None, vp)
    sig("rluref_sym_n", i64, vp)
    sig("rluref_sym_nnz_factors", i64, vp)
    sig("rluref_sym_nnz_source", i64, vp)
    sig("rluref_sym_fill_count", i64, vp)
    sig("rluref_sym_has_match", i32, vp)
    sig("rluref_sym_pattern", None, vp, vp, vp, vp)
    sig("rluref_sym_scatter", None, vp, vp, vp)
    sig("rluref_sym_source_pattern", None, vp, vp, vp)
    sig("rluref_sym_amd", None, vp, vp)
    sig("rluref_sym_match", None, vp, vp, vp, vp)
    sig("rluref_sym_hash_rows", i64, vp)
    sig("rluref_numeric_create", vp, vp, dbl, i32, i32)
    sig("rluref_numeric_destroy", None, vp)
    sig("rluref_numeric_set_exec", None, vp, i32, i32)
    sig("rluref_numeric_set_solve_exec", None, vp, i32, i32)
    sig("rluref_reset_values", i32, vp, vp)
    sig("rluref_factorize_scattered", i32, vp)
    sig("rluref_refactorize", i32, vp, vp)
    sig("rluref_numeric_valid", i32, vp)
    sig("rluref_numeric_generation", u64, vp)
    sig("rluref_numeric_get_values", None, vp, vp)
    sig("rluref_numeric_set_values", None, vp, vp, i32)
    sig("rluref_lower_solve", i32, vp, i64, vp, vp)
    sig("rluref_upper_solve", i32, vp, i64, vp, vp)
    sig("rluref_solve_system", i32, vp, i64, vp, vp)
    sig("rluref_workspace_allocation_events", u64, vp)
    sig("rluref_spmv", i32, vp, vp, vp)
    sig("rluref_relative_residual", dbl, vp, vp, vp)
    sig("rluref_dot", dbl, i64, vp, vp)
    sig("rluref_norm2", dbl, i64, vp)
    sig("rluref_refine", i32, vp, vp, vp, vp, i32, i32, dbl, vp, P(i32), P(i32), vp, P(i32))
    sig("rluref_cgs2", i32, i64, i64, vp, vp, vp, vp, P(dbl), P(i32))
    sig("rluref_run_system", i32, vp, vp, i64, i32, i32, dbl, vp, P(dbl), P(dbl), P(i32), vp)
    _lib = L
    return L


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _check(status: int):
    if status != OK:
        L = lib()
        raise RefError(status, L.rluref_last_error().decode(), int(L.rluref_last_row()))


def max_threads() -> int:
    return int(lib().rluref_max_threads())


class RefRng:
    """std::mt19937_64 held on the C++ side so seeded test loops replay exactly."""

    def __init__(self, seed: int):
        self._h = lib().rluref_rng_create(seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().rluref_rng_destroy(self._h)
            self._h = None

    def uniform_int(self, lo: int, hi: int) -> int:
        return int(lib().rluref_rng_uniform_int(self._h, lo, hi))

    def uniform_real(self, lo: float, hi: float) -> float:
        return float(lib().rluref_rng_uniform_real(self._h, lo, hi))

    def random_sparse(self, n, extra_per_row, lo, hi, diagonally_dominant) -> "RefCsr":
        """oracle::random_sparse, proj/tests/oracles.hpp:186-210."""
        return RefCsr(lib().rluref_random_sparse(self._h, n, extra_per_row, lo, hi,
                                                 1 if diagonally_dominant else 0), owned=True)

    def random_vector(self, n, lo=-1.0, hi=1.0) -> np.ndarray:
        """oracle::random_vector, proj/tests/oracles.hpp:212-218."""
        out = np.empty(n, dtype=np.float64)
        lib().rluref_random_vector(self._h, n, lo, hi, _p(out))
        return out


class RefCsr:
    def __init__(self, handle, owned: bool, keepalive=None):
        self._h = handle
        self._owned = owned
        self._keep = keepalive

    @classmethod
    def from_arrays(cls, n, row_offsets, cols, values=None) -> "RefCsr":
        ro, ci = _i64(row_offsets), _i64(cols)
        v = None if values is None else _f64(values)
        return cls(lib().rluref_csr_create(n, _p(ro), _p(ci), _p(v)), owned=True)

    @classmethod
    def from_dense(cls, M) -> "RefCsr":
        M = np.asarray(M, dtype=np.float64)
        n = M.shape[0]
        ro, ci, v = [0], [], []
        for i in range(n):
            for j in range(M.shape[1]):
                if M[i, j] != 0.0:
                    ci.append(j)
                    v.append(M[i, j])
            ro.append(len(ci))
        return cls.from_arrays(n, ro, ci, v)

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None):
            lib().rluref_csr_destroy(self._h)
            self._h = None

    @property
    def n(self) -> int:
        return int(lib().rluref_csr_n(self._h))

    @property
    def nnz(self) -> int:
        return int(lib().rluref_csr_nnz(self._h))

    def arrays(self):
        ro = np.empty(self.n + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int64)
        v = np.empty(self.nnz, dtype=np.float64)
        lib().rluref_csr_get(self._h, _p(ro), _p(ci), _p(v))
        return ro, ci, v

    def set_values(self, values):
        v = _f64(values)
        assert v.size == self.nnz
        lib().rluref_csr_set_values(self._h, _p(v))

    def spmv(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty(self.n, dtype=np.float64)
        _check(lib().rluref_spmv(self._h, _p(x), _p(y)))
        return y

    def relative_residual(self, x, b) -> float:
        x, b = _f64(x), _f64(b)
        return float(lib().rluref_relative_residual(self._h, _p(x), _p(b)))

    def to_dense(self) -> np.ndarray:
        ro, ci, v = self.arrays()
        M = np.zeros((self.n, self.n))
        for i in range(self.n):
            M[i, ci[ro[i]:ro[i + 1]]] = v[ro[i]:ro[i + 1]]
        return M


class RefSequence:
    """gen_sequence(GenConfig) — proj/src/kkt.cpp:94-207, defaults proj/include/rlu/kkt.hpp:49-60."""

    def __init__(self, n, m, topology_seed=1, y_seed=2, num_systems=0, mu0=1e-1, mu_min=1e-7,
                 reduction=0.2, delta_p=1e-8, delta_d=1e-8, keep_blocks=False):
        gen = lib().rluref_gen_sequence_blocks if keep_blocks else lib().rluref_gen_sequence
        self._h = gen(n, m, topology_seed, y_seed, num_systems, mu0, mu_min, reduction, delta_p, delta_d)
        if not self._h:
            raise RefError(ERROR, lib().rluref_last_error().decode())
        self.n_primal, self.m_dual = n, m

    def __del__(self):
        if getattr(self, "_h", None):
            lib().rluref_seq_destroy(self._h)
            self._h = None

    def __len__(self):
        return int(lib().rluref_seq_num_systems(self._h))

    @property
    def n(self) -> int:
        return int(lib().rluref_seq_n(self._h))

    @property
    def nnz(self) -> int:
        return int(lib().rluref_seq_nnz(self._h))

    def pattern(self):
        ro = np.empty(self.n + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int64)
        lib().rluref_seq_pattern(self._h, _p(ro), _p(ci))
        return ro, ci

    def values(self, k) -> np.ndarray:
        v = np.empty(self.nnz, dtype=np.float64)
        lib().rluref_seq_values(self._h, k, _p(v))
        return v

    def rhs(self, k) -> np.ndarray:
        b = np.empty(self.n, dtype=np.float64)
        lib().rluref_seq_rhs(self._h, k, _p(b))
        return b

    def mu(self, k) -> float:
        return float(lib().rluref_seq_mu(self._h, k))

    # -- KktBlocks of step k (include/rlu/kkt.hpp:14-21); only with keep_blocks=True
    def h_diag(self, k=0) -> np.ndarray:
        out = np.empty(self.n_primal, dtype=np.float64)
        lib().rluref_seq_h_diag(self._h, k, _p(out))
        return out

    def d_y(self, k) -> np.ndarray:
        out = np.empty(self.n_primal, dtype=np.float64)
        lib().rluref_seq_dy(self._h, k, _p(out))
        return out

    def deltas(self, k):
        dp, dd = C.c_double(), C.c_double()
        lib().rluref_seq_deltas(self._h, k, C.byref(dp), C.byref(dd))
        return float(dp.value), float(dd.value)

    def double_regularization(self, k):
        """The regularization step of cli::solve_sequence's escalation (src/cli.cpp:53, 148-154)."""
        _check(lib().rluref_seq_double_regularization(self._h, k))

    def matrix(self, k) -> RefCsr:
        return RefCsr(lib().rluref_seq_matrix(self._h, k), owned=False, keepalive=self)


@dataclass
class SymbolicArrays:
    """Plain-array image of rlu::SymbolicFactors (proj/include/rlu/symbolic.hpp:48-59)."""
    n: int
    row_offsets: np.ndarray   # combined_pattern.row_offsets, int64[n+1]
    col_indices: np.ndarray   # combined_pattern.col_indices, int64[nnzF]
    diag_pos: np.ndarray      # int64[n]
    scatter_map: np.ndarray   # int64[nnzA]
    scatter_scale: np.ndarray  # f64[nnzA]
    amd_forward: np.ndarray   # int64[n]
    src_row_offsets: np.ndarray
    src_col_indices: np.ndarray
    col_perm_forward: np.ndarray | None = None  # match->col_perm.forward
    row_scale: np.ndarray | None = None
    col_scale: np.ndarray | None = None
    fill_count: int = 0


class RefSymbolic:
    def __init__(self, A: RefCsr, use_scaling=True, use_amd=True):
        ms = C.c_double(0.0)
        self._h = lib().rluref_analyze(A._h, 1 if use_scaling else 0, 1 if use_amd else 0,
                                       C.byref(ms))
        if not self._h:
            L = lib()
            raise RefError(ERROR, L.rluref_last_error().decode(), int(L.rluref_last_row()))
        self.analyze_ms = ms.value

    def __del__(self):
        if getattr(self, "_h", None):
            lib().rluref_sym_destroy(self._h)
            self._h = None

    @property
    def n(self):
        return int(lib().rluref_sym_n(self._h))

    @property
    def nnz_factors(self):
        return int(lib().rluref_sym_nnz_factors(self._h))

    @property
    def nnz_source(self):
        return int(lib().rluref_sym_nnz_source(self._h))

    @property
    def hash_rows(self):
        return int(lib().rluref_sym_hash_rows(self._h))

    def arrays(self) -> SymbolicArrays:
        L = lib()
        n, nf, na = self.n, self.nnz_factors, self.nnz_source
        ro = np.empty(n + 1, dtype=np.int64)
        ci = np.empty(nf, dtype=np.int64)
        dp = np.empty(n, dtype=np.int64)
        L.rluref_sym_pattern(self._h, _p(ro), _p(ci), _p(dp))
        sm = np.empty(na, dtype=np.int64)
        ss = np.empty(na, dtype=np.float64)
        L.rluref_sym_scatter(self._h, _p(sm), _p(ss))
        amd = np.empty(n, dtype=np.int64)
        L.rluref_sym_amd(self._h, _p(amd))
        sro = np.empty(n + 1, dtype=np.int64)
        sci = np.empty(na, dtype=np.int64)
        L.rluref_sym_source_pattern(self._h, _p(sro), _p(sci))
        out = SymbolicArrays(n, ro, ci, dp, sm, ss, amd, sro, sci,
                             fill_count=int(L.rluref_sym_fill_count(self._h)))
        if L.rluref_sym_has_match(self._h):
            q = np.empty(n, dtype=np.int64)
            dr = np.empty(n, dtype=np.float64)
            dc = np.empty(n, dtype=np.float64)
            L.rluref_sym_match(self._h, _p(q), _p(dr), _p(dc))
            out.col_perm_forward, out.row_scale, out.col_scale = q, dr, dc
        return out


class RefNumeric:
    """NumericFactors + a private SolveWorkspace; entry points of numeric.hpp:42-53, trisolve.hpp:23-39."""

    def __init__(self, sym: RefSymbolic, pivot_floor=1e-30, parallel=False, workers=0):
        self._sym = sym
        self._h = lib().rluref_numeric_create(sym._h, pivot_floor, 1 if parallel else 0, workers)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().rluref_numeric_destroy(self._h)
            self._h = None

    def set_exec(self, parallel: bool, workers=0):
        lib().rluref_numeric_set_exec(self._h, 1 if parallel else 0, workers)

    def set_solve_exec(self, parallel: bool, workers=0):
        """ExecPolicy handed to solve_system only (include/rlu/trisolve.hpp:36)."""
        lib().rluref_numeric_set_solve_exec(self._h, 1 if parallel else 0, workers)

    def reset_values(self, A: RefCsr):
        _check(lib().rluref_reset_values(self._h, A._h))

    def factorize_scattered(self):
        _check(lib().rluref_factorize_scattered(self._h))

    def refactorize(self, A: RefCsr):
        _check(lib().rluref_refactorize(self._h, A._h))

    @property
    def valid(self) -> bool:
        return bool(lib().rluref_numeric_valid(self._h))

    @property
    def generation(self) -> int:
        return int(lib().rluref_numeric_generation(self._h))

    def values(self) -> np.ndarray:
        v = np.empty(self._sym.nnz_factors, dtype=np.float64)
        lib().rluref_numeric_get_values(self._h, _p(v))
        return v

    def set_values(self, values, valid=True):
        v = _f64(values)
        assert v.size == self._sym.nnz_factors
        lib().rluref_numeric_set_values(self._h, _p(v), 1 if valid else 0)

    def _vec_call(self, fn, y):
        y = _f64(y)
        x = np.empty(self._sym.n, dtype=np.float64)
        _check(fn(self._h, y.size, _p(y), _p(x)))
        return x

    def lower_solve(self, y):
        return self._vec_call(lib().rluref_lower_solve, y)

    def upper_solve(self, y):
        return self._vec_call(lib().rluref_upper_solve, y)

    def solve_system(self, b):
        return self._vec_call(lib().rluref_solve_system, b)

    @property
    def workspace_allocation_events(self) -> int:
        return int(lib().rluref_workspace_allocation_events(self._h))

    def run_system(self, seq: RefSequence, k: int, refine=True, max_iterations=20,
                   tolerance=1e-14, want_x=False):
        """Timed pass mirroring cli::solve_sequence (proj/src/cli.cpp:105-135)."""
        times = np.zeros(4, dtype=np.float64)
        rd, rf, it = C.c_double(), C.c_double(), C.c_int()
        x = np.empty(self._sym.n, dtype=np.float64) if want_x else None
        _check(lib().rluref_run_system(self._h, seq._h, k, 1 if refine else 0, max_iterations,
                                       tolerance, _p(times), C.byref(rd), C.byref(rf),
                                       C.byref(it), _p(x)))
        return dict(scatter_ms=times[0], factor_ms=times[1], trisolve_ms=times[2],
                    refine_ms=times[3], relres_direct=rd.value, relres_final=rf.value,
                    refine_iters=it.value, x=x)


@dataclass
class RefineResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_history: np.ndarray


def refine(A: RefCsr, b, x0, precond: RefNumeric | None, method="fgmres", max_iterations=20,
           tolerance=1e-14) -> RefineResult:
    """fgmres_refine / classic_refine (proj/src/refine.cpp:39-188); precond=None is the identity."""
    b, x0 = _f64(b), _f64(x0)
    x = np.empty(A.n, dtype=np.float64)
    hist = np.zeros(max(1, max_iterations) + 2, dtype=np.float64)
    it, conv, hl = C.c_int(), C.c_int(), C.c_int()
    _check(lib().rluref_refine(A._h, _p(b), _p(x0), precond._h if precond else None,
                               0 if method == "fgmres" else 1, max_iterations, tolerance, _p(x),
                               C.byref(it), C.byref(conv), _p(hist), C.byref(hl)))
    return RefineResult(x, it.value, bool(conv.value), hist[:hl.value].copy())


def cgs2(basis: np.ndarray, v: np.ndarray):
    """cgs2_orthonormalize (proj/src/refine.cpp:8-26); basis is (k, n) row-major."""
    basis = _f64(basis).reshape(-1, v.size) if basis.size else np.zeros((0, v.size))
    v = _f64(v)
    k, n = basis.shape
    coef = np.zeros(max(k, 1), dtype=np.float64)
    out = np.empty(n, dtype=np.float64)
    norm, bd = C.c_double(), C.c_int()
    _check(lib().rluref_cgs2(n, k, _p(basis), _p(v), _p(coef), _p(out), C.byref(norm),
                             C.byref(bd)))
    return coef[:k], out, norm.value, bool(bd.value)
