"""The oracle against known answers of the reference's tests and the committed fixtures.

These run without the reference tree or its bridge: tests/golden/*.npz hold inputs, the reference's
analysis arrays and the reference's outputs (made by tests/golden/make_golden.py).
"""
import numpy as np
import pytest

from oracle import oraclebridge as ob
from tests.fixtures import golden_fixture


class _Sym:
    """Natural-order, no-fill symbolic arrays for tiny dense matrices (use_scaling = use_amd = false)."""

    def __init__(self, M):
        M = np.asarray(M, dtype=float)
        n = M.shape[0]
        # fill pattern by symbolic elimination (proj/tests/oracles.hpp:112-123)
        P = M != 0
        for k in range(n):
            for i in range(k + 1, n):
                if P[i, k]:
                    P[i, k + 1:] |= P[k, k + 1:]
        ro, ci, dp, smap = [0], [], [], []
        for i in range(n):
            for j in range(n):
                if P[i, j]:
                    if j == i:
                        dp.append(len(ci))
                    if M[i, j] != 0:
                        smap.append(len(ci))
                    ci.append(j)
            ro.append(len(ci))
        self.n = n
        self.row_offsets, self.col_indices, self.diag_pos = map(np.array, (ro, ci, dp))
        self.scatter_map = np.array(smap)
        self.scatter_scale = np.ones(len(smap))
        self.amd_forward = np.arange(n)
        self.col_perm_forward = self.row_scale = self.col_scale = None
        self.a_values = M[M != 0]

    def find(self, i, j):
        lo, hi = self.row_offsets[i], self.row_offsets[i + 1]
        return lo + list(self.col_indices[lo:hi]).index(j)


def _factor(M, floor=1e-30):
    s = _Sym(M)
    F = ob.Factors(s)
    lu, failed = F.factorize(s.a_values, floor)
    return s, F, lu, failed


def test_scatter_arrow_matrix_zeroes_exactly_the_fill_slots():
    # test_numeric.cpp:105-123
    s = _Sym([[4, 1, 1, 1], [1, 3, 0, 0], [1, 0, 3, 0], [1, 0, 0, 3]])
    vals = ob.Factors(s).scatter_values(s.a_values)
    assert vals.size == 16 and int((vals == 0.0).sum()) == 6


def test_scatter_identity_puts_ones_on_the_diagonal():
    # test_numeric.cpp:125-133
    s = _Sym(np.eye(5))
    assert np.array_equal(ob.Factors(s).scatter_values(s.a_values), np.ones(5))


def test_dense_2x2_hand_elimination():
    # test_numeric.cpp:142-157: l10 = 1.5, U = [[4, 3], [0, -1.5]]
    s, F, lu, failed = _factor([[4, 3], [6, 3]])
    assert failed == -1
    assert lu[s.find(1, 0)] == 1.5 and lu[s.diag_pos[0]] == 4.0
    assert lu[s.find(0, 1)] == 3.0 and lu[s.diag_pos[1]] == -1.5


def test_scaling_the_matrix_scales_u_only():
    # test_numeric.cpp:159-171
    s, F, f1, _ = _factor([[4, 3], [6, 3]])
    _, _, f2, _ = _factor([[8, 6], [12, 6]])
    assert f1[s.find(1, 0)] == f2[s.find(1, 0)]
    assert 2.0 * f1[s.diag_pos[0]] == f2[s.diag_pos[0]] and 2.0 * f1[s.diag_pos[1]] == f2[s.diag_pos[1]]


def test_zero_pivot_reports_row_1():
    # test_numeric.cpp:173-184
    assert _factor([[1, 1, 0], [1, 1, 1], [0, 1, 1]])[3] == 1


def test_trisolve_known_answers():
    # test_trisolve.cpp:56-88
    s, F, lu, _ = _factor([[1, 0], [0, 1]])
    assert np.array_equal(F.lower_solve(lu, [3, 4]), [3, 4])
    assert np.array_equal(F.upper_solve(lu, [5, 6])[0], [5, 6])
    s, F, lu, _ = _factor([[1, 0], [2, 1]])
    assert np.array_equal(F.lower_solve(lu, [1, 4]), [1, 2])
    M = np.eye(4) - np.eye(4, k=-1)
    s, F, lu, _ = _factor(M)
    assert np.array_equal(F.lower_solve(lu, np.ones(4)), [1, 2, 3, 4])
    s, F, lu, _ = _factor([[2, 1], [0, 4]])
    assert np.array_equal(F.upper_solve(lu, [4, 8])[0], [1, 2])
    s, F, lu, _ = _factor([[2, 0], [0, 4]])
    assert np.array_equal(F.upper_solve(lu, [2, 8])[0], [1, 2])


def test_solve_system_forced_2x2():
    # test_trisolve.cpp:90-100
    s, F, lu, _ = _factor([[4, 3], [6, 3]])
    x, failed = F.solve_system(lu, [10, 12])
    assert failed == -1 and np.allclose(x, [1, 2], rtol=1e-14)


def test_fgmres_diagonal_system_identity_preconditioner():
    # test_refine.cpp:98-118
    A = ob.Csr(3, [0, 1, 2, 3], [0, 1, 2], [1, 2, 3])
    x, it, conv, hist = ob.refine(A, [1, 2, 3], np.zeros(3))
    assert conv and it <= 3 and np.allclose(x, 1.0, rtol=1e-12)
    A = ob.Csr(2, [0, 1, 2], [0, 1], [2, 2])
    x, it, conv, hist = ob.refine(A, [2, 2], [1, 1])
    assert conv and it == 0 and np.array_equal(x, [1, 1])


def test_fgmres_reports_non_convergence():
    # test_refine.cpp:148-159
    A = ob.Csr(3, [0, 1, 2, 3], [0, 1, 2], [1, 1e-8, 1])
    x, it, conv, hist = ob.refine(A, [1, 1, 1], np.zeros(3), max_iterations=2, tolerance=1e-16)
    assert not conv and it == 2


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_60", "random_sparse_120_plain"])
def test_oracle_reproduces_committed_reference_outputs(name):
    fx = golden_fixture(name)
    g = fx.golden
    for k in range(len(fx.values)):
        scattered = fx.oracle.scatter_values(fx.values[k])
        assert np.array_equal(scattered, g[f"scattered_{k}"])
        lu, failed = fx.oracle.eliminate(scattered)
        assert failed == -1 and np.array_equal(lu, g[f"lu_{k}"])
        assert np.array_equal(fx.oracle.lower_solve(lu, fx.rhs[k]), g[f"lower_{k}"])
        assert np.array_equal(fx.oracle.upper_solve(lu, fx.rhs[k])[0], g[f"upper_{k}"])
        x = fx.oracle.solve_system(lu, fx.rhs[k])[0]
        assert np.array_equal(x, g[f"x_{k}"])
        assert fx.oracle_csr(k).relative_residual(x, fx.rhs[k]) == float(g[f"relres_{k}"])
        xr, it, conv, hist = ob.refine(fx.oracle_csr(k), fx.rhs[k], x, fx.oracle, lu)
        assert np.array_equal(xr, g[f"xref_{k}"]) and it == int(g[f"iters_{k}"])
        assert np.array_equal(hist, g[f"hist_{k}"])
