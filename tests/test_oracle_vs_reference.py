"""Pins the plain-C oracle (oracle/rlu_oracle.c) to the UNMODIFIED reference (oracle/_ref), bit for bit.

Seeded loops replay the reference's own test generators (proj/tests/oracles.hpp:186-218) in the
shapes its tests use (proj/tests/test_numeric.cpp, test_trisolve.cpp, test_refine.cpp).
"""
import numpy as np
import pytest

from oracle import oraclebridge as ob
from oracle import refbridge as rb

pytestmark = pytest.mark.skipif(not rb.available(), reason="oracle/_ref/librlu_ref.so not built")


def _pair(A, use_scaling=True, use_amd=True):
    sym = rb.RefSymbolic(A, use_scaling=use_scaling, use_amd=use_amd)
    return sym, ob.Factors(sym.arrays()), rb.RefNumeric(sym)


@pytest.mark.parametrize("scaling,amd", [(True, True), (False, True), (False, False)])
def test_scatter_and_eliminate_bitwise_on_random_sparse(scaling, amd):
    rng = rb.RefRng(91)  # test_numeric.cpp:186-195 draws sizes 2..60 from rng(91)
    for _ in range(40):
        A = rng.random_sparse(rng.uniform_int(2, 60), 5, 0.1, 1.0, True)
        sym, F, num = _pair(A, scaling, amd)
        v = A.arrays()[2]
        num.reset_values(A)
        scattered = num.values()
        assert np.array_equal(scattered, F.scatter_values(v))
        num.factorize_scattered()
        lu, failed = F.eliminate(scattered)
        assert failed == -1
        assert np.array_equal(num.values(), lu)


def test_zero_pivot_row_matches_reference():
    # test_numeric.cpp:173-184: hard zero pivot at elimination step 1 in natural order
    A = rb.RefCsr.from_dense([[1, 1, 0], [1, 1, 1], [0, 1, 1]])
    sym, F, num = _pair(A, False, False)
    with pytest.raises(rb.RefError) as e:
        num.refactorize(A)
    assert e.value.status == rb.ZERO_PIVOT and e.value.row == 1
    _, failed = F.factorize(A.arrays()[2])
    assert failed == 1


def test_pivot_floor_threshold_matches_reference():
    A = rb.RefCsr.from_dense([[1e-3, 1.0], [1.0, 1.0]])
    sym = rb.RefSymbolic(A, use_scaling=False, use_amd=False)
    F = ob.Factors(sym.arrays())
    for floor, expect in ((1e-30, -1), (1e-3, 0), (1e-2, 0)):
        num = rb.RefNumeric(sym, pivot_floor=floor)
        try:
            num.refactorize(A)
            got = -1
        except rb.RefError as e:
            got = e.row
        assert got == expect
        assert F.factorize(A.arrays()[2], pivot_floor=floor)[1] == expect


@pytest.mark.parametrize("scaling", [True, False])
def test_triangular_solves_and_composition_bitwise(scaling):
    rng = rb.RefRng(303)  # test_trisolve.cpp:129-153
    for _ in range(10):
        n = rng.uniform_int(10, 200)
        A = rng.random_sparse(n, 5, 0.1, 1.0, True)
        sym, F, num = _pair(A, scaling, True)
        num.refactorize(A)
        lu = num.values()
        b = rng.random_vector(n)
        assert np.array_equal(num.lower_solve(b), F.lower_solve(lu, b))
        xu, failed = F.upper_solve(lu, b)
        assert failed == -1 and np.array_equal(num.upper_solve(b), xu)
        xs, failed = F.solve_system(lu, b)
        assert failed == -1 and np.array_equal(num.solve_system(b), xs)


def test_upper_solve_zero_diagonal_row():
    # test_trisolve.cpp:171-184: crafted 1x1 factor with a zero diagonal -> row 0
    A = rb.RefCsr.from_dense([[1.0]])
    sym, F, num = _pair(A, False, False)
    num.refactorize(A)
    num.set_values(np.array([0.0]))
    with pytest.raises(rb.RefError) as e:
        num.upper_solve(np.array([1.0]))
    assert e.value.status == rb.ZERO_PIVOT and e.value.row == 0
    _, failed = F.upper_solve(np.array([0.0]), np.array([1.0]))
    assert failed == 0


def test_spmv_dot_residual_bitwise():
    rng = rb.RefRng(11)
    for _ in range(5):
        n = rng.uniform_int(5, 300)
        A = rng.random_sparse(n, 6, 0.1, 1.0, False)
        ro, ci, v = A.arrays()
        Ao = ob.Csr(n, ro, ci, v)
        x, b = rng.random_vector(n), rng.random_vector(n)
        assert np.array_equal(A.spmv(x), Ao.spmv(x))
        assert A.relative_residual(x, b) == Ao.relative_residual(x, b)
        L = rb.lib()
        assert L.rluref_dot(n, x.ctypes.data, b.ctypes.data) == ob.dot(x, b)
        assert L.rluref_norm2(n, x.ctypes.data) == ob.norm2(x)
    z = np.zeros(4)
    assert rb.RefCsr.from_dense(np.eye(4)).relative_residual(z, z) == 0.0  # denominator clamp


def test_cgs2_bitwise():
    rng = rb.RefRng(71)  # test_refine.cpp:58-79
    n = 50
    basis = []
    for k in range(12):
        v = rng.random_vector(n)
        if basis:
            v = basis[0] + 1e-9 * v
        B = np.array(basis) if basis else np.zeros((0, n))
        c1, v1, n1, bd1 = rb.cgs2(B, v)
        c2, v2, n2, bd2 = ob.cgs2(B, v)
        assert bd1 == bd2 and n1 == n2
        assert np.array_equal(c1, c2) and np.array_equal(v1, v2)
        basis.append(v1)
    # breakdown on exact membership (test_refine.cpp:52-56)
    e0 = np.eye(3)[0]
    assert rb.cgs2(e0[None, :], e0)[3] and ob.cgs2(e0[None, :], e0)[3]


@pytest.mark.parametrize("method", ["fgmres", "classic"])
def test_refinement_bitwise_with_lu_preconditioner(method):
    rng = rb.RefRng(76)  # test_refine.cpp:219-242
    for _ in range(12):
        n = rng.uniform_int(5, 150)
        A = rng.random_sparse(n, 5, 0.1, 1.0, True)
        sym, F, num = _pair(A)
        num.refactorize(A)
        lu = num.values()
        ro, ci, v = A.arrays()
        Ao = ob.Csr(n, ro, ci, v)
        b = rng.random_vector(n)
        x0 = num.solve_system(b)
        r = rb.refine(A, b, x0, num, method=method)
        x, it, conv, hist = ob.refine(Ao, b, x0, F, lu, method=method)
        assert (r.iterations, r.converged) == (it, conv)
        assert np.array_equal(r.x, x) and np.array_equal(r.residual_history, hist)


def test_fgmres_bitwise_identity_preconditioner_full_cycle():
    rng = rb.RefRng(73)  # test_refine.cpp:120-133: tolerance 1e-30 forces the full cycle
    for _ in range(6):
        A = rng.random_sparse(50, 4, 0.1, 1.0, True)
        b = rng.random_vector(50)
        ro, ci, v = A.arrays()
        r = rb.refine(A, b, np.zeros(50), None, max_iterations=15, tolerance=1e-30)
        x, it, conv, hist = ob.refine(ob.Csr(50, ro, ci, v), b, np.zeros(50), None, None,
                                      max_iterations=15, tolerance=1e-30)
        assert (r.iterations, r.converged) == (it, conv) == (15, False)
        assert np.array_equal(r.x, x) and np.array_equal(r.residual_history, hist)


@pytest.mark.parametrize("scaling", [False, True])
def test_kkt_sequence_bitwise(scaling):
    # acceptance.cpp:236-272 shape, shrunk: analyze once, refactorize the rest
    seq = rb.RefSequence(700, 300)
    sym = rb.RefSymbolic(seq.matrix(0), use_scaling=scaling, use_amd=True)
    F, num = ob.Factors(sym.arrays()), rb.RefNumeric(sym)
    ro, ci = seq.pattern()
    for k in range(len(seq)):
        A, b = seq.matrix(k), seq.rhs(k)
        num.refactorize(A)
        lu, failed = F.factorize(seq.values(k))
        assert failed == -1 and np.array_equal(num.values(), lu)
        x0 = num.solve_system(b)
        assert np.array_equal(x0, F.solve_system(lu, b)[0])
        r = rb.refine(A, b, x0, num)
        x, it, conv, hist = ob.refine(ob.Csr(seq.n, ro, ci, seq.values(k)), b, x0, F, lu)
        assert np.array_equal(r.x, x) and it == r.iterations and conv == r.converged
        assert A.relative_residual(x, b) <= 1e-8  # kAcceptRelres, cli.hpp:25
