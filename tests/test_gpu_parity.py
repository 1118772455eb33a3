"""Parity of the CUDA path (through the C ABI) with the oracle, on the B200.

Each test restates a reference test (proj/tests/test_numeric.cpp, test_trisolve.cpp,
test_refine.cpp, acceptance.cpp) against the device implementation. Integer/index work and the
L/U values, triangular solves and SpMV are compared BIT-EXACT; refinement — whose dot products are
parallel sums on the device — is compared on the residual, with the tolerance written in the test.
"""
import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from oracle import oraclebridge as ob
from oracle import refbridge as rb
from tests.fixtures import csr_fixture, dense_fixture, golden_fixture, kkt_fixture

pytestmark = pytest.mark.gpu
# The U sweep's summation order is selectable (include/b200lu.h, B200LU_FLAG_STRICT_ORDER): bitwise
# comparisons of upper_solve / solve_system use the reference's order; the default (device
# order) is covered by test_default_sweep_order_* on the residual.
STRICT = rlu.FactorOptions(strict_order=True)
needs_ref = pytest.mark.skipif(not rb.available(), reason="oracle/_ref/librlu_ref.so not built")


# ------------------------------------------------------------------ scatter

@needs_ref
def test_scatter_places_entries_and_zeroes_fill_slots():
    # test_numeric.cpp:105-123
    fx = dense_fixture([[4, 1, 1, 1], [1, 3, 0, 0], [1, 0, 3, 0], [1, 0, 0, 3]])
    assert fx.sym.fill_count == 6
    vals = rlu.scatter_values(fx.sym, fx.matrix())
    assert vals.size == 16 and int((vals == 0.0).sum()) == 6
    assert np.array_equal(vals, fx.oracle.scatter_values(fx.values[0]))
    ident = rlu.CsrMatrix(4, 4, np.arange(5), np.arange(4), np.ones(4))
    f = rlu.NumericFactors(fx.sym)
    with pytest.raises(rlu.PatternMismatchError):
        rlu.reset_values(f, ident)
    no_values = rlu.CsrMatrix(4, 4, fx.ro, fx.ci, None)
    with pytest.raises(rlu.Error):
        rlu.reset_values(f, no_values)


@needs_ref
def test_scatter_identity_and_identity_factors():
    # test_numeric.cpp:125-140
    fx = dense_fixture(np.eye(5), use_scaling=True, use_amd=True)
    assert np.array_equal(rlu.scatter_values(fx.sym, fx.matrix()), np.ones(5))
    f = rlu.factorize(fx.sym, fx.matrix())
    assert np.array_equal(f.values[fx.sym.diag_pos], np.ones(5))


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_60", "random_sparse_120_plain"])
def test_committed_fixtures_bitwise(name):
    """Inputs + the reference's outputs from tests/golden (no reference needed at run time)."""
    fx = golden_fixture(name)
    g = fx.golden
    f = rlu.NumericFactors(fx.sym, STRICT)
    for k in range(len(fx.values)):
        rlu.reset_values(f, fx.matrix(k))
        assert not f.valid
        assert np.array_equal(f.values, g[f"scattered_{k}"])
        rlu.factorize_scattered(f)
        assert f.valid and f.generation == k + 1
        assert np.array_equal(f.values, g[f"lu_{k}"])
        assert np.array_equal(rlu.lower_solve(f, fx.rhs[k]), g[f"lower_{k}"])
        assert np.array_equal(rlu.upper_solve(f, fx.rhs[k]), g[f"upper_{k}"])
        x = rlu.solve_system(f, fx.rhs[k])
        assert np.array_equal(x, g[f"x_{k}"])
        out = rlu.fgmres_refine(f, fx.rhs[k], x)
        ref_final = fx.oracle_csr(k).relative_residual(g[f"xref_{k}"], fx.rhs[k])
        got_final = fx.oracle_csr(k).relative_residual(out.x, fx.rhs[k])
        # north star: residual at or below the reference's after refinement; both sit at the
        # rounding floor (~1e-16), where "at or below" is meaningful only up to a few ulps of it.
        assert got_final <= max(ref_final * 4, 1e-15), (got_final, ref_final)
        assert out.iterations == int(g[f"iters_{k}"])


# ------------------------------------------------------------- factorization

@needs_ref
def test_dense_2x2_hand_elimination_and_scaling():
    # test_numeric.cpp:142-171
    fx = dense_fixture([[4, 3], [6, 3]])
    f1 = rlu.factorize(fx.sym, fx.matrix())
    v = f1.values
    find = lambda i, j: fx.sym.row_offsets[i] + list(fx.sym.col_indices[fx.sym.row_offsets[i]:fx.sym.row_offsets[i + 1]]).index(j)
    assert v[find(1, 0)] == 1.5 and v[fx.sym.diag_pos[0]] == 4.0 and v[find(0, 1)] == 3.0
    assert v[fx.sym.diag_pos[1]] == -1.5
    f2 = rlu.factorize(fx.sym, fx.matrix(values=2.0 * fx.values[0]))
    v2 = f2.values
    assert v[find(1, 0)] == v2[find(1, 0)]
    assert 2.0 * v[fx.sym.diag_pos[0]] == v2[fx.sym.diag_pos[0]] and 2.0 * v[fx.sym.diag_pos[1]] == v2[fx.sym.diag_pos[1]]


@needs_ref
def test_zero_pivot_reports_lowest_row_and_invalidates():
    # test_numeric.cpp:173-184, 328-336
    fx = dense_fixture([[1, 1, 0], [1, 1, 1], [0, 1, 1]])
    f = rlu.NumericFactors(fx.sym)
    with pytest.raises(rlu.ZeroPivotError) as e:
        rlu.refactorize(f, fx.matrix())
    assert e.value.row == 1
    assert not f.valid and f.generation == 0
    with pytest.raises(rlu.Error):
        rlu.solve_system(f, np.ones(3))


@needs_ref
def test_pivot_floor_threshold():
    fx = dense_fixture([[1e-3, 1.0], [1.0, 1.0]])
    for floor, expect in ((1e-30, None), (1e-3, 0), (1e-2, 0)):
        f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(pivot_floor=floor))
        if expect is None:
            rlu.refactorize(f, fx.matrix())
            assert f.valid
        else:
            with pytest.raises(rlu.ZeroPivotError) as e:
                rlu.refactorize(f, fx.matrix())
            assert e.value.row == expect


@needs_ref
@pytest.mark.parametrize("scaling,amd", [(True, True), (False, True), (False, False)])
def test_lu_values_bitwise_on_random_sparse(scaling, amd):
    # test_numeric.cpp:186-221 shapes; expected = oracle (itself pinned bitwise to the reference)
    rng = rb.RefRng(91)
    for _ in range(40):
        A = rng.random_sparse(rng.uniform_int(2, 60), 5, 0.1, 1.0, True)
        fx = csr_fixture(A, scaling, amd)
        f = rlu.factorize(fx.sym, fx.matrix())
        expect, failed = fx.oracle.factorize(fx.values[0])
        assert failed == -1 and np.array_equal(f.values, expect)
        f.close()


@needs_ref
def test_lu_values_bitwise_with_32_bit_destination_tables(monkeypatch):
    """factor_kernel<uint32_t, ...>: the destination table of patterns with rows of more than 65 535 entries, forced
    here (B200LU_DEST32=1) on random patterns and on a KKT sequence."""
    monkeypatch.setenv("B200LU_DEST32", "1")
    rng = rb.RefRng(97)
    for _ in range(12):
        A = rng.random_sparse(rng.uniform_int(2, 80), 5, 0.1, 1.0, True)
        fx = csr_fixture(A, False, True)
        f = rlu.factorize(fx.sym, fx.matrix())
        expect, failed = fx.oracle.factorize(fx.values[0])
        assert failed == -1 and np.array_equal(f.values, expect)
        f.close()
    fx = kkt_fixture(1400, 600, num_systems=2)
    f = rlu.NumericFactors(fx.sym)
    for k in range(2):
        rlu.refactorize(f, fx.matrix(k))
        expect, failed = fx.oracle.factorize(fx.values[k])
        assert failed == -1 and np.array_equal(f.values, expect)
    f.close()


def test_empty_system_follows_the_reference_conventions():
    """A 0 x 0 system: eliminate (src/numeric.cpp:27-58) has no row that could fail, so the factors become valid and the
    generation advances; solve_system returns an empty x; fgmres_refine sees ||r|| / max(||b||, 1 if b = 0) = 0 <= tol and
    returns after 0 iterations, converged, history [0] (src/refine.cpp:51-58, src/sparse.cpp:283-288). Single handle and batch."""
    from paper_2306_14337_b200 import analysis
    from paper_2306_14337_b200.batch import BatchedFactors
    A = rlu.CsrMatrix(0, 0, np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
    sym = analysis.symbolic_analyze(A)
    assert sym.n == 0 and sym.col_indices.size == 0
    f = rlu.factorize(sym, A)
    assert f.valid and f.generation == 1 and f.values.size == 0
    rlu.refactorize(f, A)
    assert f.valid and f.generation == 2
    x = rlu.solve_system(f, np.zeros(0))
    assert x.shape == (0,)
    out = rlu.fgmres_refine(f, np.zeros(0), x)
    assert out.iterations == 0 and out.converged and list(out.residual_history) == [0.0]
    f.close()
    bf = BatchedFactors(sym, 3)
    bf.refactorize(np.zeros((3, 0)))
    xs = bf.solve_system(np.zeros((3, 0)))
    assert tuple(xs.shape) == (3, 0)
    _, outs = bf.fgmres_refine(np.zeros((3, 0)), xs, rlu.RefineConfig())
    assert [(o.iterations, bool(o.converged)) for o in outs] == [(0, True)] * 3
    bf.close()


@needs_ref
def test_handles_on_different_patterns_coexist():
    """Distinct instances may live side by side (include/rlu/numeric.hpp:19-21). The dynamic shared-memory limit of a
    kernel is per FUNCTION, process-wide: a handle created later on a smaller pattern (shorter tail rows, no wide rows)
    must not lower it under a live handle with a larger one. Large, small, batch handle of a third pattern, then the
    large one again — every result against the oracle."""
    from paper_2306_14337_b200.batch import BatchedFactors
    big = kkt_fixture(6300, 2700, num_systems=2)
    small = csr_fixture(rb.RefRng(7).random_sparse(30, 4, 0.1, 1.0, True), False, True)
    mid = kkt_fixture(700, 300, num_systems=2)
    fb = rlu.NumericFactors(big.sym, rlu.FactorOptions(strict_order=True))
    rlu.refactorize(fb, big.matrix(0))
    fs = rlu.NumericFactors(small.sym, rlu.FactorOptions(strict_order=True))
    rlu.refactorize(fs, small.matrix())
    bm = BatchedFactors(mid.sym, 5)
    bm.refactorize(np.stack([mid.values[s % 2] for s in range(5)]))
    for k in (1, 0):
        rlu.refactorize(fb, big.matrix(k))
        ref, failed = big.oracle.factorize(big.values[k])
        assert failed == -1 and np.array_equal(fb.values, ref)
        assert np.array_equal(rlu.solve_system(fb, big.rhs[k]), big.oracle.solve_system(ref, big.rhs[k])[0])
        out = rlu.fgmres_refine(fb, big.rhs[k], rlu.solve_system(fb, big.rhs[k]))
        assert out.converged
    ref_s, _ = small.oracle.factorize(small.values[0])
    assert np.array_equal(fs.values, ref_s)
    assert np.array_equal(rlu.solve_system(fs, small.rhs[0]), small.oracle.solve_system(ref_s, small.rhs[0])[0])
    ref_m, _ = mid.oracle.factorize(mid.values[1])
    assert np.array_equal(bm.values(3), ref_m)
    xm = bm.solve_system(np.stack([mid.rhs[s % 2] for s in range(5)]))
    assert np.array_equal(xm[3], mid.oracle.solve_system(ref_m, mid.rhs[1])[0])
    for h in (fb, fs, bm):
        h.close()


@needs_ref
def test_refactorize_is_bitwise_identical_to_factorize():
    # test_numeric.cpp:223-253, acceptance.cpp:190-205
    rng = rb.RefRng(93)
    for _ in range(12):
        n = rng.uniform_int(2, 40)
        A = rng.random_sparse(n, 4, 0.1, 1.0, True)
        fx = csr_fixture(A)
        vals = fx.values[0].copy()
        reused = rlu.factorize(fx.sym, fx.matrix(values=vals))
        assert reused.generation == 1
        for step in range(1, 6):
            vals = vals * np.array([rng.uniform_real(0.9, 1.1) for _ in range(vals.size)])
            rlu.refactorize(reused, fx.matrix(values=vals))
            fresh = rlu.factorize(fx.sym, fx.matrix(values=vals))
            assert np.array_equal(reused.values, fresh.values)
            assert np.array_equal(reused.values, fx.oracle.factorize(vals)[0])
            assert reused.generation == step + 1
            fresh.close()
        snapshot = reused.values
        rlu.refactorize(reused, fx.matrix(values=vals))  # unchanged values, test_numeric.cpp:245-253
        assert np.array_equal(reused.values, snapshot)
        reused.close()


@needs_ref
def test_pattern_change_requires_reanalysis():
    # test_numeric.cpp:255-275
    rng = rb.RefRng(95)
    A = rng.random_sparse(30, 3, 0.1, 1.0, True)
    fx = csr_fixture(A)
    f = rlu.factorize(fx.sym, fx.matrix())
    M = A.to_dense()
    if M[0, 29] == 0.0:
        M[0, 29] = 0.5
        wider = rb.RefCsr.from_dense(M)
        ro, ci, v = wider.arrays()
        with pytest.raises(rlu.PatternMismatchError):
            rlu.refactorize(f, rlu.CsrMatrix(30, 30, ro, ci, v))
    assert f.valid  # the guard fires before anything is touched


@needs_ref
def test_run_to_run_determinism_and_shared_symbolic():
    # test_numeric.cpp:277-326: schedule independence is bitwise; two instances share one analysis
    rng = rb.RefRng(98)
    A = rng.random_sparse(220, 5, 0.1, 1.0, True)
    fx = csr_fixture(A)
    f1, f2 = rlu.NumericFactors(fx.sym), rlu.NumericFactors(fx.sym)
    expect1 = fx.oracle.factorize(fx.values[0])[0]
    expect3 = fx.oracle.factorize(3.0 * fx.values[0])[0]
    for _ in range(20):
        rlu.refactorize(f1, fx.matrix())
        rlu.refactorize(f2, fx.matrix(values=3.0 * fx.values[0]))
        assert np.array_equal(f1.values, expect1) and np.array_equal(f2.values, expect3)


# ---------------------------------------------------------- triangular solves

@needs_ref
def test_trisolve_known_answers():
    # test_trisolve.cpp:56-100
    f = rlu.factorize(*(lambda fx: (fx.sym, fx.matrix()))(dense_fixture([[1, 0], [0, 1]])))
    assert np.array_equal(rlu.lower_solve(f, np.array([3.0, 4.0])), [3, 4])
    assert np.array_equal(rlu.upper_solve(f, np.array([5.0, 6.0])), [5, 6])
    assert np.array_equal(rlu.solve_system(f, np.array([7.0, 8.0])), [7, 8])
    fx = dense_fixture([[1, 0], [2, 1]])
    assert np.array_equal(rlu.lower_solve(rlu.factorize(fx.sym, fx.matrix()), np.array([1.0, 4.0])), [1, 2])
    fx = dense_fixture(np.eye(4) - np.eye(4, k=-1))
    assert np.array_equal(rlu.lower_solve(rlu.factorize(fx.sym, fx.matrix()), np.ones(4)), [1, 2, 3, 4])
    fx = dense_fixture([[2, 1], [0, 4]])
    assert np.array_equal(rlu.upper_solve(rlu.factorize(fx.sym, fx.matrix()), np.array([4.0, 8.0])), [1, 2])
    fx = dense_fixture([[2, 0], [0, 4]])
    assert np.array_equal(rlu.upper_solve(rlu.factorize(fx.sym, fx.matrix()), np.array([2.0, 8.0])), [1, 2])
    fx = dense_fixture([[4, 3], [6, 3]])
    x = rlu.solve_system(rlu.factorize(fx.sym, fx.matrix()), np.array([10.0, 12.0]))
    assert np.allclose(x, [1, 2], rtol=1e-14)


@needs_ref
@pytest.mark.parametrize("scaling", [True, False])
def test_trisolve_bitwise_and_composition(scaling):
    # test_trisolve.cpp:102-153
    rng = rb.RefRng(303)
    for _ in range(10):
        n = rng.uniform_int(10, 200)
        A = rng.random_sparse(n, 5, 0.1, 1.0, True)
        fx = csr_fixture(A, scaling, True)
        f = rlu.factorize(fx.sym, fx.matrix(), STRICT)
        lu = f.values
        b = rng.random_vector(n)
        lo = rlu.lower_solve(f, b)
        assert np.array_equal(lo, fx.oracle.lower_solve(lu, b))
        assert np.array_equal(rlu.upper_solve(f, b), fx.oracle.upper_solve(lu, b)[0])
        x = rlu.solve_system(f, b)
        assert np.array_equal(x, fx.oracle.solve_system(lu, b)[0])
        if not scaling:
            # all stages identity except the AMD permutation: U^-1 L^-1 on the permuted rhs
            p = fx.sym.amd_forward
            w = np.empty(n)
            w[p] = b
            t = rlu.upper_solve(f, rlu.lower_solve(f, w))
            assert np.array_equal(x, t[p])
        assert fx.oracle_csr().relative_residual(x, b) <= 1e-10  # test_trisolve.cpp:113-127
        f.close()


@needs_ref
def test_upper_solve_rejects_exact_zero_diagonal_and_dimension_errors():
    # test_trisolve.cpp:171-192
    fx = dense_fixture([[1.0]])
    f = rlu.factorize(fx.sym, fx.matrix())
    f.set_values(np.array([0.0]))
    with pytest.raises(rlu.ZeroPivotError) as e:
        rlu.upper_solve(f, np.array([1.0]))
    assert e.value.row == 0
    fx = dense_fixture([[1, 0], [0, 1]])
    f = rlu.factorize(fx.sym, fx.matrix())
    for fn, vec in ((rlu.lower_solve, [1, 2, 3]), (rlu.upper_solve, [1]), (rlu.solve_system, [1, 2, 3])):
        with pytest.raises(rlu.DimensionError):
            fn(f, np.array(vec, dtype=float))


@needs_ref
def test_no_device_allocation_after_create():
    # test_trisolve.cpp:155-169 (no allocation after the first solve), SPEC contract
    rng = rb.RefRng(304)
    A = rng.random_sparse(64, 4, 0.1, 1.0, True)
    fx = csr_fixture(A)
    f = rlu.factorize(fx.sym, fx.matrix())
    b = rng.random_vector(64)
    before = f.stats["alloc_events"]
    x0 = rlu.solve_system(f, b)
    for _ in range(200):
        assert np.array_equal(rlu.solve_system(f, b), x0)
    rlu.refactorize(f, fx.matrix())
    rlu.fgmres_refine(f, b, x0)
    assert f.stats["alloc_events"] == before


@needs_ref
@pytest.mark.parametrize("scaling", [False, True])
def test_default_sweep_order_is_deterministic_and_as_accurate(scaling):
    """Default options sum the sweeps' terms in device order (U rows last column first, the narrow
    tail of the DAG inside one CTA with a fixed tree): same terms, different rounding.
    Tolerance: the direct residual may not exceed the reference-order residual by more than 4x
    (+1e-15 absolute), and two runs must agree bit for bit."""
    fx = kkt_fixture(6300, 2700, use_scaling=scaling)
    f, fs = rlu.NumericFactors(fx.sym), rlu.NumericFactors(fx.sym, STRICT)
    for k in (0, len(fx.values) - 1):
        rlu.refactorize(f, fx.matrix(k))
        rlu.refactorize(fs, fx.matrix(k))
        assert np.array_equal(f.values, fs.values)
        b = fx.rhs[k]
        lo_fast, lo_strict = rlu.lower_solve(f, b), rlu.lower_solve(fs, b)
        assert np.array_equal(lo_strict, fx.oracle.lower_solve(fs.values, b))
        assert np.allclose(lo_fast, lo_strict, rtol=0, atol=1e-9 * np.abs(lo_strict).max())
        x, xs = rlu.solve_system(f, b), rlu.solve_system(fs, b)
        assert np.array_equal(x, rlu.solve_system(f, b))
        assert np.array_equal(xs, fx.oracle.solve_system(fs.values, b)[0])
        r, rs = _relres(fx, x, b, k), _relres(fx, xs, b, k)
        assert r <= 4 * rs + 1e-15, (r, rs)
        out = rlu.fgmres_refine(f, b, x)
        assert _relres(fx, out.x, b, k) <= 1e-14


# --------------------------------------------------------------- SpMV / BLAS

@needs_ref
def test_spmv_bitwise_and_relative_residual():
    rng = rb.RefRng(11)
    for _ in range(5):
        n = rng.uniform_int(5, 300)
        A = rng.random_sparse(n, 6, 0.1, 1.0, True)
        fx = csr_fixture(A)
        f = rlu.factorize(fx.sym, fx.matrix())
        x, b = rng.random_vector(n), rng.random_vector(n)
        assert np.array_equal(rlu.spmv(f, x), fx.oracle_csr().spmv(x))
        ref = fx.oracle_csr().relative_residual(x, b)
        assert abs(rlu.relative_residual(f, x, b) - ref) <= 1e-14 * ref  # parallel sum vs serial sum
        f.close()


# --------------------------------------------------------------- refinement

def _relres(fx, x, b, k=0):
    return fx.oracle_csr(k).relative_residual(x, b)


@needs_ref
def test_fgmres_exact_preconditioner_one_iteration():
    # test_refine.cpp:81-96
    rng = rb.RefRng(72)
    A = rng.random_sparse(60, 4, 0.1, 1.0, True)
    fx = csr_fixture(A)
    f = rlu.factorize(fx.sym, fx.matrix())
    b = rng.random_vector(60)
    out = rlu.fgmres_refine(f, b, np.zeros(60))
    assert out.converged and out.iterations == 1
    assert _relres(fx, out.x, b) <= 1e-14


@needs_ref
def test_fgmres_identity_preconditioner_contracts():
    # test_refine.cpp:98-159
    fx = dense_fixture(np.diag([1.0, 2.0, 3.0]))
    f = rlu.factorize(fx.sym, fx.matrix())
    out = rlu.fgmres_refine(f, np.array([1.0, 2.0, 3.0]), np.zeros(3), preconditioned=False)
    assert out.converged and out.iterations <= 3 and np.allclose(out.x, 1.0, rtol=1e-12)
    fx = dense_fixture(np.diag([2.0, 2.0]))
    f = rlu.factorize(fx.sym, fx.matrix())
    out = rlu.fgmres_refine(f, np.array([2.0, 2.0]), np.array([1.0, 1.0]), preconditioned=False)
    assert out.converged and out.iterations == 0 and np.array_equal(out.x, [1, 1])
    fx = dense_fixture(np.diag([1.0, 1e-8, 1.0]))
    f = rlu.factorize(fx.sym, fx.matrix())
    out = rlu.fgmres_refine(f, np.ones(3), np.zeros(3), rlu.RefineConfig(2, 1e-16), preconditioned=False)
    assert not out.converged and out.iterations == 2


@needs_ref
def test_fgmres_history_monotone_and_never_degrades():
    # test_refine.cpp:120-146; also tracks the oracle's history to 1e-10 relative (the device
    # dot products are parallel sums, so the histories agree to rounding, not to the bit)
    rng = rb.RefRng(73)
    for _ in range(6):
        A = rng.random_sparse(50, 4, 0.1, 1.0, True)
        fx = csr_fixture(A)
        f = rlu.factorize(fx.sym, fx.matrix())
        b = rng.random_vector(50)
        out = rlu.fgmres_refine(f, b, np.zeros(50), rlu.RefineConfig(15, 1e-30), preconditioned=False)
        h = out.residual_history
        assert out.iterations == 15 and len(h) == 16
        assert all(h[i] <= h[i - 1] * (1 + 1e-12) for i in range(1, len(h)))
        _, _, _, href = ob.refine(fx.oracle_csr(), b, np.zeros(50), None, None, max_iterations=15, tolerance=1e-30)
        assert np.allclose(h[:8], href[:8], rtol=1e-8)
        f.close()
    rng = rb.RefRng(74)
    for _ in range(6):
        A = rng.random_sparse(40, 4, 0.1, 1.0, False)
        fx = csr_fixture(A, use_scaling=False, use_amd=False)
        f = rlu.NumericFactors(fx.sym)
        rlu.reset_values(f, fx.matrix())
        b, x0 = rng.random_vector(40), rng.random_vector(40)
        out = rlu.fgmres_refine(f, b, x0, rlu.RefineConfig(3, 1e-14), preconditioned=False)
        assert _relres(fx, out.x, b) <= _relres(fx, x0, b) * (1 + 1e-12)
        f.close()


@needs_ref
def test_classic_refinement_wilkinson():
    # test_refine.cpp:161-176
    rng = rb.RefRng(75)
    A = rng.random_sparse(50, 4, 0.1, 1.0, True)
    fx = csr_fixture(A)
    f = rlu.factorize(fx.sym, fx.matrix())
    b = fx.oracle_csr().spmv(rng.random_vector(50))
    out = rlu.classic_refine(f, b, np.zeros(50))
    assert out.converged and out.iterations <= 2 and _relres(fx, out.x, b) <= 1e-14


@needs_ref
def test_refinement_repairs_growth_degraded_solve():
    # test_refine.cpp:178-217: 2x2 blocks [[eps,1],[1,1]] in natural order, growth 1/eps
    nb, eps = 100, 1e-8
    M = np.zeros((2 * nb, 2 * nb))
    for k in range(nb):
        M[2 * k, 2 * k], M[2 * k, 2 * k + 1], M[2 * k + 1, 2 * k], M[2 * k + 1, 2 * k + 1] = eps, 1, 1, 1
    fx = dense_fixture(M)
    b = fx.oracle_csr().spmv(np.ones(2 * nb))
    f = rlu.factorize(fx.sym, fx.matrix())
    x0 = rlu.solve_system(f, b)
    assert _relres(fx, x0, b) > 1e-12
    out = rlu.fgmres_refine(f, b, x0)
    assert out.converged and out.iterations >= 1 and _relres(fx, out.x, b) <= 1e-14
    fx2 = dense_fixture(M, use_scaling=True, use_amd=True)
    f2 = rlu.factorize(fx2.sym, fx2.matrix())
    assert _relres(fx2, rlu.solve_system(f2, b), b) <= 1e-14


@needs_ref
def test_refinement_converges_within_two_iterations():
    # test_refine.cpp:219-242
    rng = rb.RefRng(76)
    for _ in range(20):
        n = rng.uniform_int(5, 150)
        A = rng.random_sparse(n, 5, 0.1, 1.0, True)
        fx = csr_fixture(A)
        f = rlu.factorize(fx.sym, fx.matrix())
        b = rng.random_vector(n)
        x0 = rlu.solve_system(f, b)
        direct = _relres(fx, x0, b)
        out = rlu.fgmres_refine(f, b, x0)
        refined = _relres(fx, out.x, b)
        assert out.iterations <= 2 and refined <= 100 * direct + 1e-16 and refined <= 1e-14
        f.close()


# ------------------------------------------------------- KKT sequences (C1)

@needs_ref
@pytest.mark.parametrize("scaling", [False, True])
def test_kkt_sequence_c1_analyze_once_refactorize_rest(scaling):
    """BASELINE config C1 (ACTIVSg200-shaped, n+m = 9000): one analysis, 10 refactor/solve;
    acceptance.cpp:236-272 (relres <= 1e-8 on every system, median refinement iterations <= 2)."""
    fx = kkt_fixture(6300, 2700, use_scaling=scaling)
    f = rlu.NumericFactors(fx.sym, STRICT)
    ref_num = rb.RefNumeric(fx.ref_sym)
    iters = []
    for k in range(len(fx.values)):
        rlu.refactorize(f, fx.matrix(k))
        lu = f.values
        assert np.array_equal(lu, fx.oracle.factorize(fx.values[k])[0])
        b = fx.rhs[k]
        x0 = rlu.solve_system(f, b)
        assert np.array_equal(x0, fx.oracle.solve_system(lu, b)[0])
        out = rlu.fgmres_refine(f, b, x0)
        ref_num.refactorize(fx.ref_matrix(k))
        ref = rb.refine(fx.ref_matrix(k), b, ref_num.solve_system(b), ref_num)
        got, want = _relres(fx, out.x, b, k), _relres(fx, ref.x, b, k)
        assert got <= 1e-8 and got <= max(4 * want, 1e-15), (k, got, want)
        assert out.iterations == ref.iterations
        iters.append(out.iterations)
    assert f.generation == len(fx.values)
    assert sorted(iters)[len(iters) // 2] <= 2


@needs_ref
def test_device_resident_vectors_match_host_path():
    import torch
    fx = kkt_fixture(700, 300)
    f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream))
    dvals = torch.from_numpy(fx.values[0]).cuda()
    rlu.refactorize(f, rlu.CsrMatrix(fx.n, fx.n, fx.ro, fx.ci, dvals))
    assert np.array_equal(f.values, fx.oracle.factorize(fx.values[0])[0])
    db = torch.from_numpy(fx.rhs[0]).cuda()
    dx = rlu.solve_system(f, db)
    assert dx.is_cuda and np.array_equal(dx.cpu().numpy(), rlu.solve_system(f, fx.rhs[0]))
    out = rlu.fgmres_refine(f, db, dx)
    assert out.x.is_cuda and _relres(fx, out.x.cpu().numpy(), fx.rhs[0]) <= 1e-14


# ------------------------------------------------------------- scenario batches

@needs_ref
def test_scenario_batch_matches_single_handle_runs():
    """independent scenarios sharing one pattern, several in flight on one GPU
    (one handle + stream per in-flight system, FactorOptions.concurrency). Every scenario must
    come out bit-identical to a lone run with the same options."""
    from paper_2306_14337_b200.batch import ScenarioBatch
    base = kkt_fixture(700, 300, num_systems=1)
    scen = [kkt_fixture(700, 300, num_systems=1, y_seed=2 + s) for s in range(12)]
    for s in scen:  # same topology_seed -> same pattern -> one analysis
        assert np.array_equal(s.ci, base.ci) and np.array_equal(s.sym.col_indices, base.sym.col_indices)
    mats = [rlu.CsrMatrix(base.n, base.n, base.ro, base.ci, s.values[0]) for s in scen]
    rhs = [s.rhs[0] for s in scen]
    batch = ScenarioBatch(base.sym, streams=4)
    records, xs = batch.run(mats, rhs)
    lone = rlu.NumericFactors(base.sym, rlu.FactorOptions(concurrency=4))
    for s in range(len(scen)):
        rlu.refactorize(lone, mats[s])
        assert np.array_equal(lone.values, scen[s].oracle.factorize(scen[s].values[0])[0])
        x0 = rlu.solve_system(lone, rhs[s])
        out = rlu.fgmres_refine(lone, rhs[s], x0)
        assert np.array_equal(xs[s], out.x)
        assert records[s].scenario == s and records[s].failed_row == -1
        assert records[s].refine_iters == out.iterations and records[s].relres_final <= 1e-14
    batch.close()


# ---------------------------------------------------------------- cgs2_orthonormalize at the boundary
# proj/tests/test_refine.cpp:34-79 restated against b200lu_cgs2_orthonormalize.

def _identity_handle(n):
    fx = dense_fixture(np.eye(n))
    return rlu.NumericFactors(fx.sym)


def _unit(n, i):
    e = np.zeros(n)
    e[i] = 1.0
    return e


@needs_ref
def test_cgs2_exact_cases():
    f = _identity_handle(3)
    try:
        r = rlu.cgs2_orthonormalize(f, [_unit(3, 0)], _unit(3, 1))    # already orthogonal: left alone
        assert not r.breakdown and r.coefficients[0] == 0.0 and np.array_equal(r.vector, _unit(3, 1)) and r.norm == 1.0
        r = rlu.cgs2_orthonormalize(f, [_unit(3, 0)], _unit(3, 0) + _unit(3, 1))  # projects exactly
        assert not r.breakdown and r.coefficients[0] == 1.0 and np.array_equal(r.vector, _unit(3, 1))
        r = rlu.cgs2_orthonormalize(f, [_unit(3, 0)], _unit(3, 0))    # happy breakdown on subspace membership
        assert r.breakdown
        r = rlu.cgs2_orthonormalize(f, np.zeros((0, 3)), np.array([3.0, 0.0, 4.0]))  # empty basis: plain normalisation
        assert not r.breakdown and r.norm == 5.0 and np.array_equal(r.vector, np.array([0.6, 0.0, 0.8]))
        with pytest.raises(rlu.DimensionError):
            rlu.cgs2_orthonormalize(f, [_unit(3, 0)], np.ones(4))
    finally:
        f.close()


@needs_ref
def test_cgs2_restores_orthogonality_lost_by_a_single_pass():
    n = 50
    f = _identity_handle(n)
    rng = rb.RefRng(71)
    basis = []
    try:
        for k in range(20):
            v = rng.random_vector(n)
            if basis:  # nearly dependent on the basis: stresses the re-orthogonalisation pass
                v = basis[0] + 1e-9 * v
            r = rlu.cgs2_orthonormalize(f, np.array(basis), v)
            assert not r.breakdown
            for q in basis:
                assert abs(ob.dot(q, r.vector)) <= 1e-13
            # against the reference itself: same coefficients and vector up to the rounding of the dot products
            cref, vref, nref, bref = rb.cgs2(np.array(basis), v)
            assert not bref and nref == pytest.approx(r.norm, rel=1e-12)
            assert np.allclose(r.coefficients, cref, rtol=1e-12, atol=1e-15)
            basis.append(r.vector)
    finally:
        f.close()
