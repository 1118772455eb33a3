"""Parity at the BASELINE.json sizes: C2 (n = 55 700) and C3 (n = 238 000) — the oracle
still finishes in seconds there, so L/U values and solves are compared bit for bit; plus the
size-independent properties the reference tests use (refactorize == factorize, scaling linearity,
manufactured solutions)."""
import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
from tests.fixtures import kkt_fixture

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not rb.available(), reason="oracle/_ref/librlu_ref.so not built")]

C2 = (39000, 16700)
C3 = (166600, 71400)


@pytest.mark.parametrize("shape", [C2, C3], ids=["C2", "C3"])
def test_single_system_bitwise_at_full_size(shape):
    fx = kkt_fixture(*shape, num_systems=2)
    f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(strict_order=True))
    for k in range(2):
        rlu.refactorize(f, fx.matrix(k))
        ref, failed = fx.oracle.factorize(fx.values[k])
        assert failed == -1 and np.array_equal(f.values, ref)
        x = rlu.solve_system(f, fx.rhs[k])
        assert np.array_equal(x, fx.oracle.solve_system(ref, fx.rhs[k])[0])
        out = rlu.fgmres_refine(f, fx.rhs[k], x)
        assert out.converged and fx.oracle_csr(k).relative_residual(out.x, fx.rhs[k]) <= 1e-14
    # refactorize == factorize on a fresh handle, bit for bit (test_numeric.cpp:223-253)
    g = rlu.factorize(fx.sym, fx.matrix(1), rlu.FactorOptions(strict_order=True))
    assert np.array_equal(g.values, f.values)
    # default sweep order: same factors, residual as good as the reference's (3e-9 direct)
    d = rlu.factorize(fx.sym, fx.matrix(1))
    assert np.array_equal(d.values, f.values)
    xd = rlu.solve_system(d, fx.rhs[1])
    assert fx.oracle_csr(1).relative_residual(xd, fx.rhs[1]) <= 4 * fx.oracle_csr(1).relative_residual(x, fx.rhs[1])
    for h in (f, g, d):
        h.close()


def test_scaling_linearity_at_c2():
    # test_numeric.cpp:159-171: factorize(2A) has the same L and a doubled U
    fx = kkt_fixture(*C2, num_systems=1)
    f = rlu.factorize(fx.sym, fx.matrix(0))
    g = rlu.factorize(fx.sym, fx.matrix(0, 2.0 * fx.values[0]))
    a, b = f.values, g.values
    rows = np.repeat(np.arange(fx.n), np.diff(fx.sym.row_offsets))
    is_lower = fx.sym.col_indices < rows
    # scaling by 2 is exact except where an intermediate is subnormal: a few hundred fill values of this
    # matrix sit at 1e-310..1e-322 (in the reference as well), so the property is stated on the normal range
    normal = (np.abs(a) >= 1e-290) | (a == 0.0)
    assert np.count_nonzero(~normal) < 1e-3 * a.size
    assert np.array_equal(a[is_lower & normal], b[is_lower & normal])          # L unchanged
    assert np.array_equal(2.0 * a[~is_lower & normal], b[~is_lower & normal])  # U doubled
    # and the device reproduces the reference on the subnormal entries too
    assert np.array_equal(b, fx.oracle.factorize(2.0 * fx.values[0])[0])
    f.close()
    g.close()


def test_batch_bitwise_at_c2():
    """48 scenarios of C2 (y_seed = 2 + s): a sample bit for bit against the oracle, all of them on the
    residual and against a manufactured solution."""
    B = 48
    seqs = [rb.RefSequence(*C2, y_seed=2 + s, num_systems=1) for s in range(B)]
    fx = kkt_fixture(*C2, num_systems=1)
    vals = np.stack([q.values(0) for q in seqs])
    rhs = np.stack([q.rhs(0) for q in seqs])
    f = BatchedFactors(fx.sym, B, rlu.FactorOptions(refine_capacity=4))
    f.refactorize(vals)
    x = f.solve_system(rhs)
    for s in (0, 15, 16, 31, 32, 47):
        ref, failed = fx.oracle.factorize(vals[s])
        assert failed == -1 and np.array_equal(f.values(s), ref)
        assert np.array_equal(x[s], fx.oracle.solve_system(ref, rhs[s])[0])
    # run-to-run determinism of the refactorization (its updates are L2 reductions, ordered per thread):
    # the rows at the top of the elimination tree — the longest dependency chains — are where a race shows
    before = {s: f.values(s) for s in (0, 7, 21, 47)}
    f.refactorize(vals)
    for s, v in before.items():
        assert np.array_equal(f.values(s), v)
    xr, outs = f.fgmres_refine(rhs, x, rlu.RefineConfig(max_iterations=4))
    final = f.relative_residual(xr, rhs)
    assert np.all(final <= 1e-14) and all(o.converged and o.iterations <= 2 for o in outs)
    # the reference's own residual of the same solution agrees (checker: the reference's relative_residual)
    assert seqs[5].matrix(0).relative_residual(xr[5], rhs[5]) <= 1e-14
    f.close()


def test_pattern_guard_at_full_size_sees_a_change_in_any_chunk():
    """pattern_equal (src/numeric.cpp:15-17) runs on every scatter; above 2 MB the comparison is split over host
    threads: a single changed index anywhere — first row offset, last column index — must still be refused."""
    fx = kkt_fixture(*C2, num_systems=1)
    f = rlu.NumericFactors(fx.sym)
    try:
        rlu.refactorize(f, fx.matrix(0))
        for where in (1, len(fx.ci) // 2, len(fx.ci) - 1):
            ci = fx.ci.copy()
            ci[where] = ci[where] + 1 if where == len(ci) - 1 or ci[where] + 1 != ci[where + 1] else ci[where] - 1
            with pytest.raises(rlu.PatternMismatchError):
                rlu.refactorize(f, rlu.CsrMatrix(fx.n, fx.n, fx.ro, ci, fx.values[0]))
        ro = fx.ro.copy()
        ro[len(ro) // 2] += 1
        with pytest.raises(rlu.PatternMismatchError):
            rlu.refactorize(f, rlu.CsrMatrix(fx.n, fx.n, ro, fx.ci, fx.values[0]))
        with pytest.raises(rlu.PatternMismatchError):  # a value array of the wrong length
            rlu.refactorize(f, rlu.CsrMatrix(fx.n, fx.n, fx.ro, fx.ci, fx.values[0][:-1]))
        rlu.refactorize(f, fx.matrix(0))  # and the handle still works
        assert np.array_equal(f.values, fx.oracle.factorize(fx.values[0])[0])
    finally:
        f.close()
