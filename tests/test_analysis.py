"""Host-side symbolic analysis (csrc/analyze.cpp) against the unmodified reference
(rlu::symbolic_analyze, src/symbolic.cpp:156-203): every array of the product bit for bit — MC64 matching and
scale factors (src/matching.cpp), AMD order (src/ordering.cpp), fill pattern / diag_pos (src/symbolic.cpp:95-154),
scatter map and scale — plus the reference's error behaviour. No GPU involved."""
import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from oracle import refbridge as rb
from paper_2306_14337_b200.analysis import (AnalyzeOptions, StructurallySingularError, ZeroDiagonalError,
                                            symbolic_analyze)

pytestmark = pytest.mark.skipif(not rb.available(), reason="reference bridge not built")

FIELDS = ("row_offsets", "col_indices", "diag_pos", "scatter_map", "scatter_scale", "amd_forward",
          "col_perm_forward", "row_scale", "col_scale", "src_row_offsets", "src_col_indices")


def assert_same_product(ro, ci, vals, use_scaling, use_amd):
    n = len(ro) - 1
    ref = rb.RefSymbolic(rb.RefCsr.from_arrays(n, ro, ci, vals), use_scaling=use_scaling, use_amd=use_amd)
    want = ref.arrays()
    got = symbolic_analyze(rlu.CsrMatrix(n, n, ro, ci, vals), AnalyzeOptions(use_scaling, use_amd))
    for k in FIELDS:
        a, b = getattr(got, k), getattr(want, k)
        assert (a is None) == (b is None), k
        if a is not None:
            a, b = np.asarray(a), np.asarray(b)
            assert a.dtype == b.dtype and np.array_equal(a, b), k  # float arrays too: bitwise equal values
    assert got.fill_count == want.fill_count
    return got


def random_matrix(rng, n, extra, symmetric_pattern):
    """Random pattern with a full diagonal; unsymmetric unless asked otherwise."""
    M = np.zeros((n, n))
    for i in range(n):
        cols = rng.choice(n, size=min(n, extra), replace=False)
        M[i, cols] = rng.uniform(-1.0, 1.0, size=cols.size)
    if symmetric_pattern:
        M = M + 0.5 * M.T
    M[np.arange(n), np.arange(n)] = rng.uniform(0.5, 2.0, size=n) * rng.choice([-1.0, 1.0], size=n)
    ro, ci, v = [0], [], []
    for i in range(n):
        nz = np.nonzero(M[i])[0]
        ci.extend(nz.tolist())
        v.extend(M[i, nz].tolist())
        ro.append(len(ci))
    return np.array(ro, dtype=np.int64), np.array(ci, dtype=np.int64), np.array(v)


@pytest.mark.parametrize("use_scaling", [False, True])
@pytest.mark.parametrize("use_amd", [False, True])
@pytest.mark.parametrize("n,m", [(70, 30), (700, 300)])
def test_kkt_patterns_match_the_reference(n, m, use_scaling, use_amd):
    seq = rb.RefSequence(n, m, num_systems=2)
    ro, ci = seq.pattern()
    for k in range(2):  # the matching depends on the values
        assert_same_product(ro, ci, seq.values(k), use_scaling, use_amd)


@pytest.mark.parametrize("use_scaling", [False, True])
def test_c1_matches_the_reference(use_scaling):
    seq = rb.RefSequence(6300, 2700, num_systems=1)
    ro, ci = seq.pattern()
    got = assert_same_product(ro, ci, seq.values(0), use_scaling, True)
    assert got.col_indices.size == (531430 if use_scaling else 347276)


@pytest.mark.parametrize("seed", range(12))
def test_unsymmetric_random_patterns_match_the_reference(seed):
    """The pruned reachability must equal fill1's full merge on patterns with no symmetry at all (the
    MC64 path permutes columns only), with and without an ordering."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(5, 140))
    ro, ci, v = random_matrix(rng, n, int(rng.integers(1, 6)), symmetric_pattern=bool(seed % 3 == 0))
    for use_scaling in (False, True):
        for use_amd in (False, True):
            assert_same_product(ro, ci, v, use_scaling, use_amd)


def test_dense_and_diagonal_corner_cases():
    n = 9
    ro = np.arange(n + 1, dtype=np.int64)
    assert_same_product(ro, np.arange(n, dtype=np.int64), np.full(n, 2.0), True, True)  # diagonal
    M = np.random.default_rng(5).uniform(0.1, 1.0, size=(n, n))
    ro = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int64), n)
    assert_same_product(ro, ci, M.ravel(), True, True)  # dense
    assert_same_product(np.array([0, 1], dtype=np.int64), np.array([0], dtype=np.int64), np.array([3.0]), True, True)


def _ref_error(ro, ci, v, use_scaling, use_amd=True):
    with pytest.raises(rb.RefError) as e:
        rb.RefSymbolic(rb.RefCsr.from_arrays(len(ro) - 1, ro, ci, v), use_scaling=use_scaling, use_amd=use_amd)
    return e.value


def test_zero_diagonal_names_the_reference_row():
    # arrow matrix whose (2, 2) entry is missing
    M = np.array([[4.0, 1, 0, 1], [1, 4, 1, 0], [0, 1, 0, 1], [1, 0, 1, 4]])
    A = rb.RefCsr.from_dense(M)
    ro, ci, v = A.arrays()
    for use_amd in (False, True):
        want = _ref_error(ro, ci, v, False, use_amd)
        with pytest.raises(ZeroDiagonalError) as e:
            symbolic_analyze(rlu.CsrMatrix(4, 4, ro, ci, v), AnalyzeOptions(False, use_amd))
        assert e.value.row == want.row
        assert str(e.value) in str(want)


def test_structurally_singular_inputs():
    # (a) a column of explicit zeros, (b) a row of explicit zeros, (c) no perfect matching (two rows share one column)
    cases = [np.array([[1.0, 0, 2], [3, 0, 4], [5, 0, 6]]), np.array([[1.0, 2, 3], [0, 0, 0], [4, 5, 6]])]
    for M in cases:
        n = M.shape[0]
        ro = np.arange(0, n * n + 1, n, dtype=np.int64)
        ci = np.tile(np.arange(n, dtype=np.int64), n)
        want = _ref_error(ro, ci, M.ravel(), True)
        with pytest.raises(StructurallySingularError) as e:
            symbolic_analyze(rlu.CsrMatrix(n, n, ro, ci, M.ravel()), AnalyzeOptions(True, True))
        assert str(e.value) in str(want)
    M = np.array([[1.0, 0, 0, 0], [2, 0, 0, 0], [0, 1, 1, 1], [0, 1, 1, 1]])
    A = rb.RefCsr.from_dense(M)
    ro, ci, v = A.arrays()
    want = _ref_error(ro, ci, v, True)
    with pytest.raises(StructurallySingularError) as e:
        symbolic_analyze(rlu.CsrMatrix(4, 4, ro, ci, v), AnalyzeOptions(True, True))
    # (the reference's own message says "size 0" under g++: its argument list moves the row set before the
    # message is built, src/matching.cpp:138-142; the row set itself is the contract)
    head = "structurally singular: no perfect matching, deficient row set of size "
    assert head in str(want) and str(e.value) == head + "2 starting at row 1" and str(want).endswith("starting at row 1")
    assert e.value.deficient_rows == [0, 1]


def test_argument_errors():
    ro, ci = np.array([0, 1, 2], dtype=np.int64), np.array([0, 1], dtype=np.int64)
    with pytest.raises(rlu.DimensionError):
        symbolic_analyze(rlu.CsrMatrix(2, 3, ro, ci, np.ones(2)))
    with pytest.raises(rlu.Error):  # mc64_scale: matrix has no values
        symbolic_analyze(rlu.CsrMatrix(2, 2, ro, ci, None), AnalyzeOptions(True, True))
    with pytest.raises(rlu.Error):  # unsorted columns (CsrMatrix::check_structure)
        symbolic_analyze(rlu.CsrMatrix(2, 2, np.array([0, 2, 2], dtype=np.int64), np.array([1, 0], dtype=np.int64), np.ones(2)),
                         AnalyzeOptions(False, True))
    sym = symbolic_analyze(rlu.CsrMatrix(2, 2, ro, ci, None), AnalyzeOptions(False, True))  # pattern only is enough without scaling
    assert sym.col_indices.tolist() == [0, 1] and sym.col_perm_forward is None


def test_analysis_is_faster_than_the_reference_at_c2():
    """Not a benchmark — a guard that the cost model holds: C2 with MC64 costs the reference seconds (O(N) per
    augmenting path), the product here is identical and comes several times sooner."""
    seq = rb.RefSequence(39000, 16700, num_systems=1)
    ro, ci = seq.pattern()
    vals = seq.values(0)
    ref = rb.RefSymbolic(seq.matrix(0), use_scaling=True, use_amd=True)
    got, times = symbolic_analyze(rlu.CsrMatrix(seq.n, seq.n, ro, ci, vals), AnalyzeOptions(True, True), with_times=True)
    want = ref.arrays()
    for k in FIELDS:
        assert np.array_equal(np.asarray(getattr(got, k)), np.asarray(getattr(want, k))), k
    assert times.total_ms < 0.6 * ref.analyze_ms, (times, ref.analyze_ms)
