"""Parity of the scenario-batch path (b200lu_batch_*, through the C ABI) with the oracle, on the B200.

Every scenario of a batch must reproduce the single-system results of the reference: L/U values,
lower/upper/solve_system and SpMV-based residual vectors bit-exact; refinement on the residual
(its dot products are parallel sums on the device), tolerance written in the test.
"""
import os

import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import oraclebridge as ob
from oracle import refbridge as rb
from tests.fixtures import dense_fixture, golden_fixture, kkt_fixture

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not rb.available(), reason="oracle/_ref/librlu_ref.so not built")


def _scenarios(fx, batch):
    """[batch, nnz] values and [batch, n] right-hand sides: the fixture's systems, cycled and
    rescaled so that no two scenarios are identical."""
    nsys = len(fx.values)
    vals = np.stack([fx.values[s % nsys] * (1.0 + 0.03125 * (s // nsys)) for s in range(batch)])
    rhs = np.stack([fx.rhs[s % nsys] * (1.0 - 0.0625 * (s // nsys)) for s in range(batch)])
    return vals, rhs


def _check_batch(fx, batch, refine=True):
    vals, rhs = _scenarios(fx, batch)
    f = BatchedFactors(fx.sym, batch)
    try:
        f.reset_values(vals)
        for s in {0, batch - 1}:
            assert not f.valid(s)
            assert np.array_equal(f.values(s), fx.oracle.scatter_values(vals[s]))
        f.factorize_scattered()
        lus = []
        for s in range(batch):
            ref, failed = fx.oracle.factorize(vals[s])
            assert failed == -1 and f.valid(s)
            assert np.array_equal(f.values(s), ref), f"L/U values of scenario {s} differ from the oracle"
            lus.append(ref)
        lo, up, x = f.lower_solve(rhs), f.upper_solve(rhs), f.solve_system(rhs)
        for s in range(batch):
            assert np.array_equal(lo[s], fx.oracle.lower_solve(lus[s], rhs[s]))
            assert np.array_equal(up[s], fx.oracle.upper_solve(lus[s], rhs[s])[0])
            assert np.array_equal(x[s], fx.oracle.solve_system(lus[s], rhs[s])[0])
        rr = f.relative_residual(x, rhs)
        for s in range(batch):
            want = fx.oracle_csr(0, vals[s]).relative_residual(x[s], rhs[s])
            assert abs(rr[s] - want) <= 1e-12 * max(want, 1e-300) + 1e-30, (s, rr[s], want)
        if refine:
            xr, outcomes = f.fgmres_refine(rhs, x)
            for s in range(batch):
                A = fx.oracle_csr(0, vals[s])
                x_ref, its_ref, conv_ref, hist_ref = ob.refine(A, rhs[s], x[s], fx.oracle, lus[s])
                got, ref = A.relative_residual(xr[s], rhs[s]), A.relative_residual(x_ref, rhs[s])
                # north star: residual at or below the reference's after refinement; both sit at the
                # rounding floor, where "at or below" is meaningful only up to a few ulps of it
                assert got <= max(4 * ref, 1e-15), (s, got, ref)
                assert outcomes[s].iterations == its_ref and outcomes[s].converged == conv_ref
                assert len(outcomes[s].residual_history) == len(hist_ref)
                assert outcomes[s].residual_history[0] == pytest.approx(hist_ref[0], rel=1e-9)
    finally:
        f.close()


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_60", "random_sparse_120_plain"])
def test_batch_committed_fixtures_bitwise(name):
    """tests/golden inputs (no reference needed at run time); partial last group (batch 5)."""
    _check_batch(golden_fixture(name), 5)


@needs_ref
def test_batch_two_groups_partial():
    _check_batch(kkt_fixture(700, 300, num_systems=4), 40)


@needs_ref
@pytest.mark.parametrize("batch", [1, 32])
def test_batch_sizes_one_and_exactly_one_group(batch):
    _check_batch(kkt_fixture(700, 300, num_systems=4), batch)


@needs_ref
def test_batch_one_by_one_matrix():
    fx = dense_fixture(np.array([[2.0]]))
    f = BatchedFactors(fx.sym, 3)
    f.refactorize(np.array([[2.0], [4.0], [-8.0]]))
    x = f.solve_system(np.array([[1.0], [1.0], [1.0]]))
    assert np.array_equal(x, np.array([[0.5], [0.25], [-0.125]]))
    xr, outs = f.fgmres_refine(np.ones((3, 1)), x)
    assert np.array_equal(xr, x) and all(o.converged and o.iterations == 0 for o in outs)
    f.close()


@needs_ref
@pytest.mark.parametrize("width,mode", [(64, 1), (64, 0), (0, 0), (100000, 1)])
def test_batch_trailing_part_variants(width, mode, monkeypatch):
    """The second launch for the narrow trailing levels: mode 1 = row blocks (the default, with
    tail width 1024), mode 0 = the row kernel instantiated for latency, width 0 = no split."""
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", str(width))
    monkeypatch.setenv("B200LU_BATCH_TAIL_MODE", str(mode))
    fx = kkt_fixture(700, 300, num_systems=4)
    f = BatchedFactors(fx.sym, 17)
    info = f.info
    f.close()
    assert info["unit_scenarios"] == 32
    assert (info["blocked_rows"] > 0) == (width > 0) and (info["blocks"] > 0) == (width > 0 and mode == 1)
    _check_batch(fx, 17, refine=False)


@needs_ref
@pytest.mark.parametrize("rows,batch_len,small", [(2, 16, 1), (2, 8, 2), (4, 8, 1), (1, 32, 1), (2, 32, 0)])
def test_batch_gather_form_is_bit_exact(rows, batch_len, small, monkeypatch):
    """The experimental gather form of the trailing refactorization (csrc/gather.cuh: every target entry a batch
    of pivots touches is loaded once, updated in a register in ascending pivot order, stored once — no L2
    reductions). Slower than the default kernels and off by default; its results are the
    reference's bit for bit, with and without MC64, including a zero-pivot scenario."""
    monkeypatch.setenv("B200LU_BATCH_GATHER", "1")
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    monkeypatch.setenv("B200LU_GATHER_R", str(rows))
    monkeypatch.setenv("B200LU_GATHER_K", str(batch_len))
    monkeypatch.setenv("B200LU_GATHER_SMALL", str(small))
    fx = kkt_fixture(700, 300, num_systems=4)
    f = BatchedFactors(fx.sym, 17)
    info = f.info
    f.close()
    assert info["blocks"] > 0 and info["blocked_rows"] > 0 and not info["tiled"]
    _check_batch(fx, 17, refine=False)
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)


@needs_ref
@pytest.mark.parametrize("rows,small", [(2, 1), (2, 2), (1, 1), (2, 0)])
def test_batch_supernodal_form_is_bit_exact(rows, small, monkeypatch):
    """The experimental supernodal form of the trailing refactorization (csrc/snode.cuh: runs of up to 8 consecutive pivot
    rows with nested upper patterns, multipliers in registers, every destination entry loaded and stored once per run).
    Off by default (slower than the default kernels on the narrow trailing DAG); bit-exact."""
    monkeypatch.setenv("B200LU_BATCH_SNODE", "1")
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    monkeypatch.setenv("B200LU_SNODE_R", str(rows))
    monkeypatch.setenv("B200LU_SNODE_SMALL", str(small))
    fx = kkt_fixture(700, 300, num_systems=4)
    f = BatchedFactors(fx.sym, 17)
    info = f.info
    f.close()
    assert info["blocks"] > 0 and info["blocked_rows"] > 0 and not info["tiled"]
    _check_batch(fx, 17, refine=False)
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)
    # a banded matrix: every row of the band is one long supernode chain
    n, band = 300, 12
    M = np.zeros((n, n))
    rng = np.random.default_rng(11)
    for i in range(n):
        lo, hi = max(0, i - band), min(n, i + band + 1)
        M[i, lo:hi] = rng.uniform(-1, 1, hi - lo)
        M[i, i] = 2.0 * band + 1.0
    _check_batch(dense_fixture(M), 9, refine=False)


@needs_ref
@pytest.mark.parametrize("team", [0, 2, 4])
def test_batch_row_block_kernels_agree(team, monkeypatch):
    """B200LU_BATCH_TEAM: 0 = one warp per 2-row block (bfactor_block_kernel, the round-1 kernel), > 0 = one warp per row with
    the pivot row staged once per block (bfactor_block_team_kernel, the default, here with other occupancy targets)."""
    monkeypatch.setenv("B200LU_BATCH_TEAM", str(team))
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    _check_batch(kkt_fixture(700, 300, num_systems=4), 17, refine=False)
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)


@needs_ref
@pytest.mark.parametrize("bulk", [0, 1])
def test_batch_team_kernel_staging_modes_agree(bulk, monkeypatch):
    """B200LU_BATCH_TEAM_BULK: 1 (default) = the pivot row staged by one cp.async.bulk per pivot, awaited on an mbarrier;
    0 = per-lane 16-byte cp.async. Same values bit for bit, incl. pivot rows longer than the stage and partial groups."""
    monkeypatch.setenv("B200LU_BATCH_TEAM_BULK", str(bulk))
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    _check_batch(kkt_fixture(700, 300, num_systems=4), 33, refine=False)
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)
    n, band = 150, 70  # pivot rows of up to 70 upper entries: the part beyond the 48-entry stage goes through registers
    M = np.zeros((n, n))
    rng = np.random.default_rng(5)
    for i in range(n):
        lo, hi = max(0, i - band), min(n, i + band + 1)
        M[i, lo:hi] = rng.uniform(-1.0, 1.0, hi - lo)
        M[i, i] = 2.0 * band + 1.0
    _check_batch(dense_fixture(M), 9, refine=False)


@needs_ref
@pytest.mark.parametrize("team", [0, 3])
def test_batch_32_bit_destination_tables(team, monkeypatch):
    """Rows of more than 65 535 entries need 32-bit destination offsets; no config has such a row, so the uint32_t
    instantiations of the refactorization kernels are forced here (B200LU_BATCH_DEST32=1) and checked bit for bit."""
    monkeypatch.setenv("B200LU_BATCH_DEST32", "1")
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")  # the tiled kernel has its own destination table
    monkeypatch.setenv("B200LU_BATCH_TEAM", str(team))
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    _check_batch(kkt_fixture(700, 300, num_systems=4), 33, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "0")  # everything through the row-per-warp head kernel
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)


@needs_ref
def test_batch_zero_right_hand_side_in_one_scenario():
    """b = 0 for ONE scenario of a batch: its solution is exactly zero, relative_residual uses the denominator 1
    (src/sparse.cpp:283-288), fgmres_refine returns after 0 iterations, converged (src/refine.cpp:51-58) — while its
    neighbours in the same warp refine as usual; every scenario against the oracle."""
    fx = kkt_fixture(700, 300, num_systems=3)
    batch = 6
    vals, rhs = _scenarios(fx, batch)
    rhs[1] = 0.0
    rhs[4] = 0.0
    f = BatchedFactors(fx.sym, batch)
    try:
        f.refactorize(vals)
        x = f.solve_system(rhs)
        assert not np.any(x[1]) and not np.any(x[4])
        rr = f.relative_residual(x, rhs)
        assert rr[1] == 0.0 and rr[4] == 0.0
        xr, outcomes = f.fgmres_refine(rhs, x)
        for s in range(batch):
            lu, _ = fx.oracle.factorize(vals[s])
            A = fx.oracle_csr(0, vals[s])
            x_ref, its_ref, conv_ref, hist_ref = ob.refine(A, rhs[s], x[s], fx.oracle, lu)
            assert outcomes[s].iterations == its_ref and outcomes[s].converged == conv_ref
            assert len(outcomes[s].residual_history) == len(hist_ref)
            assert A.relative_residual(xr[s], rhs[s]) <= max(4 * A.relative_residual(x_ref, rhs[s]), 1e-15)
        assert outcomes[1].iterations == 0 and outcomes[1].converged and list(outcomes[1].residual_history) == [0.0]
        assert not np.any(xr[1])
    finally:
        f.close()


@needs_ref
@pytest.mark.timeout(300)
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_batch_non_finite_input_stays_in_its_scenario(bad):
    """A NaN / Inf among the values of ONE scenario: the reference neither fails (fabs(NaN) <= floor is false,
    src/numeric.cpp:48) nor stops; here nothing may hang on it (x is its own ready flag in the sweeps: a computed NaN
    is canonicalised, never mistaken for the pending marker), the scenario's factors carry NaN exactly where the
    oracle's do, refinement reports non-convergence, and the other scenarios of the same warp stay bit-exact."""
    fx = kkt_fixture(700, 300, num_systems=3)
    vals = np.stack([fx.values[s % 3].copy() for s in range(5)])
    rhs = np.stack([fx.rhs[s % 3] for s in range(5)])
    vals[2, 17] = bad
    vals[2, vals.shape[1] // 2] = bad
    f = BatchedFactors(fx.sym, 5)
    try:
        f.refactorize(vals)
        x = f.solve_system(rhs)
        _, outs = f.fgmres_refine(rhs, x, rlu.RefineConfig(5, 1e-14))
        for s in (0, 1, 3, 4):
            ref, failed = fx.oracle.factorize(vals[s])
            assert np.array_equal(f.values(s), ref)
            assert np.array_equal(x[s], fx.oracle.solve_system(ref, rhs[s])[0])
            assert outs[s].converged
        ref, failed = fx.oracle.factorize(vals[2])
        got = f.values(2)
        assert failed == -1 and f.valid(2)
        assert np.array_equal(np.isnan(got), np.isnan(ref)) and np.isnan(got).any()
        assert np.array_equal(got[~np.isnan(got)], ref[~np.isnan(ref)])
        assert not outs[2].converged and outs[2].iterations == 5
    finally:
        f.close()
    g = rlu.NumericFactors(fx.sym)
    A0 = fx.matrix(0)
    rlu.refactorize(g, rlu.CsrMatrix(fx.n, fx.n, A0.row_offsets, A0.col_indices, vals[2]))
    assert g.valid and np.array_equal(np.isnan(g.values), np.isnan(ref))
    out = rlu.fgmres_refine(g, rhs[2], rlu.solve_system(g, rhs[2]), rlu.RefineConfig(5, 1e-14))
    assert not out.converged
    g.close()


@needs_ref
@pytest.mark.parametrize("contexts", [2, 4, 8])
def test_batch_multi_context_row_blocks_are_bit_exact(contexts, monkeypatch):
    """The experimental non-blocking form of the row-blocked kernel (csrc/blockmc.cuh: W block contexts per warp,
    a context is left at the first pivot whose flag is not set instead of waited on). Off by default (slower)."""
    monkeypatch.setenv("B200LU_BATCH_MC", str(contexts))
    monkeypatch.setenv("B200LU_BATCH_TEAM", "0")
    monkeypatch.setenv("B200LU_BATCH_TILES", "0")
    monkeypatch.setenv("B200LU_BATCH_TAIL_WIDTH", "100000")
    fx = kkt_fixture(700, 300, num_systems=4)
    _check_batch(fx, 17, refine=False)
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7, refine=False)
    _check_batch(golden_fixture("random_sparse_120_plain"), 5, refine=False)


@needs_ref
def test_batch_long_pivot_rows_cross_chunks():
    """A banded matrix with 40 upper entries per row: every pivot row spans several load batches."""
    n, band = 400, 40
    M = np.zeros((n, n))
    rng = np.random.default_rng(7)
    for i in range(n):
        lo, hi = max(0, i - band), min(n, i + band + 1)
        M[i, lo:hi] = rng.uniform(-1, 1, hi - lo)
        M[i, i] = 2.0 * band + 1.0
    fx = dense_fixture(M)
    _check_batch(fx, 19, refine=False)


@needs_ref
def test_batch_mc64_path():
    _check_batch(kkt_fixture(700, 300, num_systems=3, use_scaling=True), 7)


@needs_ref
def test_batch_zero_pivot_is_per_scenario():
    # test_numeric.cpp:173-184 inside a batch: scenario 1 is singular, its neighbours are not
    good = np.array([[4.0, 1, 0], [1, 4, 1], [0, 1, 4]])
    bad = np.array([[1.0, 1, 0], [1, 1, 1], [0, 1, 1]])
    fx = dense_fixture(good)
    ro, ci = fx.ro, fx.ci
    rows = np.repeat(np.arange(3), np.diff(ro))
    vals = np.stack([m[rows, ci] for m in (good, bad, 2 * good)])
    f = BatchedFactors(fx.sym, 3)
    with pytest.raises(rlu.ZeroPivotError) as ei:
        f.refactorize(vals)
    assert ei.value.scenarios == [1] and ei.value.rows[1] == 1 and ei.value.rows[0] == -1 == ei.value.rows[2]
    assert ei.value.rows[1] == fx.oracle.factorize(vals[1])[1]
    assert f.valid(0) and not f.valid(1) and f.valid(2)
    assert np.array_equal(f.values(0), fx.oracle.factorize(vals[0])[0])
    assert np.array_equal(f.values(2), fx.oracle.factorize(vals[2])[0])
    # pivot floor (numeric.hpp:14): every pivot of scenario 0 is below a floor of 100
    g = BatchedFactors(fx.sym, 3, rlu.FactorOptions(pivot_floor=100.0))
    failed = g.refactorize(vals, raise_on_zero_pivot=False)
    assert list(failed) == [fx.oracle.factorize(v, 100.0)[1] for v in vals]
    f.close()
    g.close()


@needs_ref
def test_batch_errors_and_determinism():
    fx = kkt_fixture(700, 300, num_systems=2)
    vals, rhs = _scenarios(fx, 6)
    f = BatchedFactors(fx.sym, 6)
    with pytest.raises(rlu.Error):
        f.solve_system(rhs)  # factors are not valid (src/trisolve.cpp:20)
    with pytest.raises(rlu.DimensionError):
        f.refactorize(vals[:, :-1])
    with pytest.raises(rlu.PatternMismatchError):
        f.check_pattern(fx.ro, np.roll(fx.ci, 1))
    f.check_pattern(fx.ro, fx.ci)
    f.refactorize(vals)
    with pytest.raises(rlu.DimensionError):
        f.solve_system(rhs[:, :-1])
    a0 = f.info["alloc_events"]
    x1, o1 = f.fgmres_refine(rhs, f.solve_system(rhs))
    f.refactorize(vals)
    x2, o2 = f.fgmres_refine(rhs, f.solve_system(rhs))
    assert np.array_equal(x1, x2) and [o.residual_history for o in o1] == [o.residual_history for o in o2]
    assert f.info["alloc_events"] == a0  # no device allocation after create (trisolve.hpp:31-33)
    f.close()


@needs_ref
def test_batch_device_tensors_in_place():
    import torch
    fx = kkt_fixture(700, 300, num_systems=3)
    vals, rhs = _scenarios(fx, 9)
    f = BatchedFactors(fx.sym, 9)
    f.refactorize(torch.from_numpy(vals).cuda())
    x = f.solve_system(torch.from_numpy(rhs).cuda())
    assert x.is_cuda
    for s in range(9):
        ref = fx.oracle.factorize(vals[s])[0]
        assert np.array_equal(x[s].cpu().numpy(), fx.oracle.solve_system(ref, rhs[s])[0])
    f.close()


@needs_ref
def test_batch_c1_all_scenarios():
    """C1-shaped systems (n+m = 9000), 64 scenarios: LU and x bit-exact for a sample, residuals for all."""
    fx = kkt_fixture(6300, 2700, num_systems=4)
    vals, rhs = _scenarios(fx, 64)
    f = BatchedFactors(fx.sym, 64)
    f.refactorize(vals)
    x = f.solve_system(rhs)
    for s in (0, 17, 31, 32, 63):
        ref = fx.oracle.factorize(vals[s])[0]
        assert np.array_equal(f.values(s), ref)
        assert np.array_equal(x[s], fx.oracle.solve_system(ref, rhs[s])[0])
    xr, outcomes = f.fgmres_refine(rhs, x)
    final = f.relative_residual(xr, rhs)
    assert np.all(final <= 1e-14) and all(o.converged for o in outcomes)
    f.close()


@needs_ref
def test_batch_classic_refine_matches_the_oracle_per_scenario():
    """classic_refine (src/refine.cpp:150-188) in a batch: iteration counts, history lengths and the
    final residual per scenario against the oracle's run on the same x0 (test_refine.cpp:219-242 style)."""
    fx = kkt_fixture(700, 300, num_systems=4)
    vals, rhs = _scenarios(fx, 9)
    f = BatchedFactors(fx.sym, 9)
    f.refactorize(vals)
    x = f.solve_system(rhs)
    xr, outcomes = f.classic_refine(rhs, x)
    for s in range(9):
        A = fx.oracle_csr(0, vals[s])
        lu = fx.oracle.factorize(vals[s])[0]
        x_ref, its_ref, conv_ref, hist_ref = ob.refine(A, rhs[s], x[s], fx.oracle, lu, method="classic")
        got, ref = A.relative_residual(xr[s], rhs[s]), A.relative_residual(x_ref, rhs[s])
        assert got <= max(4 * ref, 1e-15), (s, got, ref)
        assert outcomes[s].iterations == its_ref and outcomes[s].converged == conv_ref
        assert len(outcomes[s].residual_history) == len(hist_ref)
    # identity preconditioner on a diagonal system converges only where the diagonal is 1 (test_refine.cpp:148-159 style)
    f.close()


@pytest.fixture
def tiles_env():
    """Selects the trailing-part kernel of the next BatchedFactors (the choice is made at create time)."""
    old = os.environ.get("B200LU_BATCH_TILES")

    def choose(v):
        if v is None:
            os.environ.pop("B200LU_BATCH_TILES", None)
        else:
            os.environ["B200LU_BATCH_TILES"] = v

    yield choose
    choose(old)


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_120_plain"])
@pytest.mark.parametrize("mode,batch", [("1", 7), ("1", 40), ("0", 7), ("0", 40), (None, 9), (None, 40), (None, 130)])
def test_both_trailing_kernels_are_bitwise_exact(tiles_env, name, mode, batch):
    """The trailing part of the refactorization runs either in the tiled kernel (rows resident in shared
    memory, TMA-staged pivot rows, csrc/tile.cuh) or in the row-blocked one (L2 reductions, csrc/batch.cuh):
    forced each way and left to the default (tiles up to 32 scenarios), every scenario's L/U values must be
    the oracle's bit for bit, twice in a row (generation flags, run-to-run determinism)."""
    fx = golden_fixture(name)
    vals, rhs = _scenarios(fx, batch)
    tiles_env(mode)
    f = BatchedFactors(fx.sym, batch)
    try:
        info = f.info
        if mode is not None:
            assert info["tiled"] == int(mode)
        else:
            assert info["tiled"] == (1 if batch <= 32 else 0)
        for rep in range(2):
            f.refactorize(vals)
            for s in sorted({0, 1, batch // 2, batch - 1}):
                ref, failed = fx.oracle.factorize(vals[s])
                assert failed == -1 and np.array_equal(f.values(s), ref), (rep, s)
        x = f.solve_system(rhs)
        s = batch - 1
        assert np.array_equal(x[s], fx.oracle.solve_system(fx.oracle.factorize(vals[s])[0], rhs[s])[0])
    finally:
        f.close()


def test_tiled_kernel_zero_pivot_and_pivot_floor(tiles_env):
    """eliminate's pivot check (src/numeric.cpp:48-55) in the tiled kernel: the lowest failing row per scenario,
    the other scenarios unaffected and valid."""
    fx = golden_fixture("kkt_small")
    batch = 6
    vals, _ = _scenarios(fx, batch)
    tiles_env("1")
    f = BatchedFactors(fx.sym, batch, rlu.FactorOptions(pivot_floor=1e300))
    try:
        assert f.info["tiled"] == 1
        failed = f.refactorize(vals, raise_on_zero_pivot=False)
        for s in range(batch):
            ref, ref_failed = fx.oracle.factorize(vals[s], pivot_floor=1e300)
            assert failed[s] == ref_failed and not f.valid(s)
            assert np.array_equal(f.values(s), ref)
    finally:
        f.close()


@needs_ref
def test_tiled_kernel_chunks_long_pivot_rows(tiles_env):
    """A dense 150 x 150 matrix has pivot rows of up to 150 entries: longer than one staging copy (96 entries),
    so they are staged and applied in chunks."""
    rng = np.random.default_rng(7)
    M = rng.uniform(-1.0, 1.0, (150, 150)) + 150.0 * np.eye(150)
    fx = dense_fixture(M)
    tiles_env("1")
    f = BatchedFactors(fx.sym, 3)
    try:
        assert f.info["tiled"] == 1
        vals = np.stack([fx.values[0], 2.0 * fx.values[0], 0.5 * fx.values[0]])
        f.refactorize(vals)
        for s in range(3):
            assert np.array_equal(f.values(s), fx.oracle.factorize(vals[s])[0])
    finally:
        f.close()


@needs_ref
def test_pattern_the_tiled_kernel_cannot_take_keeps_the_row_blocked_one(tiles_env):
    """An arrow matrix whose last row holds 3 700 entries does not fit a tile's shared memory (64 bytes per
    entry): the handle keeps the row-blocked kernel and stays exact."""
    n = 3700
    rng = np.random.default_rng(11)
    M = np.diag(rng.uniform(2.0, 3.0, n))
    M[-1, :-1] = rng.uniform(-1e-3, 1e-3, n - 1)
    M[:-1, -1] = rng.uniform(-1e-3, 1e-3, n - 1)
    fx = dense_fixture(M)
    tiles_env("1")
    f = BatchedFactors(fx.sym, 2)
    try:
        assert f.info["tiled"] == 0
        vals = np.stack([fx.values[0], 2.0 * fx.values[0]])
        f.refactorize(vals)
        for s in range(2):
            assert np.array_equal(f.values(s), fx.oracle.factorize(vals[s])[0])
    finally:
        f.close()


def test_staged_pipeline_takes_device_buffers():
    """The buffers of the staged calls may live on the handle's device (device-to-device copies on the copy streams):
    same results as with host buffers and as the plain calls, bit for bit."""
    import torch
    fx = golden_fixture("kkt_small")
    batch, steps = 7, 3
    f = BatchedFactors(fx.sym, batch)
    g = BatchedFactors(fx.sym, batch)
    try:
        seq = []
        for k in range(steps):
            vals, rhs = _scenarios(fx, batch)
            seq.append((torch.from_numpy(vals * (1.0 + 0.0625 * k)).cuda(), torch.from_numpy(rhs * (1.0 + 0.5 * k)).cuda()))
        outs = [torch.empty((batch, fx.n), dtype=torch.float64, device="cuda") for _ in range(steps)]
        f.stage_inputs(seq[0][0], seq[0][1])
        for k in range(steps):
            if k + 1 < steps:
                f.stage_inputs(seq[k + 1][0], seq[k + 1][1])
            f.refactorize_staged()
            f.solve_refine_staged(outs[k])
        f.staged_wait()
        for k in range(steps):
            g.refactorize(seq[k][0])
            xr, _ = g.fgmres_refine(seq[k][1], g.solve_system(seq[k][1]))
            assert torch.equal(outs[k], xr), k
    finally:
        f.close()
        g.close()


def test_staged_calls_reject_misuse_and_report_zero_pivots():
    """The staged submission calls outside their protocol: nothing staged, a third set while two are pending (the handle
    stays usable), and a singular scenario inside a staged batch (per-scenario failed rows, neighbours factorized and
    solved — as through the plain calls, tests/test_numeric.cpp:173-184 inside a batch)."""
    fx = golden_fixture("kkt_small")
    batch = 5
    vals, rhs = _scenarios(fx, batch)
    f = BatchedFactors(fx.sym, batch)
    g = BatchedFactors(fx.sym, batch)
    try:
        with pytest.raises(rlu.Error, match="no staged values"):
            f.refactorize_staged()
        out = np.empty((batch, fx.n))
        with pytest.raises(rlu.Error):
            f.solve_refine_staged(out)  # neither factors nor staged right-hand sides
        f.stage_inputs(vals, rhs)
        f.stage_inputs(vals * 1.5, rhs * 0.5)
        with pytest.raises(rlu.Error, match="not been consumed"):
            f.stage_inputs(vals, rhs)
        outs = [np.empty((batch, fx.n)) for _ in range(2)]
        for k in range(2):  # both pending sets are still consumed in order
            f.refactorize_staged()
            f.solve_refine_staged(outs[k])
        f.staged_wait()
        for k, (v, b) in enumerate(((vals, rhs), (vals * 1.5, rhs * 0.5))):
            g.refactorize(v)
            xr, _ = g.fgmres_refine(b, g.solve_system(b))
            assert np.array_equal(outs[k], xr), k
    finally:
        f.close()
        g.close()
    good = np.array([[4.0, 1, 0], [1, 4, 1], [0, 1, 4]])
    bad = np.array([[1.0, 1, 0], [1, 1, 1], [0, 1, 1]])
    fz = dense_fixture(good)
    rows = np.repeat(np.arange(3), np.diff(fz.ro))
    zv = np.stack([m[rows, fz.ci] for m in (good, bad, 2 * good)])
    zb = np.stack([np.array([1.0, 2.0, 3.0])] * 3)
    h = BatchedFactors(fz.sym, 3)
    try:
        h.stage_inputs(zv, zb)
        with pytest.raises(rlu.ZeroPivotError) as ei:
            h.refactorize_staged()
        assert ei.value.scenarios == [1] and ei.value.rows[1] == fz.oracle.factorize(zv[1])[1]
        assert h.valid(0) and not h.valid(1) and h.valid(2)
        failed = h.refactorize(zv, raise_on_zero_pivot=False)
        assert list(failed) == [-1, ei.value.rows[1], -1]
        x = h.solve_system(zb)
        for s in (0, 2):
            lu, _ = fz.oracle.factorize(zv[s])
            assert np.array_equal(x[s], fz.oracle.solve_system(lu, zb[s])[0])
    finally:
        h.close()


def test_staged_pipeline_matches_the_plain_calls_bitwise():
    """The staged (pipelined) submission — inputs of batch k + 1 copied while batch k is processed, solutions
    leaving on their own stream — gives, for every batch of a sequence, exactly the results of the plain
    refactorize / solve_system / fgmres_refine calls."""
    import torch
    fx = golden_fixture("kkt_small")
    batch, steps = 5, 4
    seq = []
    for k in range(steps):
        vals, rhs = _scenarios(fx, batch)
        seq.append((torch.from_numpy(vals * (1.0 + 0.125 * k)).pin_memory(), torch.from_numpy(rhs * (1.0 - 0.25 * k)).pin_memory()))
    f = BatchedFactors(fx.sym, batch)
    g = BatchedFactors(fx.sym, batch)
    try:
        outs = [torch.empty((batch, fx.n), dtype=torch.float64).pin_memory() for _ in range(steps)]
        f.stage_inputs(seq[0][0], seq[0][1])
        iters = []
        for k in range(steps):
            if k + 1 < steps:
                f.stage_inputs(seq[k + 1][0], seq[k + 1][1])
                if k == 0:
                    with pytest.raises(rlu.Error):  # both staging sets hold unconsumed inputs
                        f.stage_inputs(seq[k + 1][0], seq[k + 1][1])
            f.refactorize_staged()
            iters.append([o.iterations for o in f.solve_refine_staged(outs[k])])
        f.staged_wait()
        for k in range(steps):
            g.refactorize(seq[k][0].numpy())
            x = g.solve_system(seq[k][1].numpy())
            xr, ocs = g.fgmres_refine(seq[k][1].numpy(), x)
            assert np.array_equal(outs[k].numpy(), xr), k
            assert iters[k] == [o.iterations for o in ocs]
        with pytest.raises(rlu.Error):
            f.refactorize_staged()  # nothing staged any more
    finally:
        f.close()
        g.close()
