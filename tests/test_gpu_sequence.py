"""The sequence driver (paper_2306_14337_b200/sequence.py, mirror of cli::solve_sequence) and the
device-resident KKT value path (b200lu_kkt_update), on the B200.

Restates proj/tests/test_cli.cpp (29-86, 211-241) against the device path; the symbolic analysis is the
reference's own, through the bridge (the host oracle of DESIGN.md §1)."""
import json

import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from paper_2306_14337_b200.sequence import (KktDiagonal, KktSystem, PipelineOptions, solve_sequence)
from oracle import oraclebridge as ob
from oracle import refbridge as rb

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not rb.available(), reason="oracle/_ref/librlu_ref.so not built")]


def analyze(K, use_scaling, use_amd):
    A = rb.RefCsr.from_arrays(K.nrows, K.row_offsets, K.col_indices, np.asarray(K.values, dtype=np.float64))
    return rlu.SymbolicFactors.from_arrays(rb.RefSymbolic(A, use_scaling=use_scaling, use_amd=use_amd).arrays())


def generated(n=140, m=60, **kw):
    """gen_sequence with the blocks kept (small_config of test_cli.cpp:17-25 is n=140, m=60)."""
    q = rb.RefSequence(n, m, keep_blocks=True, **kw)
    ro, ci = q.pattern()
    systems = [KktSystem(rlu.CsrMatrix(q.n, q.n, ro, ci, q.values(k)), q.rhs(k), k, q.mu(k)) for k in range(len(q))]
    dps, dds = zip(*(q.deltas(k) for k in range(len(q))))
    blocks = KktDiagonal(n, q.h_diag(0), [q.d_y(k) for k in range(len(q))], list(dps), list(dds))
    return q, systems, blocks


def analyses(rep):
    return sum(1 for r in rep.systems if r.analyze_ms > 0.0)


def test_kkt_update_reproduces_assemble_kkt_bitwise():
    q, systems, blocks = generated()
    sym = analyze(systems[0].K, False, True)
    orc = ob.Factors(sym)
    pos = np.nonzero(np.repeat(np.arange(q.n), np.diff(systems[0].K.row_offsets)) == systems[0].K.col_indices)[0]
    f = rlu.NumericFactors(sym)
    rlu.kkt_bind(f, blocks.n_primal, blocks.h_diag, pos)
    with pytest.raises(rlu.Error):
        rlu.kkt_update(f, blocks.d_y[0], 1e-8, 1e-8)  # no full set of values yet
    rlu.reset_values(f, systems[0].K)
    for k in range(len(systems)):
        rlu.kkt_update(f, blocks.d_y[k], blocks.delta_p[k], blocks.delta_d[k])
        assert not f.valid
        assert np.array_equal(f.values, orc.scatter_values(systems[k].K.values))
        rlu.factorize_scattered(f)
        assert np.array_equal(f.values, orc.factorize(systems[k].K.values)[0])
    # the regularization step of the escalation (cli.cpp:53, 148-154), against the reference's own re-assembly
    q.double_regularization(2)
    dp, dd = q.deltas(2)
    assert (dp, dd) == (2 * blocks.delta_p[2], 2 * blocks.delta_d[2])
    rlu.kkt_update(f, blocks.d_y[2], dp, dd)
    assert np.array_equal(f.values, orc.scatter_values(q.values(2)))
    with pytest.raises(rlu.Error):
        rlu.kkt_update(f, blocks.d_y[2], -1.0, 0.0)  # src/kkt.cpp:44-46
    f.close()
    # scenario batch: every scenario its own D_y
    B = 5
    g = BatchedFactors(sym, B)
    g.kkt_bind(blocks.n_primal, blocks.h_diag, pos)
    g.reset_values(np.stack([systems[0].K.values] * B))
    g.kkt_update(np.stack([blocks.d_y[k] for k in range(B)]), blocks.delta_p[0], blocks.delta_d[0])
    g.factorize_scattered()
    for k in range(B):
        assert np.array_equal(g.values(k), orc.factorize(systems[k].K.values)[0])
    g.close()


def test_default_generated_sequence_one_analysis_ten_solved():
    # test_cli.cpp:29-45 (KLU-style path: 79-86)
    for scaling in (True, False):
        q, systems, blocks = generated()
        rep = solve_sequence(systems, analyze, PipelineOptions(use_scaling=scaling, refine="fgmres"), blocks)
        assert len(rep.systems) == 10 and analyses(rep) == 1 and rep.systems[0].analyze_ms > 0.0
        assert rep.reanalysis_count == 0 and rep.systems_solved == 10
        for r in rep.systems:
            assert r.status == "ok" and r.relres_final <= 1e-8
            assert r.relres_final <= r.relres_direct * (1 + 1e-12)
        doc = json.loads(rep.to_json())  # report_to_json's keys, src/report.cpp:30-66
        assert set(doc) == {"systems", "aggregate"} and len(doc["systems"]) == 10
        assert set(doc["systems"][0]) == {"k", "n", "nnz", "analyze_ms", "scatter_ms", "factor_ms", "trisolve_ms",
                                          "refine_ms", "refine_iters", "relres_direct", "relres_final", "status"}
        assert set(doc["aggregate"]) == {"total_ms", "mean_phase_ms", "systems_solved", "reanalysis_count"}


def test_diagonal_path_matches_full_value_path():
    """With and without the KKT blocks (device-side diagonal rewrite vs full reset_values) the
    sequence takes the same residual path, bit for bit."""
    q, systems, blocks = generated()
    opt = PipelineOptions(use_scaling=False, refine="fgmres")
    a, xa = solve_sequence(systems, analyze, opt, blocks, keep_solutions=True)
    b, xb = solve_sequence(systems, analyze, opt, None, keep_solutions=True)
    for ra, rb_, x1, x2 in zip(a.systems, b.systems, xa, xb):
        assert ra.relres_direct == rb_.relres_direct and ra.relres_final == rb_.relres_final
        assert ra.refine_iters == rb_.refine_iters and np.array_equal(x1, x2)


def test_refine_none_and_classic():
    # test_cli.cpp:47-65
    q, systems, blocks = generated()
    rep = solve_sequence(systems, analyze, PipelineOptions(refine="none"), blocks)
    for r in rep.systems:
        assert r.refine_ms == 0.0 and r.refine_iters == 0 and r.relres_final == r.relres_direct
    rep = solve_sequence(systems, analyze, PipelineOptions(refine="classic"), blocks)
    assert rep.systems_solved == 10


def test_pattern_break_triggers_exactly_one_reanalysis():
    # test_cli.cpp:67-77: an explicit zero at an absent slot of row 0 from system 3 on
    q, systems, blocks = generated()
    K0 = systems[0].K
    ro, ci = np.asarray(K0.row_offsets), np.asarray(K0.col_indices)
    col = next(c for c in range(K0.ncols) if c not in set(ci[ro[0]:ro[1]]))
    ins = ro[0] + int(np.searchsorted(ci[ro[0]:ro[1]], col))
    ro2 = ro.copy()
    ro2[1:] += 1
    ci2 = np.insert(ci, ins, col)
    for k in range(3, len(systems)):
        systems[k].K = rlu.CsrMatrix(K0.nrows, K0.ncols, ro2, ci2, np.insert(systems[k].K.values, ins, 0.0))
    rep = solve_sequence(systems, analyze, PipelineOptions(refine="fgmres"), None)
    assert rep.reanalysis_count == 1 and rep.systems_solved == 10 and analyses(rep) == 2
    assert rep.systems[3].analyze_ms > 0.0


def test_unsalvageable_system_is_reported_failed():
    # test_cli.cpp:211-241: natural order, no scaling, exact zero pivot at row 1, no blocks to strengthen
    ro, ci = np.array([0, 2, 5, 7]), np.array([0, 1, 0, 1, 2, 1, 2])
    K = rlu.CsrMatrix(3, 3, ro, ci, np.ones(7))
    rep = solve_sequence([KktSystem(K, np.ones(3))], analyze, PipelineOptions(use_scaling=False, use_amd=False), None)
    assert len(rep.systems) == 1 and rep.systems[0].status == "failed"
    assert rep.systems_solved == 0 and rep.reanalysis_count == 1
    # a permuted variant that natural order handles: same policy, solved at the first attempt
    K2 = rlu.CsrMatrix(3, 3, ro, ci, np.array([2.0, 1, 1, 3, 1, 1, 2]))
    rep = solve_sequence([KktSystem(K2, np.ones(3))], analyze, PipelineOptions(use_scaling=False, use_amd=False), None)
    assert rep.systems_solved == 1 and rep.reanalysis_count == 0


def test_regularization_escalation_on_the_device():
    """delta_d = 0 on the AMD-only path: every system hits an exact zero pivot (the oracle reports
    row 5); the policy doubles the regularization (0 -> 1e-12, cli.cpp:53) — here a device-side
    diagonal rewrite — and the retry succeeds without a re-analysis."""
    q, systems, blocks = generated(n=70, m=30, delta_d=0.0)
    sym = analyze(systems[0].K, False, True)
    assert ob.Factors(sym).factorize(systems[0].K.values)[1] == 5
    rep, xs = solve_sequence(systems, analyze, PipelineOptions(use_scaling=False, refine="fgmres"), blocks,
                             keep_solutions=True)
    assert rep.systems_solved == len(systems) and rep.reanalysis_count == 0 and analyses(rep) == 1
    # the accepted solution solves the REGULARIZED system the reference would have re-assembled
    q.double_regularization(1)
    assert q.deltas(1) == (2 * blocks.delta_p[1], 1e-12)
    assert q.matrix(1).relative_residual(xs[1], q.rhs(1)) <= 1e-8
