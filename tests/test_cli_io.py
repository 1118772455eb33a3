"""Matrix Market I/O, sequence manifests and report rendering of the device-path CLI
(`python -m paper_2306_14337_b200`), against the reference's formats: files written by the reference's own
mm_write / write_sequence layout (src/io.cpp:89-104, src/cli.cpp:175-200) load to the same arrays, the JSON and CSV
reports carry the reference's field names (src/report.cpp:30-119). CPU tests: formats and error paths; the GPU test
runs `solve-seq` end to end on a sequence on disk and applies the acceptance-style checks of
proj/tests/acceptance.cpp:236-272 (every system solved to <= 1e-8, exactly one analysis, median refinement
iterations <= 2)."""
import json
import os
import statistics

import numpy as np
import pytest

import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200 import mmio
from paper_2306_14337_b200.__main__ import run_cli
from paper_2306_14337_b200.sequence import KktSystem, SolveReport, SystemRecord
from tests.fixtures import golden_fixture


def _systems(fx):
    return [KktSystem(rlu.CsrMatrix(fx.n, fx.n, fx.ro, fx.ci, fx.values[k]), fx.rhs[k], k, 0.0) for k in range(len(fx.values))]


def test_sequence_round_trip_is_bit_exact(tmp_path):
    fx = golden_fixture("kkt_small")
    mmio.write_sequence(_systems(fx), str(tmp_path))
    text = open(tmp_path / "k_000.mtx").read().splitlines()
    assert text[0] == "%%MatrixMarket matrix coordinate real general"          # src/io.cpp:93
    assert text[1] == f"{fx.n} {fx.n} {len(fx.ci)}"
    assert sorted(os.listdir(tmp_path))[:2] == ["k_000.mtx", "k_001.mtx"] and (tmp_path / "manifest.txt").exists()
    back = mmio.load_sequence(str(tmp_path / "manifest.txt"))
    assert len(back) == len(fx.values)
    for k, s in enumerate(back):
        assert s.k == k and np.array_equal(s.K.row_offsets, fx.ro) and np.array_equal(s.K.col_indices, fx.ci)
        assert np.array_equal(s.K.values, fx.values[k]) and np.array_equal(s.rhs, fx.rhs[k])   # %.17g round trip


def test_mm_read_symmetric_duplicates_comments_and_errors(tmp_path):
    p = tmp_path / "a.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n3 3 4\n1 1 2.0\n3 1 -1.5\n2 2 1.0\n3 1 0.5\n")
    n, nc, ro, ci, v = mmio.mm_read(str(p))
    assert (n, nc) == (3, 3) and list(ro) == [0, 2, 3, 4] and list(ci) == [0, 2, 1, 0]
    assert list(v) == [2.0, -1.0, 1.0, -1.0]      # the mirrored entry exists, duplicates are summed
    for body, what in [("", "empty file"), ("%%MatrixMarket matrix array real general\n1 1\n", "unsupported format"),
                       ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n", "unsupported field"),
                       ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
                       ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "unexpected end of file")]:
        p.write_text(body)
        with pytest.raises(mmio.IoError, match=what):
            mmio.mm_read(str(p))
    with pytest.raises(mmio.IoError, match="cannot open"):
        mmio.mm_read(str(tmp_path / "missing.mtx"))


def test_manifest_rules(tmp_path):
    fx = golden_fixture("kkt_small")
    mmio.write_sequence(_systems(fx)[:2], str(tmp_path))
    (tmp_path / "m2.txt").write_text("k_000.mtx\n\n")               # a missing rhs defaults to K * ones
    s = mmio.load_sequence(str(tmp_path / "m2.txt"))[0]
    assert np.array_equal(s.rhs, fx.oracle_csr(0).spmv(np.ones(fx.n)))
    (tmp_path / "empty.txt").write_text("\n")
    with pytest.raises(mmio.IoError, match="no systems"):
        mmio.load_sequence(str(tmp_path / "empty.txt"))
    mmio.mm_write(str(tmp_path / "other.mtx"), 2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    (tmp_path / "m3.txt").write_text("k_000.mtx\nother.mtx\n")
    with pytest.raises(rlu.PatternMismatchError, match="index 1"):
        mmio.load_sequence(str(tmp_path / "m3.txt"))


def test_report_json_csv_layout_and_cli_report_command(tmp_path, capsys):
    rep = SolveReport(systems=[SystemRecord(0, 10, 40, 1.5, 0.1, 0.2, 0.3, 0.4, 1, 3e-9, 1.5e-16, "ok"),
                               SystemRecord(1, 10, 40, 0.0, 0.1, 0.2, 0.3, 0.4, 2, 1e-3, 1e-3, "failed")], total_ms=9.0)
    rep.finalize()
    d = json.loads(rep.to_json())
    assert list(d) == ["systems", "aggregate"] and list(d["aggregate"]) == ["total_ms", "mean_phase_ms", "systems_solved", "reanalysis_count"]
    assert list(d["systems"][0]) == ["k", "n", "nnz", "analyze_ms", "scatter_ms", "factor_ms", "trisolve_ms", "refine_ms",
                                    "refine_iters", "relres_direct", "relres_final", "status"]     # src/report.cpp:35-46
    assert d["aggregate"]["systems_solved"] == 1 and d["aggregate"]["mean_phase_ms"]["analyze"] == 0.75
    csv = rep.to_csv().splitlines()
    assert csv[0] == "k,n,nnz,analyze_ms,scatter_ms,factor_ms,trisolve_ms,refine_ms,refine_iters,relres_direct,relres_final,status"
    assert csv[1].startswith("0,10,40,1.5,") and csv[1].endswith(",ok") and csv[2].endswith(",failed")
    assert csv[3] == "# total_ms,9" and csv[-2] == "# systems_solved,1" and csv[-1] == "# reanalysis_count,0"
    again = SolveReport.from_json(rep.to_json())
    assert again.to_json() == rep.to_json()
    path = tmp_path / "rep.json"
    path.write_text(rep.to_json())
    assert run_cli(["report", str(path), "--format", "csv"]) == 0
    assert capsys.readouterr().out == rep.to_csv()
    path.write_text("{not json")
    assert run_cli(["report", str(path)]) == 1 and "malformed report" in capsys.readouterr().err
    assert run_cli(["solve-seq", "--input", str(tmp_path / "nope.txt"), "--analyzer", "tests.test_cli_io:_ref_analyze"]) == 1


def _ref_analyze(K, use_scaling, use_amd):
    """The reference's symbolic_analyze through the test bridge (the host oracle of DESIGN.md §1)."""
    from oracle import refbridge as rb
    A = rb.RefCsr.from_arrays(K.nrows, K.row_offsets, K.col_indices, np.asarray(K.values, dtype=np.float64))
    return rlu.SymbolicFactors.from_arrays(rb.RefSymbolic(A, use_scaling=use_scaling, use_amd=use_amd).arrays())


@pytest.mark.gpu
@pytest.mark.parametrize("scaling,refine,analyzer", [("none", "fgmres", "reference"), ("mc64", "classic", "reference"),
                                                     ("none", "fgmres", "builtin"), ("mc64", "fgmres", "builtin")])
def test_solve_seq_from_disk_meets_the_acceptance_checks(tmp_path, scaling, refine, analyzer):
    from oracle import refbridge as rb
    if not rb.available():
        pytest.skip("oracle/_ref/librlu_ref.so not built")
    q = rb.RefSequence(1400, 600)   # n + m = 2000, proj/tests/acceptance.cpp:239-240
    ro, ci = q.pattern()
    mmio.write_sequence([KktSystem(rlu.CsrMatrix(q.n, q.n, ro, ci, q.values(k)), q.rhs(k), k, q.mu(k)) for k in range(len(q))],
                        str(tmp_path / "seq"))
    out = tmp_path / "report.json"
    # the built-in analysis (csrc/analyze.cpp) is the default; the reference's own is the substitute provider
    provider = ["--analyzer", "tests.test_cli_io:_ref_analyze"] if analyzer == "reference" else []
    rc = run_cli(["solve-seq", "--input", str(tmp_path / "seq" / "manifest.txt"), *provider,
                  "--scaling", scaling, "--refine", refine, "--out", str(out)])
    assert rc == 0
    rep = SolveReport.from_json(out.read_text())
    assert len(rep.systems) == len(q) == rep.systems_solved and rep.reanalysis_count == 0
    assert all(r.status == "ok" and r.relres_final <= 1e-8 for r in rep.systems)          # acceptance.cpp:255-262
    assert sum(1 for r in rep.systems if r.analyze_ms > 0.0) == 1                          # exactly one analysis
    assert statistics.median(r.refine_iters for r in rep.systems) <= 2
    assert run_cli(["report", str(out), "--format", "csv", "--out", str(tmp_path / "r.csv")]) == 0
    assert (tmp_path / "r.csv").read_text().splitlines()[0].startswith("k,n,nnz,analyze_ms")
