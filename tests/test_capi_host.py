"""CPU-side checks of the shipped library: it loads, exports exactly what include/b200lu.h declares,
refuses to compute without a device (no CPU fallback), and its host-side schedule derivation is a
valid replacement for the reference scheduler's claim order (include/rlu/schedule.hpp:49-79)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2306_14337_b200 import _capi
from tests.fixtures import golden_fixture

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "b200lu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(b200lu_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _capi.lib()
    declared = _declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(L, name), f"{name} declared in include/b200lu.h but not exported"
    assert set(declared) == set(_capi.EXPORTS), "ctypes binding and header disagree"


def test_product_does_not_touch_the_oracle():
    """The shipped package must never import, link or load anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2306_14337_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "rlu_oracle" not in text and "refbridge" not in text and "oraclebridge" not in text, f
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, flags=re.M), f
    out = os.popen(f"ldd {_capi.LIB_PATH}").read()
    assert "librlu" not in out


def _view(sym):
    v = _capi.SymbolicView()
    v.n, v.nnz_factors, v.nnz_source = sym.n, int(sym.row_offsets[-1]), len(sym.scatter_map)
    v.row_offsets, v.col_indices, v.diag_pos = (a.ctypes.data for a in (sym.row_offsets, sym.col_indices, sym.diag_pos))
    v.scatter_map, v.scatter_scale, v.amd_forward = sym.scatter_map.ctypes.data, sym.scatter_scale.ctypes.data, sym.amd_forward.ctypes.data
    v.source_row_offsets, v.source_col_indices = sym.src_row_offsets.ctypes.data, sym.src_col_indices.ctypes.data
    return v


@pytest.mark.skipif(_capi.lib().b200lu_device_count() > 0, reason="a device is present")
def test_no_device_means_no_result():
    fx = golden_fixture("kkt_small")
    h = C.c_void_p()
    st = _capi.lib().b200lu_create(C.byref(_view(fx.sym)), None, C.byref(h))
    assert st == _capi.NO_DEVICE and not h
    st = _capi.lib().b200lu_batch_create(C.byref(_view(fx.sym)), None, 4, C.byref(h))
    assert st == _capi.NO_DEVICE and not h
    import paper_2306_14337_b200 as rlu
    with pytest.raises(rlu.DeviceError):
        rlu.NumericFactors(fx.sym)


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_120_plain"])
def test_schedule_probe_orders_are_topological(name):
    fx = golden_fixture(name)
    s = fx.sym
    n = s.n
    stats = _capi.Stats()
    lo = np.empty(n, dtype=np.int32)
    uo = np.empty(n, dtype=np.int32)
    prp = np.empty(n + 1, dtype=np.int64)
    err = C.create_string_buffer(256)
    st = _capi.lib().b200lu_schedule_probe(C.byref(_view(s)), C.byref(stats), lo.ctypes.data, uo.ctypes.data,
                                            prp.ctypes.data, err, 256)
    assert st == _capi.OK, err.value
    assert sorted(lo) == list(range(n)) and sorted(uo) == list(range(n))
    pos_l = np.empty(n, dtype=np.int64)
    pos_l[lo] = np.arange(n)
    pos_u = np.empty(n, dtype=np.int64)
    pos_u[uo] = np.arange(n)
    ro, ci, dp = s.row_offsets, s.col_indices, s.diag_pos
    pairs = 0
    for i in range(n):
        for k in range(ro[i], dp[i]):      # every L dependency is claimed before its row
            assert pos_l[ci[k]] < pos_l[i]
            pairs += ro[ci[k] + 1] - dp[ci[k]] - 1
        for k in range(dp[i] + 1, ro[i + 1]):  # every U dependency is claimed before its row
            assert pos_u[ci[k]] < pos_u[i]
        assert prp[i + 1] - prp[i] == sum(ro[ci[k] + 1] - dp[ci[k]] - 1 for k in range(ro[i], dp[i]))
    assert stats.update_pairs == pairs == prp[-1]
    assert stats.nnz_lower == int((dp - ro[:-1]).sum())
    assert stats.lower_levels >= 1 and stats.upper_levels >= 1


def test_schedule_probe_rejects_broken_patterns():
    fx = golden_fixture("random_sparse_60")
    s = fx.sym
    bad_diag = s.diag_pos.copy()
    bad_diag[3] += 1
    v = _view(s)
    v.diag_pos = bad_diag.ctypes.data
    err = C.create_string_buffer(256)
    st = _capi.lib().b200lu_schedule_probe(C.byref(v), None, None, None, None, err, 256)
    assert st == _capi.INVALID_ARGUMENT and b"diag_pos[3]" in err.value
    bad_cols = s.col_indices.copy()
    lo = s.row_offsets[5]
    if s.row_offsets[6] - lo >= 2:
        bad_cols[lo], bad_cols[lo + 1] = bad_cols[lo + 1], bad_cols[lo]
        v = _view(s)
        v.col_indices = bad_cols.ctypes.data
        st = _capi.lib().b200lu_schedule_probe(C.byref(v), None, None, None, None, err, 256)
        assert st == _capi.INVALID_ARGUMENT


def _emulate(fx, k, rows_per_tile, tile_entries, tail_width, pivot_floor=1e-30, values=None):
    vals = fx.oracle.scatter_values(fx.values[k] if values is None else values)
    failed = C.c_int64(-1)
    stats = _capi.TilePlanStats()
    err = C.create_string_buffer(256)
    st = _capi.lib().b200lu_tile_plan_emulate(C.byref(_view(fx.sym)), rows_per_tile, tile_entries, tail_width,
                                              pivot_floor, vals.ctypes.data, C.byref(failed), C.byref(stats), err, 256)
    return st, vals, int(failed.value), stats, err.value.decode()


@pytest.mark.parametrize("name", ["kkt_small", "kkt_small_mc64", "random_sparse_120_plain", "random_sparse_60"])
@pytest.mark.parametrize("rows_per_tile,tile_entries", [(8, 4096), (16, 4096), (3, 150), (1, 400)])
def test_tile_plan_reproduces_the_oracle_bitwise(name, rows_per_tile, tile_entries):
    """The plan of the tiled batched refactorization (csrc/tile_plan.hpp: tiling, ascending pivot merge,
    chunking of long pivot rows, destination offsets, topological claim order), executed on the host for
    one system, gives the oracle's L/U bit for bit (eliminate, src/numeric.cpp:27-58). tail_width = a huge
    number puts every level but the first into the tiled part."""
    fx = golden_fixture(name)
    max_row = int(np.diff(fx.sym.row_offsets).max())
    tile_entries = max(tile_entries, max_row)
    for k in range(len(fx.values)):
        st, vals, failed, stats, err = _emulate(fx, k, rows_per_tile, tile_entries, 1 << 40)
        assert st == _capi.OK, err
        ref, ref_failed = fx.oracle.factorize(fx.values[k])
        assert ref_failed == -1 and failed == -1
        assert np.array_equal(vals, ref)
        assert stats.rows > 0 and stats.tiles >= -(-stats.rows // rows_per_tile)
        assert stats.fetched_entries <= stats.consumed_entries
        assert stats.largest_tile_entries <= tile_entries


def test_tile_plan_shares_pivot_rows_and_reports_zero_pivots():
    fx = golden_fixture("kkt_small")
    st, vals, failed, stats, err = _emulate(fx, 0, 8, 1 << 20, 1 << 40)
    assert st == _capi.OK, err
    assert stats.consumed_entries > 1.5 * stats.fetched_entries  # consecutive rows share their pivot rows
    # a row that is too long for a tile is refused, not mangled
    st, _, _, _, err = _emulate(fx, 0, 8, 4, 1 << 40)
    assert st == _capi.INVALID_ARGUMENT and "exceeds" in err
    # zero pivot: the lowest failing row, as eliminate reports it (src/numeric.cpp:48-55)
    v = fx.values[0].copy()
    ref, ref_failed = fx.oracle.factorize(v, pivot_floor=1e300)
    st, vals, failed, _, _ = _emulate(fx, 0, 8, 1 << 20, 1 << 40, pivot_floor=1e300)
    assert st == _capi.ZERO_PIVOT and failed == ref_failed
    assert np.array_equal(vals, ref)


def test_tile_plan_chunks_long_pivot_rows():
    """Pivot rows longer than a TMA stage (96 entries) are cut into chunks: a dense 150 x 150 matrix has
    upper parts of up to 149 entries."""
    from tests.fixtures import dense_fixture, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref/librlu_ref.so not built")
    rng = np.random.default_rng(7)
    M = rng.uniform(-1.0, 1.0, (150, 150)) + 150.0 * np.eye(150)
    fx = dense_fixture(M)
    st, vals, failed, stats, err = _emulate(fx, 0, 8, 4096, 1 << 40)
    assert st == _capi.OK, err
    assert stats.items > stats.rows  # chunked externals
    assert np.array_equal(vals, fx.oracle.factorize(fx.values[0])[0])
