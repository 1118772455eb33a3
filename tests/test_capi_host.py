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
