"""Seeded inputs for the parity tests, the smoke test and the bench.

Inputs come from the reference's own generators through the reference bridge
(`oracle/_ref/librlu_ref.so`: gen_sequence, proj/src/kkt.cpp:94-207; random_sparse,
proj/tests/oracles.hpp:186-210) and its symbolic analysis (proj/src/symbolic.cpp:156-203), or
from the committed fixtures under tests/golden/ (made by tests/golden/make_golden.py).
"""
from __future__ import annotations

import functools
import os
from dataclasses import dataclass, field

import numpy as np

import paper_2306_14337_b200 as rlu
from oracle import oraclebridge as ob
from oracle import refbridge as rb

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Fixture:
    n: int
    ro: np.ndarray            # source pattern
    ci: np.ndarray
    values: list              # per system, source-CSR order
    rhs: list
    sym: rlu.SymbolicFactors  # arrays of the reference's SymbolicFactors
    oracle: ob.Factors = None
    ref_seq: object = None    # RefSequence / RefCsr holders when built from the reference
    ref_sym: object = None
    ref_mats: list = field(default_factory=list)
    golden: dict = field(default_factory=dict)

    def matrix(self, k=0, values=None) -> rlu.CsrMatrix:
        return rlu.CsrMatrix(self.n, self.n, self.ro, self.ci, self.values[k] if values is None else values)

    def oracle_csr(self, k=0, values=None) -> ob.Csr:
        return ob.Csr(self.n, self.ro, self.ci, self.values[k] if values is None else values)

    def ref_matrix(self, k=0) -> "rb.RefCsr":
        if self.ref_seq is not None and isinstance(self.ref_seq, rb.RefSequence):
            return self.ref_seq.matrix(k)
        return self.ref_mats[k]


def have_reference() -> bool:
    return rb.available()


@functools.lru_cache(maxsize=8)
def kkt_fixture(n, m, num_systems=0, use_scaling=False, use_amd=True, topology_seed=1, y_seed=2,
                delta_p=1e-8, delta_d=1e-8) -> Fixture:
    """Generated KKT sequence + analysis, SURVEY §8d. (n, m) = (6300, 2700) is C1, (39000, 16700)
    C2, (166600, 71400) C3, (1120000, 480000) C4."""
    seq = rb.RefSequence(n, m, topology_seed=topology_seed, y_seed=y_seed, num_systems=num_systems,
                         delta_p=delta_p, delta_d=delta_d)
    ro, ci = seq.pattern()
    ref_sym = rb.RefSymbolic(seq.matrix(0), use_scaling=use_scaling, use_amd=use_amd)
    arrays = ref_sym.arrays()
    fx = Fixture(seq.n, ro, ci, [seq.values(k) for k in range(len(seq))],
                 [seq.rhs(k) for k in range(len(seq))], rlu.SymbolicFactors.from_arrays(arrays),
                 ob.Factors(arrays), seq, ref_sym)
    return fx


def csr_fixture(A: "rb.RefCsr", use_scaling=True, use_amd=True, rhs=None) -> Fixture:
    ro, ci, v = A.arrays()
    ref_sym = rb.RefSymbolic(A, use_scaling=use_scaling, use_amd=use_amd)
    arrays = ref_sym.arrays()
    return Fixture(A.n, ro, ci, [v], [rhs if rhs is not None else np.ones(A.n)],
                   rlu.SymbolicFactors.from_arrays(arrays), ob.Factors(arrays), None, ref_sym, [A])


def dense_fixture(M, use_scaling=False, use_amd=False, rhs=None) -> Fixture:
    return csr_fixture(rb.RefCsr.from_dense(M), use_scaling, use_amd, rhs)


class _GoldenSym:
    pass


@functools.lru_cache(maxsize=8)
def golden_fixture(name: str) -> Fixture:
    """Committed fixture: inputs, the reference's analysis arrays and the reference's outputs."""
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"))
    s = _GoldenSym()
    for k in ("row_offsets", "col_indices", "diag_pos", "scatter_map", "scatter_scale", "amd_forward",
              "src_row_offsets", "src_col_indices"):
        setattr(s, k, z["sym_" + k])
    s.n = int(z["n"])
    for k in ("col_perm_forward", "row_scale", "col_scale"):
        setattr(s, k, z["sym_" + k] if ("sym_" + k) in z.files else None)
    s.fill_count = int(z["fill_count"])
    nsys = int(z["num_systems"])
    fx = Fixture(s.n, z["src_row_offsets"], z["src_col_indices"], [z[f"values_{k}"] for k in range(nsys)],
                 [z[f"rhs_{k}"] for k in range(nsys)], rlu.SymbolicFactors.from_arrays(s), ob.Factors(s))
    fx.golden = {k: z[k] for k in z.files if k.startswith(("lu_", "x_", "scattered_", "xref_", "relres_",
                                                           "hist_", "iters_", "lower_", "upper_"))}
    return fx
