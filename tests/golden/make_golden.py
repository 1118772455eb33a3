"""Generates the committed golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (where /root/reference exists and `make -C oracle ref` has been run):
    python tests/golden/make_golden.py
Outputs (committed): tests/golden/*.npz, tests/golden/checksums.json
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import refbridge as rb  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sym_dict(arrays):
    d = {"n": arrays.n, "fill_count": arrays.fill_count}
    for k in ("row_offsets", "col_indices", "diag_pos", "scatter_map", "scatter_scale", "amd_forward",
              "src_row_offsets", "src_col_indices"):
        d["sym_" + k] = getattr(arrays, k)
    if arrays.col_perm_forward is not None:
        for k in ("col_perm_forward", "row_scale", "col_scale"):
            d["sym_" + k] = getattr(arrays, k)
    return d


def run_systems(d, sym, mats, values, rhs):
    num = rb.RefNumeric(sym)
    d["num_systems"] = len(mats)
    for k, (A, v, b) in enumerate(zip(mats, values, rhs)):
        d[f"values_{k}"], d[f"rhs_{k}"] = v, b
        num.reset_values(A)
        d[f"scattered_{k}"] = num.values()
        num.factorize_scattered()
        d[f"lu_{k}"] = num.values()
        d[f"lower_{k}"] = num.lower_solve(b)
        d[f"upper_{k}"] = num.upper_solve(b)
        x = num.solve_system(b)
        d[f"x_{k}"] = x
        d[f"relres_{k}"] = A.relative_residual(x, b)
        r = rb.refine(A, b, x, num)
        d[f"xref_{k}"], d[f"hist_{k}"], d[f"iters_{k}"] = r.x, r.residual_history, r.iterations


def kkt_small(name, scaling):
    seq = rb.RefSequence(140, 60)
    sym = rb.RefSymbolic(seq.matrix(0), use_scaling=scaling, use_amd=True)
    ro, ci = seq.pattern()
    d = sym_dict(sym.arrays())
    d["src_row_offsets"], d["src_col_indices"] = ro, ci
    K = len(seq)
    run_systems(d, sym, [seq.matrix(k) for k in range(K)], [seq.values(k) for k in range(K)],
                [seq.rhs(k) for k in range(K)])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)


def random_sparse_case(name, seed, n, extra, dd, scaling, amd):
    rng = rb.RefRng(seed)
    A = rng.random_sparse(n, extra, 0.1, 1.0, dd)
    b = rng.random_vector(n)
    sym = rb.RefSymbolic(A, use_scaling=scaling, use_amd=amd)
    ro, ci, v = A.arrays()
    d = sym_dict(sym.arrays())
    d["src_row_offsets"], d["src_col_indices"] = ro, ci
    run_systems(d, sym, [A], [v], [b])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)


def checksums():
    out = {}
    for name, n, m in (("C1", 6300, 2700), ("C2", 39000, 16700), ("C3", 166600, 71400)):
        seq = rb.RefSequence(n, m)
        sym = rb.RefSymbolic(seq.matrix(0), use_scaling=False, use_amd=True)
        arr = sym.arrays()
        num = rb.RefNumeric(sym)
        entry = {"n": seq.n, "nnz": seq.nnz, "nnz_factors": sym.nnz_factors, "num_systems": len(seq),
                 "pattern_sha": sha(arr.col_indices), "amd_sha": sha(arr.amd_forward),
                 "scatter_map_sha": sha(arr.scatter_map), "systems": {}}
        for k in (0, len(seq) - 1):
            A, b = seq.matrix(k), seq.rhs(k)
            num.refactorize(A)
            x = num.solve_system(b)
            r = rb.refine(A, b, x, num)
            entry["systems"][str(k)] = {
                "values_sha": sha(seq.values(k)), "rhs_sha": sha(b), "lu_sha": sha(num.values()),
                "x_sha": sha(x), "relres_direct": A.relative_residual(x, b),
                "relres_final": A.relative_residual(r.x, b), "refine_iters": r.iterations,
            }
        out[name] = entry
        print(name, json.dumps(entry["systems"], indent=1))
    with open(os.path.join(HERE, "checksums.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    kkt_small("kkt_small", False)
    kkt_small("kkt_small_mc64", True)
    random_sparse_case("random_sparse_60", 72, 60, 4, True, True, True)
    random_sparse_case("random_sparse_120_plain", 98, 120, 5, True, False, False)
    checksums()
