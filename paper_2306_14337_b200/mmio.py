"""Matrix Market I/O and sequence manifests — the formats `rlu solve-seq --input` reads and `rlu gen --out`
writes (reference proj/src/io.cpp:25-104, proj/src/kkt.cpp:209-256, proj/src/cli.cpp:175-200), so that a
sequence written by the reference can be solved on the device path and vice versa.

Supported, as in the reference: `%%MatrixMarket matrix coordinate real {general|symmetric}`; 1-based
indices; duplicate entries are summed and explicit zeros kept (CooMatrix::canonicalize,
proj/src/sparse.cpp); values are written with `%.17g` (round-trip exact).
"""
from __future__ import annotations

import os

import numpy as np

from . import solver as rlu


class IoError(rlu.Error):
    """rlu::IoError (include/rlu/errors.hpp)."""


def _fail(path, line, what):
    raise IoError(f"{path}:{line}: {what}")


def mm_read(path: str):
    """mm_read (src/io.cpp:25-87) + coo_to_csr: returns (nrows, ncols, row_offsets, col_indices, values) with
    sorted unique columns per row (duplicates summed in file order, as canonicalize does)."""
    try:
        f = open(path, "r")
    except OSError:
        raise IoError(f"cannot open {path}")
    with f:
        line = f.readline()
        lineno = 1
        if not line:
            _fail(path, 1, "empty file, expected Matrix Market banner")
        parts = line.split()
        parts += [""] * (5 - len(parts))
        tag, obj, fmt, fld, symm = (p.lower() for p in parts[:5])
        if tag != "%%matrixmarket":
            _fail(path, lineno, "malformed banner: " + line.rstrip("\n"))
        if obj != "matrix":
            _fail(path, lineno, "unsupported object: " + parts[1])
        if fmt != "coordinate":
            _fail(path, lineno, "unsupported format: " + parts[2])
        if fld != "real":
            _fail(path, lineno, "unsupported field: " + parts[3])
        if symm not in ("general", "symmetric"):
            _fail(path, lineno, "unsupported symmetry: " + parts[4])
        while True:  # size line, after any comment lines
            line = f.readline()
            if not line:
                _fail(path, lineno + 1, "missing size line")
            lineno += 1
            if line.startswith("%") or not line.strip():
                continue
            try:
                nrows, ncols, nnz = (int(t) for t in line.split()[:3])
            except ValueError:
                _fail(path, lineno, "malformed size line: " + line.rstrip("\n"))
            break
        if nrows < 0 or ncols < 0 or nnz < 0:
            _fail(path, lineno, "negative size")
        rows, cols, vals = [], [], []
        seen = 0
        while seen < nnz:
            line = f.readline()
            if not line:
                _fail(path, lineno + 1, f"unexpected end of file, expected {nnz} entries, got {seen}")
            lineno += 1
            if line.startswith("%") or not line.strip():
                continue
            t = line.split()
            try:
                r, c, v = int(t[0]), int(t[1]), float(t[2])
            except (ValueError, IndexError):
                _fail(path, lineno, "malformed entry: " + line.rstrip("\n"))
            if r < 1 or r > nrows or c < 1 or c > ncols:
                _fail(path, lineno, f"index ({r}, {c}) out of range for {nrows} x {ncols}")
            rows.append(r - 1)
            cols.append(c - 1)
            vals.append(v)
            if symm == "symmetric" and r != c:
                rows.append(c - 1)
                cols.append(r - 1)
                vals.append(v)
            seen += 1
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))  # stable: duplicates keep file order, then summed left to right
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        new = np.ones(rows.size, dtype=bool)
        new[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        starts = np.nonzero(new)[0]
        if starts.size != rows.size:  # sum duplicates sequentially (left to right, like canonicalize)
            out = np.empty(starts.size)
            ends = np.append(starts[1:], rows.size)
            for q, (a, b) in enumerate(zip(starts, ends)):
                s = vals[a]
                for t in range(a + 1, b):
                    s += vals[t]
                out[q] = s
            vals = out
        rows, cols = rows[starts], cols[starts]
    row_offsets = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(row_offsets, rows + 1, 1)
    row_offsets = np.cumsum(row_offsets)
    return nrows, ncols, row_offsets, cols, vals


def mm_write(path: str, nrows: int, ncols: int, row_offsets, col_indices, values=None):
    """mm_write (src/io.cpp:89-104)."""
    ro, ci = np.asarray(row_offsets), np.asarray(col_indices)
    try:
        f = open(path, "w")
    except OSError:
        raise IoError(f"cannot open {path} for writing")
    with f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{nrows} {ncols} {len(ci)}\n")
        for i in range(nrows):
            for k in range(int(ro[i]), int(ro[i + 1])):
                v = 0.0 if values is None else float(values[k])
                f.write(f"{i + 1} {int(ci[k]) + 1} {v:.17g}\n")


def load_sequence(manifest_path: str):
    """load_sequence (src/kkt.cpp:209-256): one matrix file per line, an optional right-hand-side file in the
    second column, paths relative to the manifest; patterns must agree across systems; a missing rhs is
    K * ones. Returns a list of sequence.KktSystem."""
    from .sequence import KktSystem
    try:
        lines = open(manifest_path).read().splitlines()
    except OSError:
        raise IoError(f"cannot open manifest {manifest_path}")
    base = os.path.dirname(manifest_path)
    systems, template = [], None
    for line in lines:
        if not line.strip():
            continue
        t = line.split()
        mat_file, rhs_file = t[0], (t[1] if len(t) > 1 else "")
        n, nc, ro, ci, v = mm_read(os.path.join(base, mat_file))
        if n != nc:
            raise IoError(mat_file + ": sequence matrices must be square")
        if rhs_file:
            rn, rc, rro, rci, rv = mm_read(os.path.join(base, rhs_file))
            if rc != 1 or rn != n:
                raise IoError(f"{rhs_file}: right-hand side must be a {n} x 1 vector")
            rhs = np.zeros(n)
            rhs[np.repeat(np.arange(rn), np.diff(rro))] = rv
        else:  # spmv(K, ones): left-to-right accumulation per row (src/sparse.cpp:135-141)
            rhs = np.array([float(np.add.accumulate(v[ro[i]:ro[i + 1]])[-1]) if ro[i + 1] > ro[i] else 0.0 for i in range(n)])
        k = len(systems)
        if template is None:
            template = (ro, ci)
        elif not (np.array_equal(ro, template[0]) and np.array_equal(ci, template[1])):
            raise rlu.PatternMismatchError(f"pattern mismatch at index {k}")
        systems.append(KktSystem(rlu.CsrMatrix(n, n, ro, ci, v), rhs, k, 0.0))
    if not systems:
        raise IoError(f"manifest lists no systems: {manifest_path}")
    return systems


def write_sequence(systems, directory: str):
    """write_sequence (src/cli.cpp:175-200): k_%03d.mtx, rhs_%03d.mtx and manifest.txt."""
    os.makedirs(directory, exist_ok=True)
    with open(os.path.join(directory, "manifest.txt"), "w") as manifest:
        for s in systems:
            kname, rname = f"k_{s.k:03d}.mtx", f"rhs_{s.k:03d}.mtx"
            K = s.K
            mm_write(os.path.join(directory, kname), K.nrows, K.ncols, K.row_offsets, K.col_indices, K.values)
            n = len(s.rhs)
            mm_write(os.path.join(directory, rname), n, 1, np.arange(n + 1), np.zeros(n, dtype=np.int64), s.rhs)
            manifest.write(f"{kname} {rname}\n")
