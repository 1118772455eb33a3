"""Structure probe (dev tool): level widths / row work of the reference's L+U pattern.

Uses the reference bridge (test infrastructure) to build the fixture; not part of the product.
"""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import refbridge as rb

def levels(n, ro, ci, dp):
    lev = np.zeros(n, dtype=np.int32)
    # row i level = 1 + max level of L-deps
    for i in range(n):
        lo, d = ro[i], dp[i]
        if d > lo:
            lev[i] = lev[ci[lo:d]].max() + 1
    return lev

def main(n, m, scaling=False):
    t = time.time()
    seq = rb.RefSequence(n, m, num_systems=1)
    print("gen", time.time() - t, "N", seq.n, "nnzA", seq.nnz)
    t = time.time()
    sym = rb.RefSymbolic(seq.matrix(0), use_scaling=scaling, use_amd=True)
    print("analyze ms", sym.analyze_ms, "nnzF", sym.nnz_factors, "hash rows", sym.hash_rows)
    s = sym.arrays()
    N = s.n
    ro, ci, dp = s.row_offsets, s.col_indices, s.diag_pos
    llen = dp - ro[:-1]
    ulen = ro[1:] - dp - 1
    print("L len: mean %.1f p50 %d p90 %d p99 %d max %d" % (llen.mean(), *np.percentile(llen, [50, 90, 99]).astype(int), llen.max()))
    print("U len: mean %.1f p50 %d p90 %d p99 %d max %d" % (ulen.mean(), *np.percentile(ulen, [50, 90, 99]).astype(int), ulen.max()))
    t = time.time()
    lev = levels(N, ro, ci, dp)
    nl = lev.max() + 1
    print("levels", nl, "t", time.time() - t)
    width = np.bincount(lev, minlength=nl)
    # work per row = sum over d in L(i) of ulen[d]
    rowid = np.repeat(np.arange(N), ro[1:] - ro[:-1])
    is_l = ci < rowid
    work = np.bincount(rowid[is_l], weights=ulen[ci[is_l]].astype(np.float64), minlength=N)
    print("pairs total", work.sum(), "pivots", is_l.sum())
    wl = np.bincount(lev, weights=work, minlength=nl)
    cum_rows = np.cumsum(width) / N
    cum_work = np.cumsum(wl) / work.sum()
    for L in [10, 50, 100, 200, 300, 500, 800, 1000, 1200, 1400, nl - 1]:
        if L < nl:
            print(f"  level<= {L}: rows {cum_rows[L]:.4f} work {cum_work[L]:.4f} width@L {width[L]} ")
    narrow = width < 32
    print("levels width<32:", narrow.sum(), "rows in them", width[narrow].sum(), "work frac", wl[narrow].sum() / work.sum())
    first_narrow = np.argmax(narrow)
    print("first narrow level", first_narrow)
    # rows in tail region (level >= first level where all subsequent are narrow)
    last_wide = np.max(np.nonzero(~narrow)[0])
    print("last wide level", last_wide, "rows after", width[last_wide + 1:].sum(), "work after", wl[last_wide + 1:].sum() / work.sum())
    tail_rows = np.nonzero(lev > last_wide)[0]
    print("tail rows idx range", tail_rows.min(), tail_rows.max(), "count", tail_rows.size, " N-min", N - tail_rows.min())
    print("tail L nnz", llen[tail_rows].sum(), "of", llen.sum(), " tail U nnz", ulen[tail_rows].sum())
    # heaviest rows
    order = np.argsort(-work)[:10]
    print("heaviest rows:", [(int(i), int(llen[i]), int(work[i]), int(lev[i])) for i in order])
    # critical path weighted by per-row serial cost (pivots) : longest path where cost(row)=llen
    # cp[i] = llen[i] + max cp[d]
    cp = np.zeros(N)
    for i in range(N):
        lo, d = ro[i], dp[i]
        cp[i] = llen[i] + (cp[ci[lo:d]].max() if d > lo else 0)
    print("critical path in pivots (serial per-row pivot cost):", cp.max())
    np.savez("/tmp/struct_%d.npz" % N, lev=lev, width=width, work=work, llen=llen, ulen=ulen)

if __name__ == "__main__":
    n, m = int(sys.argv[1]), int(sys.argv[2])
    main(n, m, len(sys.argv) > 3 and sys.argv[3] == "mc64")
