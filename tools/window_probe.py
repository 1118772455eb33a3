"""Dev tool (structure probe on the C2 pattern, host only; uses the reference bridge for the fixture)."""
import sys, os, time
import numpy as np, numba
import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import refbridge as rb

@numba.njit(cache=True)
def probe(n, ro, ci, dp, hist_end, hist_diag):
    # for each row i, pivot d in L(i), entry j in U(d) (strictly upper): dest position in row i
    pos = np.full(n, -1, np.int64)
    tot = 0
    for i in range(n):
        lo, hi = ro[i], ro[i + 1]
        for k in range(lo, hi):
            pos[ci[k]] = k - lo
        ln = hi - lo
        nl = dp[i] - lo
        for k in range(lo, dp[i]):
            d = ci[k]
            for t in range(dp[d] + 1, ro[d + 1]):
                p = pos[ci[t]]
                e = ln - 1 - p
                hist_end[min(e, hist_end.size - 1)] += 1
                q = p - nl  # relative to the diagonal: <0 L part
                hist_diag[min(max(q + 1024, 0), hist_diag.size - 1)] += 1
                tot += 1
        for k in range(lo, hi):
            pos[ci[k]] = -1
    return tot

n, m = int(sys.argv[1]), int(sys.argv[2])
seq = rb.RefSequence(n, m, num_systems=1)
sym = rb.RefSymbolic(seq.matrix(0), use_scaling=False, use_amd=True)
s = sym.arrays()
ro, ci, dp = s.row_offsets, s.col_indices, s.diag_pos
he = np.zeros(2048, np.int64); hd = np.zeros(2048, np.int64)
tot = probe(s.n, ro, ci, dp, he, hd)
print("pairs", tot)
c = np.cumsum(he) / tot
for w in (8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 512):
    print("last %d entries: %.3f" % (w, c[w - 1]))
# relative to diag
upper = hd[1024:].sum() / tot
print("U part (col>=i):", upper)
cl = np.cumsum(hd[:1024][::-1]) / tot  # L part distance 1.. from diag
for w in (8, 16, 32, 64, 128):
    print("L part within %d of diag: %.3f" % (w, cl[w - 1]))
