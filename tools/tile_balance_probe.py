"""Dev tool (structure probe on the C2 pattern, host only; uses the reference bridge for the fixture)."""
import sys, numpy as np
import os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from oracle import refbridge as rb
seq = rb.RefSequence(39000, 16700, num_systems=1)
sym = rb.RefSymbolic(seq.matrix(0), use_scaling=False, use_amd=True)
s = sym.arrays()
ro, ci, dp = s.row_offsets, s.col_indices, s.diag_pos
N = s.n
ulen = ro[1:] - dp - 1
llen = dp - ro[:-1]
lev = np.zeros(N, dtype=np.int64)
for i in range(N):
    if dp[i] > ro[i]:
        lev[i] = lev[ci[ro[i]:dp[i]]].max() + 1
width = np.bincount(lev)
# trailing cut: maximal suffix of levels narrower than 1024
cut = len(width)
while cut > 0 and width[cut - 1] < 1024: cut -= 1
tail = np.nonzero((lev >= cut) & (llen > 0))[0]
print("tail rows", tail.size, "levels", len(width) - cut, "cut", cut)
rowid = np.repeat(np.arange(N), ro[1:] - ro[:-1]); is_l = ci < rowid
steps = np.bincount(rowid[is_l], weights=np.ceil(ulen[ci[is_l]] / 8.0), minlength=N)  # m/8 steps per item
items = llen.astype(float)
for c_item in (0.0, 6.0, 12.0):
    work = steps + c_item * items
    for R in (2, 4, 8, 16):
        tot = mx = 0.0
        for b in range(0, tail.size, R):
            w = work[tail[b:b + R]]
            tot += w.sum(); mx += R * w.max()
        print(f"c_item {c_item} R {R}: efficiency {tot / mx:.3f}")
# consecutive-index gaps within tail
gaps = np.diff(tail)
print("consecutive pairs", (gaps == 1).mean())
# how different is work between consecutive tail rows
work = steps + 6 * items
r = np.minimum(work[tail[1:]], work[tail[:-1]]) / np.maximum(work[tail[1:]], work[tail[:-1]])
print("min/max work ratio of neighbours: mean %.3f p10 %.3f" % (r.mean(), np.percentile(r, 10)))
# sorted-by-work tiling (upper bound on balance if tiles could group similar rows)
order = tail[np.argsort(-work[tail])]
tot = mx = 0.0
for b in range(0, order.size, 8):
    w = work[order[b:b + 8]]; tot += w.sum(); mx += 8 * w.max()
print("R 8 grouped by work: efficiency %.3f" % (tot / mx))
