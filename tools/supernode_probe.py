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
# fundamental supernodes: U(d+1) == U(d) minus {d+1}
same = np.zeros(N, dtype=bool)   # same[d]: d+1 continues d's supernode
extra = np.zeros(N, dtype=np.int64)
for d in range(N - 1):
    a = ci[dp[d] + 1:ro[d + 1]]
    b = ci[dp[d + 1] + 1:ro[d + 2]]
    if a.size and a[0] == d + 1:
        rest = a[1:]
        if rest.size == b.size and np.array_equal(rest, b):
            same[d] = True
        else:
            # how many entries of b are not in rest (fill added) — rest subset of b always
            extra[d] = b.size - rest.size
# supernode sizes
sizes = []
cur = 1
for d in range(N - 1):
    if same[d]: cur += 1
    else: sizes.append(cur); cur = 1
sizes.append(cur)
sizes = np.array(sizes)
print("supernodes", sizes.size, "mean size %.2f" % sizes.mean(), "max", sizes.max())
# work (pairs) by pivot: m^2 ; fraction of pairs in supernodes of size >= k
start = np.concatenate([[0], np.cumsum(sizes)[:-1]])
work = ulen.astype(np.float64) ** 2
tot = work.sum()
sn_of = np.repeat(np.arange(sizes.size), sizes)
for k in (1, 2, 4, 8, 16, 32):
    mask = sizes[sn_of] >= k
    print("pairs in supernodes of size >= %d: %.3f" % (k, work[mask].sum() / tot))
# relaxed: chain d -> d+1 where d+1 is first upper entry of d (etree parent = d+1), count extra entries
chain = np.array([ro[d + 1] - dp[d] - 1 > 0 and ci[dp[d] + 1] == d + 1 for d in range(N - 1)])
print("parent == d+1 fraction (work-weighted): %.3f" % (work[:-1][chain].sum() / tot))
ex = extra[:-1][chain & ~same[:-1]]
print("non-fundamental chain links:", ex.size, "mean extra entries %.1f" % (ex.mean() if ex.size else 0))
