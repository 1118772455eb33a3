"""Dev tool: makespan lower bound of warp-per-row sync-free elimination (unlimited warps).

finish[i] = t after walking the pivots of row i in ascending order, where each pivot d
costs p0 + p1*ceil(ulen[d]/32) cycles and must start after finish[d] + hop.
"""
import sys, os, time
import numpy as np
import numba
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import refbridge as rb

@numba.njit(cache=True)
def model(n, ro, ci, dp, p0, p1, hop, epi, lanes):
    fin = np.zeros(n)
    waits = 0
    for i in range(n):
        t = 0.0
        for k in range(ro[i], dp[i]):
            d = ci[k]
            ul = ro[d + 1] - dp[d] - 1
            ready = fin[d] + hop
            if ready > t:
                t = ready
                waits += 1
            t += p0 + p1 * ((ul + lanes - 1) // lanes)
        fin[i] = t + epi
    return fin, waits

@numba.njit(cache=True)
def tri_model(n, ro, ci, dp, c, hop, epi):
    # thread-per-row lower solve; each entry costs c cycles serial
    fin = np.zeros(n)
    for i in range(n):
        t = 0.0
        for k in range(ro[i], dp[i]):
            d = ci[k]
            ready = fin[d] + hop
            if ready > t:
                t = ready
            t += c
        fin[i] = t + epi
    return fin

def main(n, m):
    seq = rb.RefSequence(n, m, num_systems=1)
    sym = rb.RefSymbolic(seq.matrix(0), use_scaling=False, use_amd=True)
    s = sym.arrays()
    ghz = 1.9
    for (p0, p1, hop, epi) in [(120, 40, 700, 300), (60, 30, 500, 200), (60, 30, 100, 100), (30, 20, 60, 60)]:
        fin, waits = model(s.n, s.row_offsets, s.col_indices, s.diag_pos, p0, p1, hop, epi, 32)
        print(f"factor p0={p0} p1={p1} hop={hop} epi={epi}: makespan {fin.max():.0f} cyc = {fin.max()/ghz/1e3:.1f} us; waits {waits}")
    for (c, hop, epi) in [(8, 700, 100), (8, 500, 50), (8, 60, 30), (1, 500, 50)]:
        fin = tri_model(s.n, s.row_offsets, s.col_indices, s.diag_pos, c, hop, epi)
        print(f"lower c={c} hop={hop} epi={epi}: makespan {fin.max():.0f} cyc = {fin.max()/ghz/1e3:.1f} us")

if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
