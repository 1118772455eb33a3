"""Dev tool (GPU box): per-hop latency of the sync-free kernels on a pure dependency chain.

A tridiagonal matrix in natural order factors into bidiagonal L and U: n dependency levels of width
1, one entry per row. time / n is the cost of one producer->consumer hand-off through L2."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from oracle import refbridge as rb
from tests.fixtures import csr_fixture

def main(n=20000, band=1):
    ro, ci, v = [0], [], []
    for i in range(n):
        for j in range(max(0, i - band), min(n, i + band + 1)):
            ci.append(j); v.append(4.0 * band if i == j else -1.0)
        ro.append(len(ci))
    A = rb.RefCsr.from_arrays(n, ro, ci, v)
    fx = csr_fixture(A, use_scaling=False, use_amd=False)
    for strict in (False, True):
        f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream, strict_order=strict))
        f.set_timing(True)
        b = torch.ones(n, dtype=torch.float64, device="cuda")
        dv = torch.from_numpy(fx.values[0]).cuda()
        for _ in range(4):
            rlu.refactorize(f, rlu.CsrMatrix(n, n, fx.ro, fx.ci, dv))
            x = rlu.solve_system(f, b)
        f.phase_times()
        reps = 5
        for _ in range(reps):
            rlu.refactorize(f, rlu.CsrMatrix(n, n, fx.ro, fx.ci, dv))
            x = rlu.solve_system(f, b)
        ph = f.phase_times()
        st = f.stats
        ok = bool(np.array_equal(f.values, fx.oracle.factorize(fx.values[0])[0]))
        print(json.dumps({"n": n, "band": band, "strict": strict, "levels": st["lower_levels"],
                          "hop_ns": {p: round(1e6 * ph[p][0] / max(ph[p][1], 1) / st["lower_levels"], 1) for p in ("factor", "lower", "upper", "tail")},
                          "launches": {p: ph[p][1] for p in ph}, "tail_rows": st["lower_tail_rows"],
                          "lu_bitwise": ok}))
        f.close()

if __name__ == "__main__":
    main(20000, 1)
    main(20000, 8)
    main(5000, 40)
