"""Dev tool (GPU box): per-level hand-off cost of the batched refactorization / sweeps on a pure
dependency chain (banded matrix in natural order: n levels of width 1, `band` entries per row)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
from tests.fixtures import csr_fixture


def main(n, band, batch):
    ro, ci, v = [0], [], []
    for i in range(n):
        for j in range(max(0, i - band), min(n, i + band + 1)):
            ci.append(j); v.append(4.0 * band if i == j else -1.0)
        ro.append(len(ci))
    A = rb.RefCsr.from_arrays(n, ro, ci, v)
    fx = csr_fixture(A, use_scaling=False, use_amd=False)
    f = BatchedFactors(fx.sym, batch, rlu.FactorOptions(refine_capacity=2))
    vals = torch.from_numpy(np.stack([fx.values[0]] * batch)).cuda()
    b = torch.ones((batch, n), dtype=torch.float64, device="cuda")
    f.set_timing(True)
    for _ in range(3):
        f.refactorize(vals); x = f.solve_system(b)
    f.phase_times()
    reps = 3
    for _ in range(reps):
        f.refactorize(vals); x = f.solve_system(b)
    ph = f.phase_times()
    ok = bool(np.array_equal(f.values(batch - 1), fx.oracle.factorize(fx.values[0])[0]))
    print(json.dumps({"n": n, "band": band, "batch": batch, "unit": f.info["unit_scenarios"],
                      "us_per_level": {p: round(1e3 * ph[p][0] / reps / n, 2) for p in ("factor", "lower", "upper")}, "bitwise": ok}))
    f.close()


if __name__ == "__main__":
    for band, batch in ((1, 32), (1, 256), (40, 32), (40, 256), (80, 256)):
        main(4000, band, batch)
