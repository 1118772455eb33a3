"""Dev tool (GPU box): one banded chain through the default-mode sweeps, for profiling."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from oracle import refbridge as rb
from tests.fixtures import csr_fixture
n, band = int(sys.argv[1]), int(sys.argv[2])
ro, ci, v = [0], [], []
for i in range(n):
    for j in range(max(0, i - band), min(n, i + band + 1)):
        ci.append(j); v.append(4.0 * band if i == j else -1.0)
    ro.append(len(ci))
fx = csr_fixture(rb.RefCsr.from_arrays(n, ro, ci, v), use_scaling=False, use_amd=False)
f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream))
b = torch.ones(n, dtype=torch.float64, device="cuda")
rlu.refactorize(f, fx.matrix())
for _ in range(3):
    x = rlu.solve_system(f, b)
torch.cuda.synchronize()
print("ok", float(x.sum()))
