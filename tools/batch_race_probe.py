"""Dev tool (GPU box): run-to-run determinism and oracle agreement of the batched refactorization over
many scenarios (looks for timing-dependent races)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
from oracle import oraclebridge as ob

n, m, B = 39000, 16700, 256
seqs = [rb.RefSequence(n, m, y_seed=2 + s, num_systems=1) for s in range(B)]
sym_ref = rb.RefSymbolic(seqs[0].matrix(0), use_scaling=False, use_amd=True)
arrays = sym_ref.arrays()
sym = rlu.SymbolicFactors.from_arrays(arrays)
vals = np.stack([q.values(0) for q in seqs])
f = BatchedFactors(sym, B, rlu.FactorOptions(refine_capacity=2))
dv = torch.from_numpy(vals).cuda()
sample = list(range(0, B, 5))
base = None
bad = 0
for run in range(4):
    f.refactorize(dv)
    cur = {s: f.values(s) for s in sample}
    if base is None:
        base = cur
    else:
        for s in sample:
            if not np.array_equal(cur[s], base[s]):
                bad += 1
                d = np.nonzero(cur[s] != base[s])[0]
                print("run", run, "scenario", s, "differs at", d.size, "slots, first", d[:5])
orc = ob.Factors(arrays)
wrong = []
for s in sample[::4]:
    ref, failed = orc.factorize(vals[s])
    if not np.array_equal(base[s], ref):
        d = np.nonzero(base[s] != ref)[0]
        rows = np.searchsorted(arrays.row_offsets, d[:8], side="right") - 1
        wrong.append((s, int(d.size), rows.tolist()))
print(json.dumps({"unit": f.info["unit_scenarios"], "nondeterministic": bad, "wrong_vs_oracle": wrong}))
