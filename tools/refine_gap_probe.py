"""Dev probe: how much of a batched fgmres_refine call is kernel time, and how much the host leaves the GPU idle."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n, m = 39000, 16700
seqs = [rb.RefSequence(n, m, y_seed=2 + s, num_systems=1) for s in range(min(batch, 16))]
A = seqs[0].matrix(0); ro, ci, va = A.arrays()
sym = rlu.symbolic_analyze(rlu.CsrMatrix(A.n, A.n, ro, ci, va), rlu.AnalyzeOptions(False, True))
vals = np.stack([seqs[s % len(seqs)].values(0) for s in range(batch)]); rhs = np.stack([seqs[s % len(seqs)].rhs(0) for s in range(batch)])
f = BatchedFactors(sym, batch, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream, refine_capacity=4))
dv, db = torch.from_numpy(vals).cuda(), torch.from_numpy(rhs).cuda()
f.refactorize(dv)
x = f.solve_system(db)
cfg = rlu.RefineConfig(max_iterations=4)
for timing in (True, False):
    f.set_timing(timing)
    for r in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
        xr, outs = f.fgmres_refine(db, x, cfg)
        e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
        ph = f.phase_times() if timing else {}
        print("timing", timing, "run", r, "host ms %.3f event ms %.3f" % (1e3 * (t1 - t0), e0.elapsed_time(e1)),
              "kernel phases ms %.3f" % sum(v[0] for v in ph.values()) if ph else "")
f.close()
