"""Dev probe: where does the time of BatchedFactors.solve_system go at C3 x 64 (verdict r01, weak #6)?"""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
n, m, batch = 166600, 71400, 64
seqs = [rb.RefSequence(n, m, y_seed=2 + s, num_systems=1) for s in range(8)]
A = seqs[0].matrix(0); ro, ci, va = A.arrays()
sym = rlu.symbolic_analyze(rlu.CsrMatrix(A.n, A.n, ro, ci, va), rlu.AnalyzeOptions(False, True))
vals = np.stack([seqs[s % 8].values(0) for s in range(batch)]); rhs = np.stack([seqs[s % 8].rhs(0) for s in range(batch)])
f = BatchedFactors(sym, batch, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream, refine_capacity=4))
dv, db = torch.from_numpy(vals).cuda(), torch.from_numpy(rhs).cuda()
f.set_timing(True)
def ev(): e = torch.cuda.Event(enable_timing=True); e.record(); return e
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0 = ev()
    f.refactorize(dv); torch.cuda.synchronize(); t1 = time.perf_counter(); e1 = ev()
    x = f.solve_system(db); torch.cuda.synchronize(); t2 = time.perf_counter(); e2 = ev()
    xr, outs = f.fgmres_refine(db, x, rlu.RefineConfig(max_iterations=4)); torch.cuda.synchronize(); t3 = time.perf_counter(); e3 = ev()
    torch.cuda.synchronize()
    ph = f.phase_times()
    print(json.dumps(dict(run=r, host_ms=[round(1e3 * (b - a), 2) for a, b in ((t0, t1), (t1, t2), (t2, t3))],
                          event_ms=[round(a.elapsed_time(b), 2) for a, b in ((e0, e1), (e1, e2), (e2, e3))],
                          phases={p: round(v[0], 2) for p, v in ph.items()}, tiled=f.info["tiled"])))
f.close()
