"""Dev tool (GPU box): times the batched refactorization alone (results are not checked: used with
experiment builds that compute garbage)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
n, m = (39000, 16700) if sys.argv[1] == "C2" else (166600, 71400)
batch = int(sys.argv[2])
seqs = [rb.RefSequence(n, m, y_seed=2 + s, num_systems=1) for s in range(min(batch, 32))]
sym = rlu.SymbolicFactors.from_arrays(rb.RefSymbolic(seqs[0].matrix(0), use_scaling=False, use_amd=True).arrays())
vals = np.stack([seqs[s % len(seqs)].values(0) for s in range(batch)])
f = BatchedFactors(sym, batch, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream, refine_capacity=2))
dv = torch.from_numpy(vals).cuda()
f.set_timing(True)
import ctypes as C
from paper_2306_14337_b200 import _capi
NAMES = ["(barrier issue)", "tile-end wait + claim", "row load", "records/shuffles/prefetch", "wait row of tile", "wait producer", "wait copy",
         "alpha", "updates", "publish+writeback", "prod: bookkeeping", "prod: wait ring space", "prod: wait flag",
         "prod: fence+issue", "-", "consumer setup"]
for r in range(3):
    f.refactorize(dv, raise_on_zero_pivot=False)
    torch.cuda.synchronize()
    print("factor ms", round(f.phase_times()["factor"][0], 3), "tiled", f.info["tiled"])
    cyc = (C.c_int64 * 16)()
    _capi.lib().b200lu_batch_tile_profile(f._h, cyc, 1)
    tot = sum(cyc) or 1
    if r == 2 and tot > 1:
        for nm, c in zip(NAMES, cyc):
            if c:
                print(f"  {nm:28s} {c / 1e9:9.3f} Gcyc  {100 * c / tot:5.1f} %")
f.close()
