"""Dev tool (GPU box): phase breakdown of the interleaved scenario-batch path.

    python tools/batch_probe.py C2 256 [reps]
Environment: B200LU_BATCH_VARIANT, B200LU_BATCH_TAIL_WIDTH / B200LU_BATCH_TAIL_MODE (experiments)."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from paper_2306_14337_b200.batch import BatchedFactors
from oracle import refbridge as rb
from oracle import oraclebridge as ob

CFG = {"C1": (6300, 2700), "C2": (39000, 16700), "C3": (166600, 71400)}


def main(name, batch, reps=3, check=2, refine_cap=4):
    n, m = CFG[name]
    t = time.time()
    seqs = [rb.RefSequence(n, m, y_seed=2 + s, num_systems=1) for s in range(batch)]
    ref_sym = rb.RefSymbolic(seqs[0].matrix(0), use_scaling=False, use_amd=True)
    arrays = ref_sym.arrays()
    sym = rlu.SymbolicFactors.from_arrays(arrays)
    vals = np.stack([q.values(0) for q in seqs])
    rhs = np.stack([q.rhs(0) for q in seqs])
    t_fix = time.time() - t
    t = time.time()
    f = BatchedFactors(sym, batch, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream,
                                                     refine_capacity=refine_cap))
    torch.cuda.synchronize()
    t_create = time.time() - t
    info = f.info
    dv, db = torch.from_numpy(vals).cuda(), torch.from_numpy(rhs).cuda()
    f.set_timing(True)
    runs = []
    for r in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        f.refactorize(dv)
        e[1].record()
        x = f.solve_system(db)
        e[2].record()
        xr, outs = f.fgmres_refine(db, x, rlu.RefineConfig(max_iterations=refine_cap))
        e[3].record()
        torch.cuda.synchronize()
        ph = f.phase_times()
        runs.append(dict(refactor_ms=round(e[0].elapsed_time(e[1]), 3), solve_ms=round(e[1].elapsed_time(e[2]), 3),
                         refine_ms=round(e[2].elapsed_time(e[3]), 3),
                         phases={p: round(v[0], 3) for p, v in ph.items()}, launches={p: v[1] for p, v in ph.items()},
                         iters=sorted(set(o.iterations for o in outs))))
    okv = okx = None
    worst = float(f.relative_residual(xr, db).max())
    if check:
        orc = ob.Factors(arrays)
        okv, okx = True, True
        xs = x.cpu().numpy()
        for s in list(range(check)) + [batch - 1]:
            ref, failed = orc.factorize(vals[s])
            okv = okv and bool(np.array_equal(f.values(s), ref))
            okx = okx and bool(np.array_equal(xs[s], orc.solve_system(ref, rhs[s])[0]))
    tot = runs[-1]["refactor_ms"] + runs[-1]["solve_ms"] + runs[-1]["refine_ms"]
    print(json.dumps(dict(name=name, batch=batch, unit=info["unit_scenarios"], blocks=info["blocks"], blocked_rows=info["blocked_rows"],
                          blocked_pairs_frac=round(info["blocked_pairs"] / max(info["update_pairs"], 1), 3),
                          grid=info["factor_grid"], fixture_s=round(t_fix, 1), create_s=round(t_create, 2),
                          device_gb=round(info["device_bytes"] / 1e9, 2), runs=runs, lu_bitwise=okv, x_bitwise=okx,
                          worst_relres_final=worst, ms_per_system=round(tot / batch, 4),
                          systems_per_s=round(1000 * batch / tot, 1))))
    sys.stdout.flush()
    f.close()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3)
