"""Dev tool (GPU box): phase breakdown of refactorize + solve + FGMRES on generated KKT systems."""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2306_14337_b200 as rlu
from tests.fixtures import kkt_fixture

def run(name, n, m, reps=5, check=True):
    t = time.time()
    fx = kkt_fixture(n, m, num_systems=3)
    t_fix = time.time() - t
    t = time.time()
    f = rlu.NumericFactors(fx.sym, rlu.FactorOptions(stream=torch.cuda.current_stream().cuda_stream, strict_order=bool(int(os.environ.get('STRICT', '0')))))
    torch.cuda.synchronize()
    t_create = time.time() - t
    st = f.stats
    dvals = [torch.from_numpy(v).cuda() for v in fx.values]
    drhs = [torch.from_numpy(b).cuda() for b in fx.rhs]
    f.set_timing(True)
    res = []
    for r in range(reps):
        k = r % len(dvals)
        A = rlu.CsrMatrix(fx.n, fx.n, fx.ro, fx.ci, dvals[k])
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        rlu.refactorize(f, A)
        e[1].record()
        x = rlu.solve_system(f, drhs[k])
        e[2].record()
        out = rlu.fgmres_refine(f, drhs[k], x)
        e[3].record()
        torch.cuda.synchronize()
        ph = f.phase_times()
        res.append(dict(refactor_ms=e[0].elapsed_time(e[1]), solve_ms=e[1].elapsed_time(e[2]),
                        refine_ms=e[2].elapsed_time(e[3]), iters=out.iterations,
                        phases={p: round(v[0], 4) for p, v in ph.items()}, launches={p: v[1] for p, v in ph.items()}))
        if check and r < len(dvals):
            lu = f.values
            ref, failed = fx.oracle.factorize(fx.values[k])
            okv = bool(np.array_equal(lu, ref))
            xo = fx.oracle.solve_system(ref, fx.rhs[k])[0]
            okx = bool(np.array_equal(x.cpu().numpy(), xo)) if f.options.strict_order else float(fx.oracle_csr(k).relative_residual(x.cpu().numpy(), fx.rhs[k]))
            rr = fx.oracle_csr(k).relative_residual(out.x.cpu().numpy(), fx.rhs[k])
            res[-1].update(lu_bitwise=okv, x_bitwise=okx, relres_final=rr)
    print(json.dumps(dict(name=name, fixture_s=round(t_fix, 2), create_s=round(t_create, 3), stats=st, runs=res), indent=None))
    sys.stdout.flush()
    f.close()

if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C2", "C3"]
    cfg = {"C1": (6300, 2700), "C2": (39000, 16700), "C3": (166600, 71400), "C4": (1120000, 480000)}
    for w in which:
        run(w, *cfg[w], check=(w != "C4"))
