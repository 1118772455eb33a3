"""Dev tool: condenses tools/gpu_probe.py JSON lines to one line per config."""
import json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        if line:
            print("#", line[:300])
        continue
    d = json.loads(line)
    runs = d["runs"]
    last = runs[-1]
    ok = [(r.get("lu_bitwise"), r.get("x_bitwise")) for r in runs if "lu_bitwise" in r]
    med = lambda key: sorted(r[key] for r in runs)[len(runs) // 2]
    ph = {p: round(sorted(r["phases"][p] for r in runs)[len(runs) // 2], 3) for p in last["phases"]}
    print(f"[{tag}] {d['name']}: refactor {med('refactor_ms'):.3f} ms, solve {med('solve_ms'):.3f} ms, refine {med('refine_ms'):.3f} ms"
          f" | kernels {ph} | parity {ok} relres {[r.get('relres_final') for r in runs if 'relres_final' in r][:1]}")
