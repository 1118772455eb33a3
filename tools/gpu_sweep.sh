#!/bin/bash
# GPU box: full GPU test suite, smoke, then the default bench line and the reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
python __graft_entry__.py smoke 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c5.json 2>> gpurun_out/bench_c5.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_c5.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "ms/system", d["ms_per_system"], "e2e", d["e2e"]["value"], "kkt", d["e2e_kkt_diagonal"]["value"], "plain", d.get("plain_calls"))
print("phases", d["phases_ms_per_step"]); print("roofline", {k: d["roofline"][k] for k in ("achieved","frac","avg_launch_ms")}, d["roofline"]["whole_step"])
print("records", d["records"]); print("cpu", {k: d["cpu_baseline"][k] for k in ("value","cores","sample")})
print("single", d["single_system"]["value"], d["single_system"]["ms_per_step"], d["single_system"]["roofline"]["frac"])
print("clocks", d["clocks"], "launches", d["gpu_launches"])
r=json.loads(open("gpurun_out/bench_ref_c5.json").read().strip().splitlines()[-1])
print("reference arm", r["value"], r["cpu_baseline"]["sample"])
PY
