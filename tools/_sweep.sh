python __graft_entry__.py smoke 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-single > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -3 gpurun_out/bench_c5.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_c5.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "kkt", d["e2e_kkt_diagonal"]["value"], d["e2e_kkt_diagonal"]["ms_per_step"], d["e2e_kkt_diagonal"]["bitwise_equal_to_full_value_submission"])
print("phases", d["phases_ms_per_step"])
PY
