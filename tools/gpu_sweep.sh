#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err; tail -3 gpurun_out/bench_batch.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_batch.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms/step", d["ms_per_step"], "e2e", d["e2e"]["value"])
print("batch", json.dumps(d.get("batch"))[:900])
print("clocks", d["clocks"])
PY
for sidx in 2 4 16; do
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --streams $sidx 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); b=d['batch']; print('streams', b['streams_per_gpu'], 'batch systems/s', round(b['value'],1), 'ms/system', round(b['ms_per_system'],3))"
done
