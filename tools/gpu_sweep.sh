#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python tools/chain_probe.py 2>&1 | grep -v '"strict": true' | tail -3 | cut -c1-200
python tools/gpu_probe.py C1 C2 C3 2>&1 | python tools/probe_summary.py "default"
STRICT=1 python tools/gpu_probe.py C3 2>&1 | python tools/probe_summary.py "strict"
python tools/gpu_probe.py C4 2>&1 | python tools/probe_summary.py "C4"
