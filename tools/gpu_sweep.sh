#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python tools/chain_probe.py 2>&1 | grep -v '"strict": true' | tail -3 | cut -c1-120
python tools/gpu_probe.py C2 C3 2>&1 | python tools/probe_summary.py "default"
B200LU_FACTOR_SPLIT=1 python tools/gpu_probe.py C3 2>&1 | python tools/probe_summary.py "factor split"
