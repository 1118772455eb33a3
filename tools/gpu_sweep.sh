#!/bin/bash
# Dev tool (GPU box): tests + probes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/chain_probe.py 2>&1 | tail -8
python tools/gpu_probe.py C1 C2 C3 2>&1 | python tools/probe_summary.py "default"
STRICT=1 python tools/gpu_probe.py C3 2>&1 | python tools/probe_summary.py "strict"
