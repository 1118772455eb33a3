#!/bin/bash
# Dev tool (GPU box): tests + probes.
mkdir -p gpurun_out
python -m pytest tests/test_cpp_shim.py -q 2>&1 | tail -3
./tests/cpp/test_shim
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
python tools/gpu_probe.py C3 2>&1 | python tools/probe_summary.py "default"
