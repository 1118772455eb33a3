#!/bin/bash
# GPU box: GPU tests, bench line + reference arm + ncu launch list + full captures of the dominant kernels.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 600 gpurun_out/bench_c5.json; tail -5 gpurun_out/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c5.json 2>> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_ref_c5.json
python tools/batch_probe.py C3 64 2 > gpurun_out/probe_c3x64.json 2>> gpurun_out/bench_c5.err; tail -c 900 gpurun_out/probe_c3x64.json


# launch list of the same command (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
# full captures, after warm-up
ncu --set full --clock-control none --import-source on -k regex:bfactor_kernel -s 3 -c 1 -o gpurun_out/prof_bfactor python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_factor.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bfactor_block_kernel -s 3 -c 1 -o gpurun_out/prof_bblock python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single >> gpurun_out/ncu_factor.log 2>&1
tail -3 gpurun_out/ncu_factor.log
ncu --set full --clock-control none --import-source on -k regex:btri_kernel -s 18 -c 3 -o gpurun_out/prof_btri python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_tri.log 2>&1
ls -la gpurun_out
