#!/bin/bash
# GPU box: bench line + ncu launch list + one full capture of the dominant kernel.
set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
python bench.py --steps 20 --warmup 3 --workload C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2>> gpurun_out/bench_c3.err; tail -c 1500 gpurun_out/bench_c2.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c3.json 2>> gpurun_out/bench_c3.err; tail -c 1500 gpurun_out/bench_ref_c3.json
# launch list of the same command (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
tail -3 gpurun_out/ncu_bench.log
# full capture of the dominant kernel (factor_kernel), 2 launches after warm-up
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 2 -o gpurun_out/prof_factor python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_factor.log 2>&1
tail -3 gpurun_out/ncu_factor.log
ncu --set full --clock-control none --import-source on -k regex:tri_kernel -s 8 -c 2 -o gpurun_out/prof_tri python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tri.log 2>&1
ls -la gpurun_out
