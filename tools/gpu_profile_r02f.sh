#!/bin/bash
# GPU box, end of round 2: bench lines with the NVML clock sampler, the c3_batch block and the four-slot scatter;
# launch list of the default command. The dominant kernels are those of r02e (full captures there).
set -x
mkdir -p gpurun_out
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_ref_c5.json 2> gpurun_out/r02f_bench.err
python bench.py --steps 10 --warmup 3 > gpurun_out/r02f_bench_c5.json 2>> gpurun_out/r02f_bench.err; tail -c 300 gpurun_out/r02f_bench.err
python bench.py --steps 10 --warmup 3 --scenarios 32 --no-single --no-cpu-baseline > gpurun_out/r02f_bench_c5x32.json 2>> gpurun_out/r02f_bench.err
B200LU_BENCH_ONE_DEVICE=1 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_2ranks_one_device.json 2>> gpurun_out/r02f_bench.err
python bench.py --workload C3 --steps 10 --warmup 3 > gpurun_out/r02f_bench_c3.json 2>> gpurun_out/r02f_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02f_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/ncu_bench.log
ls -la gpurun_out | grep r02f
