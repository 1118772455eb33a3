#!/bin/bash
# GPU box, round 2: bench lines (default C5 x 256, the 32-scenario shard of the 8-GPU configuration, the reference
# arm), ncu launch lists of the same commands, full captures of the dominant kernels. Everything lands in gpurun_out/.
set -x
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/r02e_bench_c5.json 2> gpurun_out/r02e_bench_c5.err; tail -c 300 gpurun_out/r02e_bench_c5.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02e_bench_ref_c5.json 2>> gpurun_out/r02e_bench_c5.err
python bench.py --steps 10 --warmup 3 --scenarios 32 --no-single --no-cpu-baseline > gpurun_out/r02e_bench_c5x32.json 2>> gpurun_out/r02e_bench_c5.err
B200LU_BENCH_ONE_DEVICE=1 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_2ranks_one_device.json 2>> gpurun_out/r02e_bench_c5.err
# launch lists (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02e_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02e_launches_c5x32.csv python bench.py --steps 2 --warmup 3 --scenarios 32 --no-cpu-baseline --no-single > gpurun_out/ncu_bench32.log 2>&1
# full captures, after warm-up
ncu --set full --clock-control none --import-source on -k regex:bfactor_block_team_kernel -s 3 -c 1 -f -o gpurun_out/r02e_prof_bblock python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_factor.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bfactor_kernel -s 3 -c 1 -f -o gpurun_out/r02e_prof_bhead python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single >> gpurun_out/ncu_factor.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bfactor_tile_kernel -s 3 -c 1 -f -o gpurun_out/r02e_prof_btile python bench.py --steps 2 --warmup 3 --scenarios 32 --no-cpu-baseline --no-single >> gpurun_out/ncu_factor.log 2>&1
tail -3 gpurun_out/ncu_factor.log
ls -la gpurun_out | tail -20
# single system C3 (the north star's named config) and C4
python bench.py --workload C3 --steps 10 --warmup 3 > gpurun_out/r02e_bench_c3.json 2>> gpurun_out/r02e_bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02e_launches_c3.csv python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:factor_kernel -s 3 -c 1 -f -o gpurun_out/r02e_prof_factor_c3 python bench.py --workload C3 --steps 2 --warmup 3 --no-cpu-baseline >> gpurun_out/ncu_factor.log 2>&1
# the two experimental trailing forms, for the record (C2 x 256)
ls -la gpurun_out | tail -30
ncu --set full --clock-control none --import-source on -k regex:btri_upper_team_kernel -s 6 -c 1 -f -o gpurun_out/r02e_prof_utri python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/ncu_utri.log 2>&1
