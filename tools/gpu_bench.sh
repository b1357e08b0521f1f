#!/bin/bash
# One GPU session: tests, bench line, launch list, full ncu capture of the factor kernel.
set -x
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK > gpurun_out/clocks_before.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} \
   > gpurun_out/ncu_launch.out 2>&1
echo "ncu launches rc=$?" >> gpurun_out/bench.err
BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -c 1 -o gpurun_out/prof_factor python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} \
   > gpurun_out/ncu_full.out 2>&1
echo "ncu full rc=$?" >> gpurun_out/bench.err
