#!/bin/bash
# full ncu capture (source-level stall sampling) of the factor kernel on the bench workload
mkdir -p gpurun_out
BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -c 1 -o gpurun_out/prof_factor -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_full.out 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.out
