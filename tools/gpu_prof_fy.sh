#!/bin/bash
mkdir -p gpurun_out
BENCH_PROFILE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"fy_" -c 2 -o gpurun_out/prof_fy -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_fy.out 2>&1
