#!/bin/bash
mkdir -p gpurun_out
for c in 1 4; do
SPTK_TC_CTAS=$c BENCH_PROFILE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_tc -c 1 -o gpurun_out/prof_c$c python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_c$c.out 2>&1
done
