#!/bin/bash
# full ncu of the factor kernel + alternative-kernel timings
mkdir -p gpurun_out
BENCH_PROFILE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -s 1 -c 1 -o gpurun_out/prof_factor -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_full.out 2>&1
for tc in 0 2; do
  SPTK_TC=$tc timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_tc$tc.json 2>&1
done
