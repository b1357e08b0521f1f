#!/bin/bash
mkdir -p gpurun_out
for m in 1 2; do
SPTK_TC=$m BENCH_PROFILE=1 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_tc -c 1 -o gpurun_out/prof_tcm$m python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_tc$m.out 2>&1
echo "rc=$?" >> gpurun_out/ncu_tc$m.out
done
