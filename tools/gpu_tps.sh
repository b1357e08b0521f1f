#!/bin/bash
mkdir -p gpurun_out/tps
O=gpurun_out/tps
SPTK_TC=0 timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 > $O/b.json 2>/dev/null
SPTK_TC=0 BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -c 1 -o $O/prof_tps -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
