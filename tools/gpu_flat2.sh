#!/bin/bash
O=gpurun_out/flat2; mkdir -p $O
for w in 24 32 48; do
  SPTK_FY_MAIN=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 --workers $w > $O/w$w.json 2> $O/w$w.err
done
SPTK_FY_MAIN=1 BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --workers 32 > $O/w32_tl.json 2> $O/w32_tl.err
SPTK_FY_MAIN=1 BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workers 32 > $O/ncu_launch.out 2>&1
