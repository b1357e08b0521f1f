#!/bin/bash
O=gpurun_out/r2s3y; mkdir -p $O
for pr in "0,0,0" "0,-1,0" "-1,-1,-1" "0,-1,-1"; do
  SPTK_PRIO=$pr BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > "$O/prio_$pr.json" 2> "$O/prio_$pr.err"
done
SPTK_SCHED=burst BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/burst.json 2> $O/burst.err
SPTK_SCHED=burst SPTK_TC_CTAS=4 SPTK_SAMPLER_SLOTS=0 BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/burst4.json 2> $O/burst4.err
