#!/bin/bash
mkdir -p gpurun_out/sched
O=gpurun_out/sched
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do
timeout 300 $B > $O/base$rep.json 2>/dev/null
SPTK_TC_CTAS=4 SPTK_FY_MAIN=1 timeout 300 $B > $O/c4m1_$rep.json 2>/dev/null
SPTK_FY_MAIN=1 timeout 300 $B > $O/c3m1_$rep.json 2>/dev/null
SPTK_TC_CTAS=4 timeout 300 $B > $O/c4m0_$rep.json 2>/dev/null
done
SPTK_TC_CTAS=4 SPTK_FY_MAIN=1 BENCH_TIMELINE=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 > $O/c4m1_tl.json 2> $O/c4m1_tl.err
for r in 8 32; do
timeout 300 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r${r}_base.json 2>/dev/null
SPTK_TC_CTAS=4 SPTK_FY_MAIN=1 timeout 300 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r${r}_c4m1.json 2>/dev/null
SPTK_FY_MAIN=1 timeout 300 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r${r}_m1.json 2>/dev/null
done
