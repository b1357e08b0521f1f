#!/bin/bash
mkdir -p gpurun_out
for pf in 1 3; do
SPTK_TC_PREFETCH=$pf BENCH_TIMELINE=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 7 --warmup 3 > gpurun_out/pf$pf.json 2> gpurun_out/pf$pf.err
SPTK_TC_PREFETCH=$pf SPTK_EXP_SKIP=perm timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 7 --warmup 3 > gpurun_out/pf${pf}_noperm.json 2> gpurun_out/pf${pf}_noperm.err
done
SPTK_TC_PREFETCH=3 timeout 300 python tools/tc2_stamps.py > gpurun_out/stamps_pf3.txt 2>&1
