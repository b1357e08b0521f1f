#!/bin/bash
# sampler-stage contention experiments (SPTK_EXP_SKIP) + J=64 convergence check
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --steps 6 --warmup 3"
for sk in none psi jseq perm psi,jseq psi,jseq,perm; do
  SPTK_EXP_SKIP=$sk BENCH_TIMELINE=1 timeout 300 $B > gpurun_out/exp_$sk.json 2> gpurun_out/exp_$sk.err
done
for c in 2 4; do SPTK_TC_CTAS=$c timeout 300 $B > gpurun_out/exp_ctas$c.json 2> gpurun_out/exp_ctas$c.err; done
SPTK_TC=0 timeout 300 python bench.py --rank 64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j64_wps.json 2>&1
timeout 300 python bench.py --rank 64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j64_tc4.json 2>&1
timeout 300 python bench.py --rank 64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --alpha-a 0.0003 > gpurun_out/j64_tc4_a3.json 2>&1
BENCH_TIMELINE=1 timeout 300 python bench.py --rank 64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j64_tl.json 2> gpurun_out/j64_tl.err
