#!/bin/bash
O=gpurun_out/slots6; mkdir -p $O
for s in 16 48 148 296; do
  SPTK_SAMPLER_SLOTS=$s timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 8 > $O/s$s.json 2> $O/s$s.err
done
SPTK_SCHED=burst timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 8 > $O/burst.json 2> $O/burst.err
for x in psi jseq perm psi,jseq,perm; do SPTK_EXP_SKIP=$x timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 8 > $O/skip$x.json 2> $O/skip$x.err; done
