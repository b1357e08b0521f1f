#!/bin/bash
O=gpurun_out/flat6; mkdir -p $O
for s in 0 16 48 148 296; do
  SPTK_SAMPLER_SLOTS=$s timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers 24 > $O/s$s.json 2> $O/s$s.err
done
SPTK_FY_MAIN=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers 24 > $O/main.json 2> $O/main.err
SPTK_EXP_SKIP=psi timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers 24 > $O/skippsi.json 2> $O/skippsi.err
SPTK_EXP_SKIP=perm timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers 24 > $O/skipperm.json 2> $O/skipperm.err
