#!/bin/bash
O=gpurun_out/r2s3z; mkdir -p $O
for e in 1 3 5 7; do
  SPTK_TMA_EARLY=$e timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/early$e.json 2> $O/early$e.err
done
