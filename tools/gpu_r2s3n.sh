#!/bin/bash
O=gpurun_out/r2s3n; mkdir -p $O
for w in 24 32 48 64; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers $w --steps 10 > $O/w$w.json 2> $O/w$w.err
done
for sl in 48 148; do
  SPTK_SAMPLER_SLOTS=$sl timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers 32 --steps 10 > $O/w32_s$sl.json 2> $O/w32_s$sl.err
done
