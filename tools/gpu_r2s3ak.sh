#!/bin/bash
O=gpurun_out/r2s3ak; mkdir -p $O
for w in 12 16 18 20; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers $w > $O/w$w.json 2> $O/w$w.err
done
