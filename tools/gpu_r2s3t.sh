#!/bin/bash
O=gpurun_out/r2s3t; mkdir -p $O
for w in 16 24; do
timeout 900 python bench.py --config y4 --no-cpu-baseline --no-e2e --steps 5 --workers $w > $O/y4_w$w.json 2> $O/y4_w$w.err
done
for w in 8; do
timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 --workers $w > $O/o6_w$w.json 2> $O/o6_w$w.err
done
