#!/bin/bash
mkdir -p gpurun_out/tc3s
O=gpurun_out/tc3s
B="python bench.py --no-e2e --no-cpu-baseline --warmup 3 --steps 5 --rank 32"
for sl in 0 16 48 96; do SPTK_SAMPLER_SLOTS3=$sl timeout 300 $B > $O/s$sl.json 2>/dev/null; done
