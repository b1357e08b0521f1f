#!/bin/bash
mkdir -p gpurun_out/slots3
O=gpurun_out/slots3
B="python bench.py --no-e2e --no-cpu-baseline --warmup 3"
for sl in 48 96; do
SPTK_SAMPLER_SLOTS=$sl timeout 300 $B --steps 5 --rank 8 > $O/r8_s$sl.json 2>/dev/null
SPTK_SAMPLER_SLOTS=$sl timeout 900 $B --steps 5 --config y4 > $O/y4_s$sl.json 2>/dev/null
done
for sl in 8 32; do SPTK_SAMPLER_SLOTS=$sl timeout 300 $B --steps 10 > $O/nf_s$sl.json 2>/dev/null; done
