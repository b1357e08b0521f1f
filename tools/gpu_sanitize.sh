#!/bin/bash
O=gpurun_out/sanitize; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for w in factor exact sampler fused; do
    timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_cases.py $w > $O/${tool}_$w.log 2>&1
    echo "rc=$?" >> $O/${tool}_$w.log
  done
done
