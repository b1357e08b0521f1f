#!/bin/bash
# factor time on 20M NF-shaped samples + RMSE vs reference on nf8m, per configuration
mkdir -p gpurun_out
out=gpurun_out/explore.log; : > $out
for tc in 1 2; do for mask in 0 6; do for ctas in 1 2 4; do
  echo "=== tc=$tc mask=$mask ctas=$ctas" >> $out
  SPTK_TC=$tc SPTK_ATOMIC_MASK=$mask SPTK_TC_CTAS=$ctas timeout 120 python tools/hot_probe1.py >> $out 2>&1
  SPTK_TC=$tc SPTK_ATOMIC_MASK=$mask SPTK_TC_CTAS=$ctas timeout 120 python tools/rmse_probe.py hogwild:$tc 2>&1 | cut -c1-200 >> $out
done; done; done
