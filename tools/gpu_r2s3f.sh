#!/bin/bash
# Hogwild contention at the per-rank block shape of 8-GPU DSGD (NF mode 2: 2182/8 = 272 rows)
O=gpurun_out/r2s3f; mkdir -p $O
for d in 480189,17770,2182 480189,17770,1091 480189,17770,272; do
  DIMS=$d NNZ=20000000 EPOCHS=3 timeout 300 python tools/smoke_probe.py >> $O/probe.log 2>&1
  SPTK_TC_GRID=72 DIMS=$d NNZ=20000000 EPOCHS=3 timeout 300 python tools/smoke_probe.py >> $O/probe.log 2>&1
done
