#!/bin/bash
O=gpurun_out/r2s3ap; mkdir -p $O
SPTK_TMA2=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_tma2 -s 3 -c 1 -o $O/tma2 \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --rank 32 > $O/ncu.out 2>&1
bash tools/ncu_export.sh $O/tma2.ncu-rep
