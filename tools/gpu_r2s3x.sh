#!/bin/bash
O=gpurun_out/r2s3x; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_fy_kernel" -s 1 -c 1 -o $O/bfy \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
bash tools/ncu_export.sh $O/bfy.ncu-rep
