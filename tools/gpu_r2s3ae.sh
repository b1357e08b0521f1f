#!/bin/bash
O=gpurun_out/r2s3ae; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_fy_kernel|block_jgen_kernel" -s 2 -c 2 -o $O/bfy \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
ncu -i $O/bfy.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > $O/bfy.cuda.csv.gz
bash tools/ncu_export.sh $O/bfy.ncu-rep
