#!/bin/bash
O=gpurun_out/r2s3s; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_fy_kernel|block_jgen_kernel|lp_exit_kernel" -s 3 -c 3 -o $O/samplers \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
bash tools/ncu_export.sh $O/samplers.ncu-rep
