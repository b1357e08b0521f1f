#!/bin/bash
O=gpurun_out/samp_ncu; mkdir -p $O
BENCH_PROFILE=1 timeout 1500 ncu --set full --clock-control none --profile-from-start off \
  -k regex:"fy_target|fy_emit|msd_pass1|msd_pass2|msd_count|perm_phaseA|perm_phaseB|lp_exit|perm_resolve" -c 12 \
  -o $O/samp -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/samp.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
