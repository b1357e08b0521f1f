#!/bin/bash
O=gpurun_out/r2s3v; mkdir -p $O
BENCH_PROFILE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_cfg1x.csv python bench.py --config cfg1 --mode exact --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_cfg1.out 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"core_exact_sum|factor_dep_kernel|core_exact_terms" -s 6 -c 3 -o $O/cfg1x \
   python bench.py --config cfg1 --mode exact --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_full.out 2>&1
bash tools/ncu_export.sh $O/cfg1x.ncu-rep
