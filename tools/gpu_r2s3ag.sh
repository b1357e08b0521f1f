#!/bin/bash
# round record: headline bench (e2e + cpu leg), reference arm, timeline, launch list, ncu of the factor kernel
O=gpurun_out/r2s3ag; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_tma_kernel -s 3 -c 1 -o $O/factor_full \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.out 2>&1
bash tools/ncu_export.sh $O/factor_full.ncu-rep
