#!/bin/bash
O=gpurun_out/r2s3e; mkdir -p $O
BENCH_DSGD_SIM=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/sim2.json 2> $O/sim2.err
SPTK_TC_GRID=148 BENCH_DSGD_SIM=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/sim2_g148.json 2> $O/sim2_g148.err
BENCH_SIM_FUSED=0 BENCH_DSGD_SIM=2 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/sim2_nf.json 2> $O/sim2_nf.err
SPTK_TC_GRID=148 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/w1_g148.json 2> $O/w1_g148.err
BENCH_PROFILE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_cfg1x.csv python bench.py --config cfg1 --mode exact --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_cfg1.out 2>&1
