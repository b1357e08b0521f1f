#!/bin/bash
O=gpurun_out/r2s3q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/sampler.log 2>&1; echo "rc=$?" >> $O/sampler.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w24.json 2> $O/w24.err
SPTK_LP_TWO_STAGE=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w24_old.json 2> $O/w24_old.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
timeout 1800 python -m pytest tests/test_gpu_curves.py -q -p no:cacheprovider -s > $O/curves.log 2>&1; echo "rc=$?" >> $O/curves.log
