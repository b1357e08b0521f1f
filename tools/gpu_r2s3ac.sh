#!/bin/bash
O=gpurun_out/r2s3ac; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/sampler.log 2>&1; echo "rc=$?" >> $O/sampler.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w24.json 2> $O/w24.err
SPTK_LP_PRE=256 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w24_256.json 2> $O/w24_256.err
SPTK_LP_PRE=256 BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches256.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu256.out 2>&1
