#!/bin/bash
O=gpurun_out/r2s3ad; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/sampler.log 2>&1; echo "rc=$?" >> $O/sampler.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w24_$i.json 2> $O/w24_$i.err; done
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
