#!/bin/bash
O=gpurun_out/r2s3l; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/sampler.log 2>&1; echo "rc=$?" >> $O/sampler.log
for w in 16 32; do
BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers $w --steps 10 > $O/w$w.json 2> $O/w$w.err
done
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_w16.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workers 16 > $O/ncu_launch16.out 2>&1
