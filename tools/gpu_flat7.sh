#!/bin/bash
O=gpurun_out/flat7; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/samp.log 2>&1; echo "rc=$?" >> $O/samp.log
timeout 300 python tools/blockperm_bench.py > $O/bp_time.log 2>&1
for w in 24 32; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers $w > $O/w$w.json 2> $O/w$w.err
done
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workers 32 > $O/ncu_launch.out 2>&1
