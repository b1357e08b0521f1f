#!/bin/bash
O=gpurun_out/r2s3ab; mkdir -p $O
for L in 512 1024 2048; do
  SPTK_LP_PRE=$L timeout 300 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x -k choice > $O/choice$L.log 2>&1; echo "rc=$?" >> $O/choice$L.log
  SPTK_LP_PRE=$L BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches$L.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu$L.out 2>&1
done
