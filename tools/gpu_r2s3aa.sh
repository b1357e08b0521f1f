#!/bin/bash
O=gpurun_out/r2s3aa; mkdir -p $O
for w in 20 24 28; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers $w > $O/w$w.json 2> $O/w$w.err
done
for sl in 8 32; do
  SPTK_SAMPLER_SLOTS=$sl timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/s$sl.json 2> $O/s$sl.err
done
timeout 1500 python -m pytest tests/test_gpu_train.py -q -p no:cacheprovider -k netflix -s > $O/nf_curve.log 2>&1; echo "rc=$?" >> $O/nf_curve.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "conflict_free" > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
