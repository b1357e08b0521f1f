#!/bin/bash
O=gpurun_out/r2s3aj; mkdir -p $O
for J in 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank $J --steps 10 > $O/nf_j$J.json 2> $O/nf_j$J.err
done
timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 > $O/o6.json 2> $O/o6.err
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "conflict_free" > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
