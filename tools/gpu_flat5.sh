#!/bin/bash
O=gpurun_out/flat5; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x -k "block_perm" > $O/samp.log 2>&1; echo "rc=$?" >> $O/samp.log
timeout 300 python tools/blockperm_bench.py > $O/bp_time.log 2>&1
NB=7200 M=24 timeout 300 python tools/blockperm_bench.py > $O/bp_time24.log 2>&1
for w in 16 24 32; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 --workers $w > $O/w$w.json 2> $O/w$w.err
done
BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --workers 24 > $O/w24_tl.json 2> $O/w24_tl.err
