#!/bin/bash
O=gpurun_out/flat3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -x > $O/samp.log 2>&1; echo "rc=$?" >> $O/samp.log
timeout 300 python tools/blockperm_bench.py > $O/bp_time.log 2>&1
for w in 24 32; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 --workers $w > $O/w$w.json 2> $O/w$w.err
  SPTK_FY_MAIN=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 --workers $w > $O/w${w}m.json 2> $O/w${w}m.err
done
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 > $O/w1.json 2> $O/w1.err
BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --workers 32 > $O/w32_tl.json 2> $O/w32_tl.err
