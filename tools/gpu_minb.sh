#!/bin/bash
O=gpurun_out/minb; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "conflict_free" -x > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
MODES=6 timeout 300 python tools/tma_bench.py > $O/bench5.log 2>&1
SPTK_TC_CTAS=4 MODES=6 timeout 300 python tools/tma_bench.py > $O/bench4.log 2>&1
for w in 32; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers $w > $O/w$w.json 2> $O/w$w.err
  SPTK_SAMPLER_SLOTS=148 timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --workers $w > $O/w${w}s148.json 2> $O/w${w}s148.err
done
