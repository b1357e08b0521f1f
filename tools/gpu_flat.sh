#!/bin/bash
O=gpurun_out/flat; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_sampler.py -q -p no:cacheprovider -k "block_perm" > $O/bp.log 2>&1; echo "rc=$?" >> $O/bp.log
for w in 20 32 48; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 8 --workers $w > $O/w$w.json 2> $O/w$w.err
done
BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --workers 32 > $O/w32_tl.json 2> $O/w32_tl.err
