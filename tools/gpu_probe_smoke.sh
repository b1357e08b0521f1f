#!/bin/bash
O=gpurun_out/probe1; mkdir -p $O
for tc in 6 1; do for g in 0 148 37 8; do
  if [ $g = 0 ]; then unset SPTK_TC_GRID; else export SPTK_TC_GRID=$g; fi
  SPTK_TC=$tc timeout 120 python tools/smoke_probe.py >> $O/probe.log 2>&1
done; done
unset SPTK_TC_GRID
DIMS=30000,12000,3000 timeout 120 python tools/smoke_probe.py >> $O/probe.log 2>&1
DIMS=48000,1777,2182 timeout 120 python tools/smoke_probe.py >> $O/probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exact.py -q -p no:cacheprovider -x > $O/exact.log 2>&1; echo "rc=$?" >> $O/exact.log
python bench.py --config cfg1 --mode exact --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1_exact.json 2> $O/cfg1_exact.err
