#!/bin/bash
mkdir -p gpurun_out/grid
O=gpurun_out/grid
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
timeout 300 $B > $O/base.json 2>/dev/null
for g in 420 400 370 340 296; do SPTK_TC_GRID=$g timeout 300 $B > $O/g$g.json 2>/dev/null; done
for g in 500 560; do SPTK_TC_CTAS=4 SPTK_TC_GRID=$g timeout 300 $B > $O/c4g$g.json 2>/dev/null; done
