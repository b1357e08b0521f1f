#!/bin/bash
mkdir -p gpurun_out/grid2
O=gpurun_out/grid2
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do
timeout 300 $B > $O/base_$rep.json 2>/dev/null
for g in 520 545 560 575; do SPTK_TC_CTAS=4 SPTK_TC_GRID=$g timeout 300 $B > $O/c4g${g}_$rep.json 2>/dev/null; done
done
for g in 545 560; do SPTK_TC_CTAS=4 SPTK_TC_GRID=$g timeout 300 python bench.py --rank 8 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r8_c4g$g.json 2>/dev/null; done
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "partition" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
