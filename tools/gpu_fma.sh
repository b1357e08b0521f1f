#!/bin/bash
mkdir -p gpurun_out/fma
O=gpurun_out/fma
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "conflict_free" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
timeout 300 $B > $O/base.json 2>/dev/null
SPTK_TC=5 timeout 300 $B > $O/fma3.json 2>/dev/null
SPTK_TC=5 SPTK_TC_CTAS=4 timeout 300 $B > $O/fma4.json 2>/dev/null
SPTK_TC=5 SPTK_TC_CTAS=2 timeout 300 $B > $O/fma2.json 2>/dev/null
SPTK_TC=5 timeout 300 python bench.py --rank 8 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/fma_r8.json 2>/dev/null
SPTK_TC=5 SPTK_TC_CTAS=4 timeout 300 python bench.py --rank 8 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/fma_r8c4.json 2>/dev/null
SPTK_TC=5 BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_ -c 1 -o $O/prof_fma -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
