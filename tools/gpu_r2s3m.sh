#!/bin/bash
O=gpurun_out/r2s3m; mkdir -p $O
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_cases.py factor > $O/racecheck_factor.log 2>&1; echo "rc=$?" >> $O/racecheck_factor.log
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "conflict_free" > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
for J in 4 8; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank $J --steps 10 > $O/tc_j$J.json 2> $O/tc_j$J.err
  SPTK_FMA_RANKS=$J timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank $J --steps 10 > $O/fma_j$J.json 2> $O/fma_j$J.err
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_ -s 3 -c 1 -o $O/tc_j$J \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --rank $J > $O/ncu_tc_j$J.out 2>&1
  SPTK_FMA_RANKS=$J timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_ -s 3 -c 1 -o $O/fma_j$J \
     python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --rank $J > $O/ncu_fma_j$J.out 2>&1
  bash tools/ncu_export.sh $O/tc_j$J.ncu-rep
  bash tools/ncu_export.sh $O/fma_j$J.ncu-rep
done
SPTK_FMA_RANKS=16 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/fma_j16.json 2> $O/fma_j16.err
