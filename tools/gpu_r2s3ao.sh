#!/bin/bash
O=gpurun_out/r2s3ao; mkdir -p $O
SPTK_TMA2=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "conflict_free and 32" > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
SPTK_TMA2=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank 32 --steps 5 > $O/j32_tma2.json 2> $O/j32_tma2.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank 32 --steps 5 > $O/j32_tc3.json 2> $O/j32_tc3.err
SPTK_TMA2=1 timeout 900 python -m pytest tests/test_gpu_curves.py -q -p no:cacheprovider -s -k "j32" > $O/curve.log 2>&1; echo "rc=$?" >> $O/curve.log
