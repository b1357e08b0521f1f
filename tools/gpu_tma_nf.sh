#!/bin/bash
O=gpurun_out/tma_nf; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_train.py -q -p no:cacheprovider -k "netflix" -s > $O/nf_rmse.log 2>&1; echo "rc=$?" >> $O/nf_rmse.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
SPTK_TMA_EARLY=7 timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench_e7.json 2> $O/bench_e7.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
