#!/bin/bash
O=gpurun_out/tma3; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "conflict_free" -x > $O/cf.log 2>&1; echo "rc=$?" >> $O/cf.log
timeout 300 python tools/tma_bench.py > $O/bench.log 2>&1
SPTK_TMA_EARLY=7 timeout 300 env MODES=6 python tools/tma_bench.py > $O/bench_early7.log 2>&1
