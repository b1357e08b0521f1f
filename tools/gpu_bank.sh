#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_train.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
BENCH_TIMELINE=1 timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 7 --warmup 3 > gpurun_out/bank.json 2> gpurun_out/bank.err
SPTK_EXP_SKIP=perm timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 7 --warmup 3 > gpurun_out/bank_noperm.json 2> gpurun_out/bank_noperm.err
for r in 8 32 64; do timeout 600 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bank_r$r.json 2> gpurun_out/bank_r$r.err; done
timeout 300 python tools/tc2_stamps.py > gpurun_out/stamps.txt 2>&1
