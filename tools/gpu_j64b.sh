#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "uniform_ranks or (conflict_free and 64)" > gpurun_out/pytest_j64.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_j64.log
for a in 0.001 0.0003 0.0001; do
BENCH_TIMELINE=1 timeout 600 python bench.py --rank 64 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --alpha-a $a > gpurun_out/j64_a$a.json 2> gpurun_out/j64_a$a.err
done
timeout 600 python bench.py --rank 32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j32.json 2> gpurun_out/j32.err
