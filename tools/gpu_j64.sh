#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "conflict_free and 64" > gpurun_out/pytest_j64.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_j64.log
timeout 600 python bench.py --rank 64 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_j64.json 2> gpurun_out/bench_j64.err
echo "bench rc=$?" >> gpurun_out/bench_j64.err
