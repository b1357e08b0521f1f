#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
BENCH_TIMELINE=1 timeout 600 python bench.py --rank 64 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --alpha-a 0.0003 > gpurun_out/j64.json 2> gpurun_out/j64.err
timeout 600 python bench.py --rank 32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j32.json 2> gpurun_out/j32.err
BENCH_TIMELINE=1 timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_launch.out 2>&1
