#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "conflict_free" -p no:cacheprovider > gpurun_out/tc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/tc_tests.log
for m in 1 2; do export SPTK_DEBUG=1;
  SPTK_TC=$m timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_tc$m.json 2> gpurun_out/bench_tc$m.err
  echo "rc=$?" >> gpurun_out/bench_tc$m.err
done
timeout 600 python tools/rmse_probe.py hogwild:1 hogwild:2 > gpurun_out/rmse_probe.log 2>&1
