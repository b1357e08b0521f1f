#!/bin/bash
# quick: factor tests, 2 bench runs, ncu launch times of the factor kernel, stamps
mkdir -p gpurun_out/q
O=gpurun_out/q
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "factor" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 ${BENCH_ARGS}"
for rep in 1 2; do timeout 300 $B > $O/b$rep.json 2>/dev/null; done
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:factor_t \
   --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > $O/ncu.out 2>&1
timeout 300 python tools/tc2_stamps.py > $O/stamps.txt 2>&1
