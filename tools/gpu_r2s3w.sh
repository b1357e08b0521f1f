#!/bin/bash
O=gpurun_out/r2s3w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_exact.py tests/test_gpu_train.py tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "exact or seq or core or cfg1 or reproduces" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BENCH_TIMELINE=1 timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1.json 2> $O/cfg1.err
BENCH_PROFILE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_cfg1x.csv python bench.py --config cfg1 --mode exact --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_cfg1.out 2>&1
