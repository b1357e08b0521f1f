#!/bin/bash
O=gpurun_out/r2s3c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_kernels.py tests/test_gpu_exact.py tests/test_gpu_dist.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BENCH_TIMELINE=1 timeout 300 python bench.py --config cfg1 --mode exact --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1_exact.json 2> $O/cfg1_exact.err
BENCH_TIMELINE=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers 32 --steps 5 > $O/w32_tl.json 2> $O/w32_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_w32.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workers 32 > $O/ncu_launch32.out 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_tma_kernel -s 3 -c 1 -o $O/v6_nf \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_v6.out 2>&1
