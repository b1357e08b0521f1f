#!/bin/bash
O=gpurun_out/r2s3h; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_dsgd_fused.py -q -p no:cacheprovider -x > $O/fused.log 2>&1; echo "rc=$?" >> $O/fused.log
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_exact.py tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "exact or seq or core or train or cfg1" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BENCH_TIMELINE=1 timeout 300 python bench.py --config cfg1 --mode exact --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1_exact.json 2> $O/cfg1_exact.err
for m in 4 8; do
BENCH_DSGD_SIM=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/sim$m.json 2> $O/sim$m.err
done
