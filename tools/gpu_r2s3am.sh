#!/bin/bash
O=gpurun_out/r2s3am; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_exact.py tests/test_gpu_dsgd_fused.py tests/test_gpu_dist.py tests/test_gpu_train.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BENCH_TIMELINE=1 timeout 300 python bench.py --config cfg1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1.json 2> $O/cfg1.err
timeout 1200 python -m pytest tests/test_gpu_curves.py -q -p no:cacheprovider -s -k "nf99 or o6_100m" > $O/curves.log 2>&1; echo "rc=$?" >> $O/curves.log
for w in 10 12; do timeout 900 python bench.py --config y4 --no-cpu-baseline --no-e2e --steps 5 --workers $w > $O/y4_w$w.json 2> $O/y4_w$w.err; done
for w in 6 10; do timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 --workers $w > $O/o6_w$w.json 2> $O/o6_w$w.err; done
