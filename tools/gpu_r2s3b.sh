#!/bin/bash
O=gpurun_out/r2s3b; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
BENCH_TIMELINE=1 timeout 300 python bench.py --config cfg1 --mode exact --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1_exact.json 2> $O/cfg1_exact.err
timeout 300 python bench.py --config cfg1 --mode hogwild --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/cfg1_hog.json 2> $O/cfg1_hog.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers 16 > $O/bench_w16.json 2> $O/bench_w16.err
timeout 1200 python -m pytest tests/test_gpu_train.py tests/test_gpu_kernels.py tests/test_gpu_exact.py -q -p no:cacheprovider -x -rxX > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 1500 python -m pytest tests/test_gpu_curves.py -q -p no:cacheprovider -s > $O/curves.log 2>&1; echo "rc=$?" >> $O/curves.log
