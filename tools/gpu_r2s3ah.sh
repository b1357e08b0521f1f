#!/bin/bash
O=gpurun_out/r2s3ah; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_train.py tests/test_gpu_dsgd_fused.py tests/test_gpu_dist.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_trace.py > $O/trace.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
