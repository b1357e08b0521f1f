#!/bin/bash
O=gpurun_out/r2s3ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_facade.py tests/test_gpu_train.py -q -p no:cacheprovider -x -k "eval or predict or rmse or score or cfg1 or reproduces" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_trace.py > $O/trace.log 2>&1
SPTK_EVAL_PIPE=0 timeout 600 python tools/e2e_trace.py > $O/trace_old.log 2>&1
