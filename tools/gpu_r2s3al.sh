#!/bin/bash
O=gpurun_out/r2s3al; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dsgd_fused.py tests/test_gpu_train.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/ring_$i.json 2> $O/ring_$i.err
  SPTK_LIB=libsptk_minb5.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/minb5_$i.json 2> $O/minb5_$i.err
done
SPTK_LIB=libsptk_minb5.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k conflict_free > $O/cf5.log 2>&1; echo "rc=$?" >> $O/cf5.log
