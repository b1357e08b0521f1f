#!/bin/bash
mkdir -p gpurun_out/diet
O=gpurun_out/diet
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_train.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --warmup 3"
timeout 300 $B --steps 10 > $O/nf.json 2>/dev/null
timeout 300 $B --steps 10 > $O/nf2.json 2>/dev/null
timeout 300 $B --steps 5 --rank 8 > $O/r8.json 2>/dev/null
timeout 300 $B --steps 5 --rank 4 > $O/r4.json 2>/dev/null
timeout 900 $B --steps 5 --config y4 > $O/y4.json 2>/dev/null
SPTK_DEBUG=1 timeout 900 $B --steps 1 --config y4 > /dev/null 2> $O/y4_dbg.err
timeout 1500 $B --steps 3 --config o6 > $O/o6.json 2>/dev/null
