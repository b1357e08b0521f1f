#!/bin/bash
mkdir -p gpurun_out/prio
O=gpurun_out/prio
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "64" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do
timeout 300 $B > $O/base$rep.json 2>/dev/null
SPTK_LEMIRE_SERIAL=1 timeout 300 $B > $O/serial$rep.json 2>/dev/null
SPTK_PRIO=0,-1,0 timeout 300 $B > $O/prioA$rep.json 2>/dev/null
SPTK_PRIO=-1,-1,0 timeout 300 $B > $O/prioB$rep.json 2>/dev/null
SPTK_PRIO=0,-1,0 SPTK_LEMIRE_SERIAL=1 timeout 300 $B > $O/prioAs$rep.json 2>/dev/null
done
timeout 600 python bench.py --rank 64 --alpha-a 0.0003 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/rank64.json 2> $O/rank64.err
