#!/bin/bash
mkdir -p gpurun_out/fe
O=gpurun_out/fe
timeout 600 python -m pytest tests/test_gpu_sampler.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2 3; do timeout 300 $B > $O/b$rep.json 2>/dev/null; done
