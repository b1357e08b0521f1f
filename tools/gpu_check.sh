#!/bin/bash
O=gpurun_out/check; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rxXf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
