#!/bin/bash
mkdir -p gpurun_out/evtc
O=gpurun_out/evtc
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
