#!/bin/bash
mkdir -p gpurun_out/ev
O=gpurun_out/ev
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "eval or predict or train or smoke or estimator" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
