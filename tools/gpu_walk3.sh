#!/bin/bash
mkdir -p gpurun_out/w3
O=gpurun_out/w3
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -k regex:lp_ \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
for rep in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3 > $O/b$rep.json 2>/dev/null; done
