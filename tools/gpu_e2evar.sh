#!/bin/bash
mkdir -p gpurun_out/e2evar
O=gpurun_out/e2evar
for rep in 1 2 3; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b$rep.json 2>/dev/null; done
timeout 600 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
free -g > $O/free.txt; nproc >> $O/free.txt; cat /proc/loadavg >> $O/free.txt
