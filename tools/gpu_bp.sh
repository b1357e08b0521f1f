#!/bin/bash
O=gpurun_out/bp3; mkdir -p $O
timeout 600 ncu --set full --import-source on -k regex:block_ -s 2 -c 2 -o $O/bp -f python tools/blockperm_bench.py > $O/ncu.log 2>&1
ncu -i $O/bp.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/bp.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
