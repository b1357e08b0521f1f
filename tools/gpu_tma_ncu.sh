#!/bin/bash
O=gpurun_out/tma_ncu; mkdir -p $O
MODES=6 NNZ=20000000 timeout 900 ncu --set full --import-source on -k regex:factor_tma -s 1 -c 1 -o $O/tma -f python tools/tma_bench.py > $O/ncu.log 2>&1
ncu -i $O/tma.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/tma.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
