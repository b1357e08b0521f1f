#!/bin/bash
O=gpurun_out/r2s3an; mkdir -p $O
timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 > $O/o6.json 2> $O/o6.err
SPTK_LIB=libsptk_v.so timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 > $O/o6_v.json 2> $O/o6_v.err
