#!/bin/bash
O=gpurun_out/r2s3i; mkdir -p $O
for pe in "1 1" "0 1" "0 0" "1 0"; do set -- $pe
PREFETCH=$1 USE_EPOCH=$2 timeout 120 python tools/fused_debug.py >> $O/dbg.log 2>&1
done
E=1 PREFETCH=1 USE_EPOCH=1 timeout 120 python tools/fused_debug.py >> $O/dbg.log 2>&1
