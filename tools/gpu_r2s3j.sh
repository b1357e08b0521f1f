#!/bin/bash
O=gpurun_out/r2s3j; mkdir -p $O
E=1 timeout 300 python tools/fused_debug2.py > $O/dbg1.log 2>&1
E=2 timeout 300 python tools/fused_debug2.py > $O/dbg2.log 2>&1
