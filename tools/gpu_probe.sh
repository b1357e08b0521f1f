#!/bin/bash
O=gpurun_out/probe; mkdir -p $O; rm -f $O/tma2.log
for a in 1 2 3; do timeout 60 tools/probe/tma_probe 1 $a >> $O/tma2.log 2>&1; echo "rc=$?" >> $O/tma2.log; done
