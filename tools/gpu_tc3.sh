#!/bin/bash
mkdir -p gpurun_out/tc3
O=gpurun_out/tc3
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
timeout 300 $B > $O/base.json 2>/dev/null
SPTK_TC=4 timeout 300 $B > $O/tc4m.json 2>/dev/null
SPTK_TC=4 SPTK_TC_CTAS=3 timeout 300 $B > $O/tc4m_c3.json 2>/dev/null
SPTK_TC=4 SPTK_EXP_SKIP=perm timeout 300 $B > $O/tc4m_noperm.json 2>/dev/null
SPTK_TC=4 SPTK_TC_CTAS=3 SPTK_EXP_SKIP=perm timeout 300 $B > $O/tc4m_c3_noperm.json 2>/dev/null
SPTK_TC=4 SPTK_DEBUG=1 timeout 300 $B --steps 1 > /dev/null 2> $O/dbg.txt
SPTK_TC=4 timeout 600 python bench.py --config y4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/y4_tc4m.json 2>/dev/null
