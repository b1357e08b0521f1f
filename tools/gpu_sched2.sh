#!/bin/bash
mkdir -p gpurun_out/sched2
O=gpurun_out/sched2
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -x -k "conflict_free" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --steps 10 --warmup 3"
for rep in 1 2; do
timeout 300 $B > $O/base$rep.json 2>/dev/null
SPTK_SCHED=burst SPTK_TC_CTAS=4 timeout 300 $B > $O/burst4_$rep.json 2>/dev/null
SPTK_SCHED=burst timeout 300 $B > $O/burst3_$rep.json 2>/dev/null
done
SPTK_SCHED=burst SPTK_TC_CTAS=4 BENCH_TIMELINE=1 timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 > $O/burst_tl.json 2> $O/burst_tl.err
for r in 8 32; do
timeout 300 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r${r}_base.json 2>/dev/null
SPTK_SCHED=burst SPTK_TC_CTAS=4 timeout 300 python bench.py --rank $r --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r${r}_burst4.json 2>/dev/null
done
SPTK_TC_CTAS=1 timeout 300 python bench.py --rank 32 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r32_ctas1.json 2>/dev/null
SPTK_SCHED=burst timeout 300 python bench.py --rank 64 --alpha-a 0.0003 --no-e2e --no-cpu-baseline --steps 5 --warmup 3 > $O/r64_burst.json 2>/dev/null
