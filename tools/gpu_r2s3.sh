#!/bin/bash
# Session-3 baseline of round 2: gpu tests, smoke, bench lines W=1/16/32, launch list.
O=gpurun_out/r2s3; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_w1.json 2> $O/bench_w1.err
for w in 16 32; do
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --workers $w > $O/bench_w$w.json 2> $O/bench_w$w.err
done
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_w1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches_w16.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --workers 16 > $O/ncu_launch16.out 2>&1
echo done > $O/round.done
