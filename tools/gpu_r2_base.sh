#!/bin/bash
# Round-2 baseline on a fresh box: gpu tests, bench line, stream timeline, launch list.
O=gpurun_out/r2base; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
echo done > $O/round.done
