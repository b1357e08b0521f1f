#!/bin/bash
# One GPU session for the record: gpu tests, smoke, bench (ours + reference arm),
# launch list, full ncu capture of the factor kernel, stream timeline.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/bench_tl.json 2> gpurun_out/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_launch.out 2>&1
BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -c 1 -o gpurun_out/prof_factor -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
   > gpurun_out/ncu_full.out 2>&1
echo done > gpurun_out/round.done
