#!/bin/bash
# Round record: gpu tests, smoke, bench (ours + reference arm), timeline, launch list,
# full ncu capture of the factor kernel, rank sweep, Y4 / O6 / cfg1 lines, per-rank DSGD estimates.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
BENCH_PROFILE=1 timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:factor_t -c 1 -o $O/prof_factor -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_full.out 2>&1
for r in 4 8 32 64; do
  a=""; [ $r = 64 ] && a="--alpha-a 0.0003"
  timeout 600 python bench.py --rank $r $a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/rank$r.json 2> $O/rank$r.err
done
timeout 900 python bench.py --config y4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/y4.json 2> $O/y4.err
timeout 900 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > $O/cfg1.json 2> $O/cfg1.err
timeout 1500 python bench.py --config o6 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/o6.json 2> $O/o6.err
for m in 2 4 8; do BENCH_DSGD_SIM=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/dsgd$m.json 2> $O/dsgd$m.err; done
echo done > $O/round.done
