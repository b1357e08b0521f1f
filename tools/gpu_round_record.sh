#!/bin/bash
# Final round record: full GPU suite + smoke, headline bench (e2e + cpu leg),
# reference arm, timeline, launch list, ncu --set full of the factor kernel, every config's line.
O=gpurun_out/round; mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rxXf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err
BENCH_TIMELINE=1 timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 > $O/bench_tl.json 2> $O/bench_tl.err
BENCH_PROFILE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off \
   --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.out 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_tma_kernel -s 3 -c 1 -o $O/factor_full \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full.out 2>&1
bash tools/ncu_export.sh $O/factor_full.ncu-rep
for J in 4 8 32 64; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank $J --steps 5 > $O/nf_j$J.json 2> $O/nf_j$J.err
done
timeout 900 python bench.py --config y4 --no-cpu-baseline --no-e2e --steps 5 > $O/y4.json 2> $O/y4.err
timeout 900 python bench.py --config cfg1 --no-cpu-baseline --no-e2e --steps 5 > $O/cfg1.json 2> $O/cfg1.err
timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 > $O/o6.json 2> $O/o6.err
for m in 2 4 8; do
  BENCH_DSGD_SIM=$m timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 16 > $O/sim$m.json 2> $O/sim$m.err
done
BENCH_DSGD_SIM=8 timeout 900 python bench.py --config y4 --no-cpu-baseline --no-e2e --steps 6 > $O/sim8_y4.json 2> $O/sim8_y4.err
