#!/bin/bash
O=gpurun_out/r2s3o; mkdir -p $O
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" > $O/props.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers 24 --steps 10 > $O/w24.json 2> $O/w24.err
SPTK_L2_PERSIST=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --workers 24 --steps 10 > $O/w24_l2.json 2> $O/w24_l2.err
SPTK_L2_PERSIST=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/w1_l2.json 2> $O/w1_l2.err
SPTK_L2_PERSIST=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:factor_tma -s 3 -c 2 \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --workers 24 > $O/ncu_l2.out 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:factor_tma -s 3 -c 2 \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --workers 24 > $O/ncu_base.out 2>&1
