# block-permutation change check: sampler parity tests, the block-permutation timing, NF bench
O=gpurun_out/fy; mkdir -p $O
python -m pytest tests/test_gpu_sampler.py tests/test_gpu_train.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
M=20 NB=12384 python tools/blockperm_bench.py > $O/bp.log 2>&1
python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err
BENCH_TIMELINE=1 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_tl.json 2> $O/bench_tl.err
tail -3 $O/pytest.log; cat $O/bp.log; cat $O/bench.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["test_rmse"], d["roofline"]["kernel_ms"])'; grep timeline $O/bench_tl.err | tail -2
