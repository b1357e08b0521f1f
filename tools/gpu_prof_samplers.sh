set -x
O=gpurun_out/samp; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"block_fy_kernel|block_jgen_kernel|lp_runs_kernel" -c 3 -o $O/samp \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu.out 2>&1
bash tools/ncu_export.sh $O/samp.ncu-rep
ls -la $O
