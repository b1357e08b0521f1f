#!/bin/bash
# re-entry sanity: gpu tests, smoke, one bench line, tcgen05 phase stamps
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 300 python tools/tc2_stamps.py > gpurun_out/stamps.txt 2>&1
