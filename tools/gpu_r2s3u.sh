#!/bin/bash
O=gpurun_out/r2s3u; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rxXf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
