#!/bin/bash
mkdir -p gpurun_out/up
O=gpurun_out/up
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/e2e_phases.py > $O/e2e_phases.txt 2>&1
for t in 4 8 16; do SPTK_H2D_THREADS=$t timeout 300 python -c "
import time,numpy as np,torch
from paper_2204_07104_b200.schedule import upload
a=np.random.default_rng(0).integers(0,1<<30,(99_072_112,3))
for r in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter(); d=upload(a); torch.cuda.synchronize(); t1=time.perf_counter()
    print('threads $t', round(t1-t0,3), 's', round(a.nbytes/(t1-t0)/1e9,1), 'GB/s'); del d
" >> $O/h2d.txt 2>&1; done
nproc >> $O/h2d.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
