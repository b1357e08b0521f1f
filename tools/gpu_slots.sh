#!/bin/bash
mkdir -p gpurun_out/slots
O=gpurun_out/slots
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --no-e2e --no-cpu-baseline --warmup 3"
for sl in 16 8 24; do SPTK_SAMPLER_SLOTS=$sl timeout 300 $B --steps 10 > $O/nf_s$sl.json 2>/dev/null; done
timeout 300 $B --steps 10 > $O/nf_default.json 2>/dev/null
SPTK_DEBUG=1 timeout 300 $B --steps 1 > /dev/null 2> $O/dbg.err
for r in 4 8; do timeout 300 $B --steps 5 --rank $r > $O/r$r.json 2>/dev/null; done
timeout 900 $B --steps 5 --config y4 > $O/y4.json 2>/dev/null
timeout 1500 $B --steps 3 --config o6 > $O/o6.json 2>/dev/null
