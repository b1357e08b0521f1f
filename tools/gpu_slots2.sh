#!/bin/bash
mkdir -p gpurun_out/slots2
O=gpurun_out/slots2
B="python bench.py --no-e2e --no-cpu-baseline --warmup 3"
timeout 300 $B --steps 10 > $O/nf.json 2>/dev/null
for r in 4 8; do timeout 300 $B --steps 5 --rank $r > $O/r$r.json 2>/dev/null; done
timeout 900 $B --steps 5 --config y4 > $O/y4.json 2>/dev/null
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/nf_e2e.json 2>/dev/null
