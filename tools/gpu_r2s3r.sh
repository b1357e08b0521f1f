#!/bin/bash
# round table: every config's bench line (no e2e / cpu legs except the headline)
O=gpurun_out/r2s3r; mkdir -p $O
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err
for J in 4 8 32 64; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --rank $J --steps 5 > $O/nf_j$J.json 2> $O/nf_j$J.err
done
timeout 900 python bench.py --config y4 --no-cpu-baseline --no-e2e --steps 5 > $O/y4.json 2> $O/y4.err
timeout 900 python bench.py --config cfg1 --no-cpu-baseline --no-e2e --steps 5 > $O/cfg1.json 2> $O/cfg1.err
timeout 900 python bench.py --config cfg1 --mode hogwild --no-cpu-baseline --no-e2e --steps 5 > $O/cfg1h.json 2> $O/cfg1h.err
timeout 1500 python bench.py --config o6 --no-cpu-baseline --no-e2e --steps 3 > $O/o6.json 2> $O/o6.err
