#!/bin/bash
# Per-rank dynamics of 8-GPU DSGD on one GPU: W=8 blocks launched one by one (SPTK_FLAT=0),
# each block with the full grid in flight (no Hogwild cap) or capped
O=gpurun_out/r2s3g; mkdir -p $O
SPTK_FLAT=0 SPTK_HOGWILD_SPAN=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e --workers 8 --steps 5 > $O/w8_nocap.json 2> $O/w8_nocap.err
SPTK_FLAT=0 SPTK_HOGWILD_SPAN=16 timeout 900 python bench.py --no-cpu-baseline --no-e2e --workers 8 --steps 5 > $O/w8_span16.json 2> $O/w8_span16.err
SPTK_FLAT=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e --workers 8 --steps 5 > $O/w8_span64.json 2> $O/w8_span64.err
