#!/bin/bash
O=gpurun_out/r2a; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python -m pytest tests/test_facade.py -q -p no:cacheprovider > $O/facade.log 2>&1; echo "rc=$?" >> $O/facade.log
timeout 300 python tools/tc2_stamps.py > $O/stamps.log 2>&1
