#!/bin/bash
# ncu_export.sh REP: raw + details CSV next to the report, then drop the report
# (keeps gpurun_out under the 64 MiB copy-back limit)
rep=$1
ncu -i $rep --page raw --csv > ${rep%.ncu-rep}.raw.csv 2>/dev/null
ncu -i $rep --page details --csv > ${rep%.ncu-rep}.details.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source sass 2>/dev/null | gzip > ${rep%.ncu-rep}.sass.csv.gz
rm -f $rep
