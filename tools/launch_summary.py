"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(f) if not l.startswith("==")))
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows:
        k = r[ki].split("(")[0][:80]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f, "total ms", round(tot / 1e6, 3))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{v[1] / 1e6:9.3f} ms {v[0]:6d}  {k}")
