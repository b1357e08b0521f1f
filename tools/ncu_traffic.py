"""profiles/factor_traffic.json from an ncu --set full capture of the factor kernel."""
import csv, io, json, subprocess, sys
rep, workload = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
vals = []
for r in rows[2:]:
    if "factor" not in r[h.index("Kernel Name")]:
        continue
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = float(r[h.index(k)]); unit = u[h.index(k)]
        tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    vals.append(tot)
out = {"workload": workload, "bytes_per_launch": sum(vals) / len(vals), "launches": len(vals), "source": rep}
json.dump(out, open("profiles/factor_traffic.json", "w"), indent=1)
print(out)
