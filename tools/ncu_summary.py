#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (gpu__time_duration csv)
and/or a --set full report (.ncu-rep), read here with `ncu -i`.

  python tools/ncu_summary.py --launches gpurun_out/launches.csv --steps 2
  python tools/ncu_summary.py --rep gpurun_out/prof_factor.ncu-rep
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= mi:
            continue
        k = re.sub(r"\(.*", "", r[ki])[:60]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[mi].replace(",", "")) / 1e6
    tot = sum(v[1] for v in agg.values())
    out = [f"launch list {path}: {sum(v[0] for v in agg.values())} launches, {tot:.3f} ms total "
           f"(ncu-serialised, cold cache) over {steps} step(s) -> {tot / steps:.3f} ms/step"]
    out.append(f"{'launches':>8} {'ms':>9} {'share':>6}  kernel")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{n:8d} {v:9.3f} {100 * v / tot:5.1f}%  {k}")
    return "\n".join(out)


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"ncu --set full report {path}"]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"kernel: {re.sub(r'[(].*', '', name)[:80]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k} = {r[i]} {units[i]}")
        stalls = []
        for i, k in enumerate(hdr):
            m = re.match(r"smsp__average_warp(s_issue_stalled|_latency_issue_stalled)_(\w+)_per_issue_active\.ratio", k)
            if m:
                try:
                    stalls.append((float(r[i]), m.group(2)))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            out.append("  top stalls (cycles per issued instruction): " +
                       ", ".join(f"{n}={v:.2f}" for v, n in stalls[:8]))
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--rep", action="append", default=[])
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches, a.steps))
    for p in a.rep:
        print(rep(p))
