#!/usr/bin/env python
"""Compose a profiles/ summary from a tools/gpu_final.sh output directory.

  python tools/profile_summary.py gpurun_out/final profiles/r01_d_final.txt "title"
"""
import json
import os
import subprocess
import sys


def first_json(path):
    try:
        for line in open(path):
            if line.startswith("{"):
                return json.loads(line)
    except OSError:
        pass
    return None


def main():
    src, dst = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else "round record"
    here = os.path.dirname(os.path.abspath(__file__))
    out = [f"# {title}: tools/gpu_final.sh on one B200", ""]
    for name, label in (("pytest_gpu.log", "pytest -m gpu"), ("smoke.log", "smoke()")):
        p = os.path.join(src, name)
        if os.path.exists(p):
            lines = open(p).read().strip().splitlines()
            out += [f"## {label}", *lines[-2:], ""]
    out.append("## bench line (python bench.py)")
    out.append(open(os.path.join(src, "bench.json")).read().strip())
    out.append("")
    out.append("## reference arm (python bench.py --impl reference --steps 2 --warmup 1)")
    out.append(open(os.path.join(src, "bench_ref.json")).read().strip())
    out.append("")
    out.append("## other configurations (bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline unless noted)")
    out.append(f"{'config':34s} {'ms/epoch':>9s} {'G nnz/s':>8s} {'factor ms':>9s} {'kernel':>22s} {'frac':>6s} {'test RMSE':>9s}")
    for f, label in (("bench.json", "NF J=R=16 (headline)"), ("rank4.json", "NF J=R=4"), ("rank8.json", "NF J=R=8"),
                     ("rank32.json", "NF J=R=32"), ("rank64.json", "NF J=R=64 (alpha_a 3e-4)"),
                     ("y4.json", "Y4 250M N=4 J=R=16"), ("o6.json", "O6 1e9 N=6 J=R=8 (3 steps)"),
                     ("cfg1.json", "cfg1 1K^3 90K J=R=8 (10 steps)")):
        d = first_json(os.path.join(src, f))
        if not d:
            continue
        rf = d.get("roofline") or {}
        rm = d.get("test_rmse")
        out.append(f"{label:34s} {d['ms_per_step']:9.2f} {d['value'] / 1e9:8.3f} {rf.get('kernel_ms') or 0:9.2f} "
                   f"{rf.get('kernel', ''):>22s} {rf.get('frac') or 0:6.3f} {rm if rm is None else round(rm, 4)!s:>9s}")
    out.append("")
    out.append("## per-rank DSGD epoch estimates (BENCH_DSGD_SIM=M: one rank's blocks, samplers and core phase, no exchanges)")
    for m in (2, 4, 8):
        d = first_json(os.path.join(src, f"dsgd{m}.json"))
        if d:
            out.append(f"M={m} {d['ms_per_step']:.2f} ms per epoch per rank")
    out.append("")
    tl = os.path.join(src, "bench_tl.err")
    if os.path.exists(tl):
        out.append("## per-epoch stream timeline (ms from epoch start; BENCH_TIMELINE=1)")
        out += [ln.strip() for ln in open(tl) if "timeline" in ln][-2:]
        out.append("")
    out.append("## launch list (2 timed epochs, each also drawing the next epochs' samples)")
    out.append(subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), "--launches",
                               os.path.join(src, "launches.csv"), "--steps", "2"],
                              capture_output=True, text=True).stdout.strip())
    out.append("")
    out.append("## factor kernel, ncu --set full")
    out.append(subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), "--rep",
                               os.path.join(src, "prof_factor.ncu-rep")], capture_output=True, text=True).stdout.strip())
    open(dst, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
