"""Summarise the ncu artefacts of one GPU round trip (gpurun_out/) into
profiles/<tag>/ (tracked): per-kernel launch list, the dominant kernel's
SOL / occupancy / stall summary, its source-line hot spots and the
dram traffic per launch that bench.py reports as roofline.traffic.

usage: python scripts/summarize_profiles.py TAG [render_report_tag]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rtag = sys.argv[2] if len(sys.argv) > 2 else tag
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)

# 1. launch list: per-kernel mean duration and share of one view
rows = list(csv.reader(open(os.path.join(src, f"launches_{tag}.csv"))))
hdr, d = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        k = r[hdr.index("Kernel Name")].split("(")[0]
        d.setdefault(k, []).append(float(r[hdr.index("Metric Value")]) / 1e3)
views = len(d.get("k_init", [1]))
tot = sum(sum(v) for v in d.values()) / views
with open(os.path.join(dst, "launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised)\n")
    f.write(f"# {views} views of bench.py; per-view sum of kernel times {tot:.1f} us\n")
    f.write(f"{'kernel':44s} {'launches/view':>13s} {'mean us':>10s} {'us/view':>10s} {'share':>7s}\n")
    for k, v in d.items():
        per_view = sum(v) / views
        f.write(f"{k:44s} {len(v)/views:13.1f} {sum(v)/len(v):10.1f} {per_view:10.1f} "
                f"{per_view/tot*100:6.1f}%\n")
print(open(os.path.join(dst, "launches.txt")).read())

# 2. dominant-kernel capture: details + raw metrics + source hot spots
rep = os.path.join(src, f"prof_render_{rtag}.ncu-rep")
if os.path.exists(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    keep = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Memory Workload Analysis",
            "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Launch Statistics",
            "Instruction Statistics")
    lines = []
    dr = list(csv.reader(io.StringIO(det)))
    dh = dr[0]
    si, mi, ui, vi = (dh.index(c) for c in ("Section Name", "Metric Name", "Metric Unit",
                                             "Metric Value"))
    for r in dr[1:]:
        if len(r) > vi and r[si] in keep and r[mi]:
            lines.append(f"{r[si]:32s} | {r[mi]:45s} | {r[vi]:>16s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, u, v = rr[0], rr[1], rr[2]
    def metric(name):
        i = h.index(name)
        x = float(v[i].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                 "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(u[i], 1)
        return x * scale
    rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
    dur = metric("gpu__time_duration.sum")
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warp_latency_issue_stalled_") or \
           name.startswith("smsp__average_warps_issue_stalled_"):
            if name.endswith("_per_issue_active.ratio"):
                try:
                    stalls[name.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = \
                        float(v[i])
                except ValueError:
                    pass
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:10]
    with open(os.path.join(dst, "k_render_ncu.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, one k_render launch ({rep.split('/')[-1]})\n")
        f.write(f"# dram read {rd/1e6:.1f} MB + write {wr/1e6:.1f} MB = {(rd+wr)/1e6:.1f} MB per launch,"
                f" {dur*1e3:.3f} ms\n")
        f.write("\n".join(lines) + "\n\n# warp stall reasons (cycles per issued instruction)\n")
        for k, x in top:
            f.write(f"{k:32s} {x:8.3f}\n")
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_lines.py"), rep, "50"],
                         capture_output=True, text=True).stdout
    with open(os.path.join(dst, "k_render_hotspots.txt"), "w") as f:
        f.write("# stall samples (%s) and executed warp instructions (%i) per CUDA source line\n")
        f.write(hot)
    with open(os.path.join(ROOT, "profiles", "k6_traffic.json"), "w") as f:
        json.dump({"kernel": "k_render", "bytes_per_launch": rd + wr, "dram_read": rd,
                   "dram_write": wr, "duration_s_under_ncu": dur, "source": f"profiles/{tag}"}, f,
                  indent=1)
    print(open(os.path.join(dst, "k_render_ncu.txt")).read()[:3000])
