"""Per-kernel ncu summaries from one `ncu --set full` capture of a C3 view
(scripts/ncu_capture.sh): for every in-repo kernel K0..K6, the duration,
DRAM bytes read + written, achieved DRAM GB/s against the measured HBM peak,
SM / DRAM speed-of-light, issue-slot and FP64-pipe utilisation, achieved
occupancy, registers, and the top warp-stall reasons (cycles per issued
instruction).  Writes profiles/<tag>/ncu_<kernel>.txt, profiles/<tag>/
ncu_kernels.txt (the table) and profiles/ncu_kernels.json (what bench.py
attaches to roofline.per_kernel).

usage: python scripts/ncu_kernels.py TAG [rep]   (rep default gpurun_out/TAG/full.ncu-rep)
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rep = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", tag, "full.ncu-rep")
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0

# bench.py KERNELS groups (K2 = 3 scan launches, K3 = duplicate + row duplicate, ...)
GROUP = [("K0 init", ("k_init",)),
         ("K1 preprocess", ("k_preprocess", "k_rows_count")),
         ("K2 scan", ("k_scan_partials", "k_scan_top", "k_scan_final")),
         ("K3 duplicate", ("k_duplicate", "k_rows_dup")),
         ("K4 sort", ("k_sort_hist", "k_onesweep")),
         ("K5 ranges", ("k_ranges",)),
         ("K6 render", ("k_render", "k_render_globalz", "k_render_pixelsort",
                        "k_render_window"))]

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def num(r, name, default=None):
    i = col.get(name)
    if i is None or i >= len(r):
        return default
    v = r[i].replace(",", "").strip()
    try:
        return float(v)
    except ValueError:
        return default


def unit(name):
    return units[col[name]] if name in col else ""


def base(name):
    n = re.sub(r"^void ", "", name).split("(")[0].split("<")[0]
    return n.split("::")[-1]


def to_us(v, u):
    return v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                "msecond": 1e3, "s": 1e6, "second": 1e6}.get(u, 1.0)


def to_bytes(v, u):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


STALL = re.compile(r"smsp__average_warps_issue_stalled_(.+)_per_issue_active\.ratio$")
stall_cols = [(m.group(1), h) for h in hdr for m in [STALL.match(h)] if m]
fp64_cols = [h for h in ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                         "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
             if h in col]
launches = collections.OrderedDict()
for r in data:
    k = base(r[col["Kernel Name"]])
    d = {
        "us": to_us(num(r, "gpu__time_duration.sum", 0.0), unit("gpu__time_duration.sum")),
        "dram_read": to_bytes(num(r, "dram__bytes_read.sum", 0.0), unit("dram__bytes_read.sum")),
        "dram_write": to_bytes(num(r, "dram__bytes_write.sum", 0.0),
                               unit("dram__bytes_write.sum")),
        "dram_sol": num(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_sol": num(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "issue": num(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "occ": num(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "regs": num(r, "launch__registers_per_thread"),
        "ipc": num(r, "sm__inst_executed.avg.per_cycle_active"),
        "grid": r[col["Grid Size"]] if "Grid Size" in col else "",
        "block": r[col["Block Size"]] if "Block Size" in col else "",
        "fp64": {h: num(r, h) for h in fp64_cols},
        "stalls": {nm: num(r, h, 0.0) for nm, h in stall_cols},
    }
    launches.setdefault(k, []).append(d)

summary = {"source": os.path.relpath(rep, ROOT), "peak_gbs": PEAK, "kernels": {}, "launches": {}}
lines = [f"# ncu --set full --clock-control none, one C3 view (cold caches, serialised); "
         f"HBM peak {PEAK:.0f} GB/s (MEASURED_PEAKS.json)",
         f"{'kernel':22s} {'n':>2s} {'us':>8s} {'DRAM MB':>8s} {'GB/s':>7s} {'%peak':>6s} "
         f"{'SM%':>5s} {'issue%':>6s} {'occ%':>5s} {'regs':>4s}  top stalls (cycles/issue)"]
for k, ls in launches.items():
    us = sum(x["us"] for x in ls)
    by = sum(x["dram_read"] + x["dram_write"] for x in ls)
    gbs = by / (us * 1e-6) / 1e9 if us else 0.0
    w = [x["us"] for x in ls]

    def wavg(key):
        vals = [(x[key], x["us"]) for x in ls if x[key] is not None]
        return sum(v * t for v, t in vals) / max(sum(t for _, t in vals), 1e-9) if vals else None

    st = collections.Counter()
    for x in ls:
        for nm, v in x["stalls"].items():
            st[nm] += v * x["us"] / max(sum(w), 1e-9)
    top = [(nm, round(v, 3)) for nm, v in st.most_common(5)]
    fp = {}
    for h in fp64_cols:
        vals = [(x["fp64"][h], x["us"]) for x in ls if x["fp64"].get(h) is not None]
        if vals:
            fp[h] = sum(v * t for v, t in vals) / max(sum(t for _, t in vals), 1e-9)
    rec = {"launches": len(ls), "us": us, "dram_bytes": by, "achieved_gbs": gbs,
           "frac_of_peak": gbs / PEAK, "dram_sol_pct": wavg("dram_sol"),
           "sm_sol_pct": wavg("sm_sol"), "issue_active_pct": wavg("issue"),
           "achieved_occupancy_pct": wavg("occ"), "ipc": wavg("ipc"),
           "registers": ls[0]["regs"], "grid": ls[0]["grid"], "block": ls[0]["block"],
           "top_stalls": top, "fp64_pct": fp}
    summary["launches"][k] = rec
    lines.append(f"{k:22s} {len(ls):2d} {us:8.1f} {by / 1e6:8.1f} {gbs:7.0f} {100 * gbs / PEAK:6.1f} "
                 f"{rec['sm_sol_pct'] or 0:5.1f} {rec['issue_active_pct'] or 0:6.1f} "
                 f"{rec['achieved_occupancy_pct'] or 0:5.1f} {int(rec['registers'] or 0):4d}  "
                 + ", ".join(f"{n} {v:.2f}" for n, v in top[:3]))
    with open(os.path.join(dst, f"ncu_{k}.txt"), "w") as f:
        f.write(f"# {k}: {len(ls)} launch(es) of one C3 view, ncu --set full ({summary['source']})\n")
        f.write(json.dumps(rec, indent=1) + "\n")

for g, names in GROUP:
    parts = [summary["launches"][n] for n in names if n in summary["launches"]]
    if not parts:
        continue
    us = sum(p["us"] for p in parts)
    by = sum(p["dram_bytes"] for p in parts)
    main = max(parts, key=lambda p: p["us"])
    fp = main["fp64_pct"].get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
    summary["kernels"][g] = {
        "us_ncu": us, "dram_bytes_per_view": by, "dram_gbs_ncu": by / (us * 1e-6) / 1e9,
        "dram_frac_of_peak_ncu": by / (us * 1e-6) / 1e9 / PEAK,
        "issue_active_frac": (main["issue_active_pct"] or 0) / 100.0,
        "fp64_pipe_frac": fp / 100.0 if fp is not None else None,
        "achieved_occupancy": (main["achieved_occupancy_pct"] or 0) / 100.0,
        "top_stalls": main["top_stalls"], "kernels": [n for n in names if n in summary["launches"]]}

with open(os.path.join(dst, "ncu_kernels.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
    if fp64_cols:
        f.write("\nFP64 pipe columns: " + ", ".join(fp64_cols) + "\n")
with open(os.path.join(ROOT, "profiles", "ncu_kernels.json"), "w") as f:
    json.dump(summary, f, indent=1)
print("\n".join(lines))
