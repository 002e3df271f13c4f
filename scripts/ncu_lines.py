"""Aggregate an ncu source page (cuda,sass view) by CUDA source line:
stall samples and executed instructions.
usage: ncu_lines.py report.ncu-rep [top] [kernel filter, e.g. regex:k_render]"""
import csv, subprocess, sys, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kfilt = ["-k", sys.argv[3]] if len(sys.argv) > 3 else []   # e.g. regex:k_render
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
                     + kfilt, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data = []; f = "?"; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-": continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        i = int(r[hdr.index("Instructions Executed")] or 0)
    except ValueError:
        continue
    stalls = {h: int(v) for h, v in zip(hdr, r) if h.startswith("stall_") and "Not Issued" not in h and v.isdigit() and int(v) > 0}
    data.append((s, i, f, r[0], r[1][:90], stalls))
ts = sum(d[0] for d in data) or 1; ti = sum(d[1] for d in data) or 1
print(f"samples {ts}  warp-instructions {ti}")
for d in sorted(data, key=lambda d: -d[0])[:top]:
    st = sorted(d[5].items(), key=lambda kv: -kv[1])[:3]
    st = " ".join(f"{k[6:]}:{v*100//max(d[0],1)}" for k, v in st)
    print(f"{d[0]/ts*100:5.1f}%s {d[1]/ti*100:5.1f}%i {d[2]}:{d[3]:<5} {d[4]:<90} [{st}]")
