"""Per-CUDA-source-line summary of one ncu --set full report (run where ncu
is): executed warp instructions and warp-stall samples (with the dominant
stall reason) per line, top N lines, plus totals per stall reason.

usage: python scripts/ncu_lines.py <report.ncu-rep> [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, errors="replace").stdout
rows = list(csv.reader(raw.splitlines()))
hdr, file, cur = None, None, None
lines = collections.OrderedDict()
reasons_tot = collections.Counter()
fn = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        fn = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0] != "":
        cur = (file, r[0], r[1].strip()[:90])
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ins = int(d.get("Instructions Executed") or 0)
        smp = int(d.get("Warp Stall Sampling (All Samples)") or 0)
    except ValueError:
        continue
    e = lines.setdefault(cur, [0, 0, collections.Counter()])
    e[0] += ins
    e[1] += smp
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k and v and v.isdigit():
            e[2][k[6:]] += int(v)
            reasons_tot[k[6:]] += int(v)
ti = sum(v[0] for v in lines.values()) or 1
ts = sum(v[1] for v in lines.values()) or 1
print(f"{fn}\nwarp instructions {ti}, stall samples {ts}")
print("stall reasons: " + ", ".join(f"{k} {100 * v / ts:.1f}%" for k, v in reasons_tot.most_common(8)))
print(f"{'inst%':>6} {'stall%':>6}  top-stall          line")
for k, v in sorted(lines.items(), key=lambda kv: -(kv[1][0] / ti + kv[1][1] / ts))[:top]:
    if k is None:
        continue
    reason = v[2].most_common(1)[0][0] if v[2] else "-"
    print(f"{100 * v[0] / ti:6.1f} {100 * v[1] / ts:6.1f}  {reason:18s} {k[0]}:{k[1]} {k[2]}")
