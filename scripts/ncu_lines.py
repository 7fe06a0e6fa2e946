"""Summarise an ncu source page (cuda,sass CSV) per CUDA source line:
warp-stall samples and executed warp instructions, top-N lines."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
file = None
stats = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samples = int(r[4]); inst = int(r[7])
    except (ValueError, IndexError):
        continue
    stats.append((samples, inst, f"{file}:{r[0]}", r[1].strip()[:90]))
tot_s = sum(s[0] for s in stats) or 1
tot_i = sum(s[1] for s in stats) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_i}")
for s in sorted(stats, reverse=True)[:top]:
    print(f"{100*s[0]/tot_s:5.1f}% smp {100*s[1]/tot_i:5.1f}% inst  {s[2]:18s} {s[3]}")
