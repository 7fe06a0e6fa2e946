"""Executed-instruction mix per SASS opcode of an ncu report (source page,
sass view): python scripts/ncu_opmix.py <report.ncu-rep> [top]."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
cnt = collections.Counter()
for r in rows[2:]:
    if len(r) <= ie:
        continue
    ins = r[1].strip().split()
    if not ins:
        continue
    op = ins[1] if ins[0].startswith("@") else ins[0]
    try:
        cnt[op.split(".")[0]] += int(r[ie])
    except ValueError:
        pass
tot = sum(cnt.values())
print(f"warp instructions {tot / 1e6:.1f}M")
for op, c in cnt.most_common(top):
    print(f"{op:12s} {100 * c / tot:5.1f}%")
